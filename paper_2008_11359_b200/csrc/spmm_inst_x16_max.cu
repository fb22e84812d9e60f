// spmm_inst_x16_max.cu -- bf16-storage gSpMM instantiations, reducer max.
#define FG_RED R_MAX
#include "spmm_inst_x16.cuh"
