// spmm_inst_x16_min.cu -- bf16-storage gSpMM instantiations, reducer min.
#define FG_RED R_MIN
#include "spmm_inst_x16.cuh"
