// spmm_inst_x16_sum.cu -- bf16-storage gSpMM instantiations, reducer sum.
#define FG_RED R_SUM
#include "spmm_inst_x16.cuh"
