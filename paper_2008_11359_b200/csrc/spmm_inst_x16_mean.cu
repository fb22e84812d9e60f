// spmm_inst_x16_mean.cu -- bf16-storage gSpMM instantiations, reducer mean.
#define FG_RED R_MEAN
#include "spmm_inst_x16.cuh"
