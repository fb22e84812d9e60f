// spmm_inst_mean_base.cu -- gSpMM instantiations: reducer mean, copy_u / u_mul_e.
#define FG_RED R_MEAN
#define FG_OPSET 0
#include "spmm_inst.cuh"
