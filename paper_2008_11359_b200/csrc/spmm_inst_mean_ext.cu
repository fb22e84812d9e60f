// spmm_inst_mean_ext.cu -- gSpMM instantiations: reducer mean, u_add_e / copy_e (row f4).
#define FG_RED R_MEAN
#define FG_OPSET 1
#include "spmm_inst.cuh"
