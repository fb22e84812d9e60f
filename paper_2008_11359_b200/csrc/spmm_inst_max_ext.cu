// spmm_inst_max_ext.cu -- gSpMM instantiations: reducer max, u_add_e / copy_e (row f4).
#define FG_RED R_MAX
#define FG_OPSET 1
#include "spmm_inst.cuh"
