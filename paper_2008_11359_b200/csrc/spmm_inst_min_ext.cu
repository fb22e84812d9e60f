// spmm_inst_min_ext.cu -- gSpMM instantiations: reducer min, u_add_e / copy_e (row f4).
#define FG_RED R_MIN
#define FG_OPSET 1
#include "spmm_inst.cuh"
