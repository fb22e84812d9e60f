// spmm_inst_sum_ext.cu -- gSpMM instantiations: reducer sum, u_add_e / copy_e (row f4).
#define FG_RED R_SUM
#define FG_OPSET 1
#include "spmm_inst.cuh"
