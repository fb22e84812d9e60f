// spmm_inst_sum_base.cu -- gSpMM instantiations: reducer sum, copy_u / u_mul_e.
#define FG_RED R_SUM
#define FG_OPSET 0
#include "spmm_inst.cuh"
