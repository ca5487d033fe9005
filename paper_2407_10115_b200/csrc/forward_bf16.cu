// K1 instantiation for bf16 tables.
#define DFFM_INST_T __nv_bfloat16
#include "forward_inst.cuh"
