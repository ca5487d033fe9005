// K1 instantiation for f32 tables.
#define DFFM_INST_T float
#include "forward_inst.cuh"
