// K1 instantiation for u16 tables.
#define DFFM_INST_T uint16_t
#include "forward_inst.cuh"
