// K2: sequential Adagrad trainer -- placeholder until the persistent kernel lands.
#include "common.cuh"

using namespace dffm;

extern "C" int64_t dffm_train_scratch_bytes(const dffm_model*, int32_t) { return 0; }

extern "C" int dffm_train_sequential(const dffm_model*, const dffm_train_state*, const int32_t*,
                                     const float*, const uint8_t*, int32_t, int64_t, double*,
                                     void*, uint64_t*, void*) {
  set_error("dffm_train_sequential: not built in this revision");
  return DFFM_SIZING;
}
