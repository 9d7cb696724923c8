// K5: backward of the gathered sparse flash attention (placeholder until the
// tcgen05 backward lands; returns PARAM so callers fail loudly).
#include "common.cuh"

extern "C" size_t omni_sparse_attn_bwd_workspace(int n_q_heads, int seq_len) {
  return 16;
}

extern "C" int omni_sparse_attn_bwd(const void*, const void*, const void*, const void*, const void*, const float*,
                                    const int32_t*, const int32_t*, const int32_t*, const int32_t*, int, int, int,
                                    int, int, float*, float*, float*, float*, void*, void*) {
  OMNI_CHECK(false, OMNI_E_PARAM, "sparse attention backward not built yet");
  return OMNI_OK;
}
