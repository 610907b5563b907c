// fused.cu -- single-pass fused decode kernels (placeholder until v2).
#include "common.cuh"

extern "C" int bh_fused_supported(const bh_stream*, int) { return 0; }
extern "C" size_t bh_fused_workspace_bytes(const bh_stream*, int, const bh_tune*) { return 0; }
extern "C" int bh_fused_decode(const bh_stream*, int, const bh_tune*, uint16_t*, void*, size_t, void*, void*) {
  return BH_BAD_ARGUMENT;
}
