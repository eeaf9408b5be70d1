// Fused sm_100a kernels for 65536-sample chunks: placeholder until the
// cluster kernels land (the generic path handles every length meanwhile).
#include "fgc_internal.h"

namespace fgc {

struct FusedTables {};

bool fused_available() { return false; }
fgc_status fused_tables_init(FusedTables** t, cudaStream_t) {
  *t = nullptr;
  set_error("fused kernels unavailable");
  return FGC_ERR_UNSUPPORTED;
}
void fused_tables_free(FusedTables*) {}
fgc_status launch_fused_compress(const FusedTables*, const ChunkInfo*, uint32_t, uint32_t, const void*, int, int,
                                 const QuantParams&, uint8_t*, uint32_t*, cudaStream_t) {
  return FGC_ERR_UNSUPPORTED;
}
fgc_status launch_fused_decode(const FusedTables*, const ChunkInfo*, uint32_t, uint32_t, const uint8_t*, int,
                               uint64_t, const Weights&, const QuantParams&, float*, cudaStream_t) {
  return FGC_ERR_UNSUPPORTED;
}
fgc_status launch_fused_spectrum(const FusedTables*, const ChunkInfo*, uint32_t, uint32_t, const void*, int, int,
                                 float2*, uint32_t*, cudaStream_t) {
  return FGC_ERR_UNSUPPORTED;
}
fgc_status launch_fused_inverse(const FusedTables*, const ChunkInfo*, uint32_t, uint32_t, const float2*, float*,
                                cudaStream_t) {
  return FGC_ERR_UNSUPPORTED;
}

}  // namespace fgc
