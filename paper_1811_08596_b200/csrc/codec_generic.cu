// Generic-length codec kernels: count-mode selection + quantize + pack from
// a spectrum in global memory, and the decode + weighted accumulate of W
// messages.  Used for tail chunks, any chunk length the fused kernels
// (fused.cu) do not take, and the stage-injection entry point.
//
// Reference stages restated here:
//   truncate, count mode    spectral.py:124-156 (stable argsort, k = ceil(theta*bins))
//   _interleave + encode    codec.py:174-180, 197-202; quantizer.py:217-236
//   pack + bitmap bytes     packer.py:41-58, 73-75; quantizer.py:266-273
//   unpack + decode + avg   packer.py:61-70, quantizer.py:239-253, simulator.py:547
#include <cuda_runtime.h>
#include <math.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"
#include "select_pack.cuh"
#include "decode_acc.cuh"

namespace fgc {

namespace {

inline uint32_t cdiv(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

// ------------------------------------------------------------- select + pack

using namespace sel;

template <typename CT, int TH = kSelThreads>
__global__ void __launch_bounds__(TH) k_select_pack(const ChunkInfo* chunks, uint32_t first, Coeffs<CT> coeffs,
                                                    int exact_only, QuantParams q, uint8_t* message,
                                                    uint8_t* kept_mask, uint32_t* flags,
                                                    const uint32_t* only_if, PieceCounter pc,
                                                    const uint8_t* drop_mask) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SelectSharedT<TH>& sh = *reinterpret_cast<SelectSharedT<TH>*>(smem_raw);
  if (only_if && only_if[first + blockIdx.x] == 0u) return;
  const ChunkInfo ci = chunks[first + blockIdx.x];
  Coeffs<CT> cf = coeffs;
  cf.p += ci.bin_off;
  select_pack_chunk<CT, TH>(sh, ci, cf, exact_only, q, message, kept_mask, flags, drop_mask);
  if (pc.cnt) {                                  // segment complete: count it for the exchange
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) atomicAdd(&pc.cnt[(first + blockIdx.x - pc.first) / pc.per], 1u);
  }
}

// ------------------------------------------------------------- decode + accumulate

constexpr int kDecThreads = 512;

template <int kDecThreads>
__global__ void __launch_bounds__(kDecThreads) k_decode_accumulate(const ChunkInfo* chunks, uint32_t first,
                                                                   const uint8_t* messages, int W, int w0, int G,
                                                                   uint64_t stride, Weights wts, QuantParams q,
                                                                   float2* spectrum) {
  extern __shared__ __align__(16) uint32_t pref[];    // G x bm_words exclusive popcount prefixes
  __shared__ uint32_t scan[40];
  decode_accumulate_chunk<kDecThreads>(chunks[first + blockIdx.x], messages, W, w0, G, stride, wts, q, spectrum,
                                       pref, scan);
}

}  // namespace

// ------------------------------------------------------------- launchers

fgc_status launch_select_pack(const ChunkInfo* d_chunks, uint32_t first, uint32_t count, const void* spectrum,
                              int coeff_f64, const QuantParams& q, uint8_t* message, uint8_t* kept_mask,
                              uint32_t* flags, cudaStream_t s, const uint32_t* only_if, PieceCounter pc,
                              const uint8_t* drop_mask) {
  if (!count) return FGC_OK;
  static bool attr = false;
  const size_t smem = sizeof(SelectShared);
  constexpr int kWide = 1024;
  const size_t smem_w = sizeof(SelectSharedT<kWide>);
  if (!attr) {
    FGC_CUDA(cudaFuncSetAttribute(k_select_pack<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FGC_CUDA(cudaFuncSetAttribute(k_select_pack<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    FGC_CUDA(cudaFuncSetAttribute(k_select_pack<float2, kWide>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem_w));
    attr = true;
  }
  // a few chunks (a plan's tail class beside the fused grid): one wide CTA
  // each -- the chunk's select + pack is a latency chain of tiles, and the
  // tail's kernel chain runs beside the fused grid on the side stream
  static const int wide = [] { const char* e = getenv("FGC_WIDE_TAIL"); return e ? atoi(e) : 1; }();
  if (!coeff_f64 && wide && count <= 4) {
    Coeffs<float2> c{static_cast<const float2*>(spectrum)};
    k_select_pack<float2, kWide><<<count, kWide, smem_w, s>>>(d_chunks, first, c, 0, q, message, kept_mask, flags,
                                                              only_if, pc, drop_mask);
    FGC_LAUNCHED(1);
    return FGC_OK;
  }
  if (coeff_f64) {
    Coeffs<double2> c{static_cast<const double2*>(spectrum)};
    k_select_pack<double2><<<count, kSelThreads, smem, s>>>(d_chunks, first, c, 1, q, message, kept_mask, flags,
                                                            only_if, pc, drop_mask);
  } else {
    Coeffs<float2> c{static_cast<const float2*>(spectrum)};
    k_select_pack<float2><<<count, kSelThreads, smem, s>>>(d_chunks, first, c, 0, q, message, kept_mask, flags,
                                                           only_if, pc, drop_mask);
  }
  FGC_LAUNCHED(1);
  return FGC_OK;
}

// Sender-side reconstruction error by Parseval (the simulator's err_ratio,
// simulator.py:538-542, without a decode): per chunk,
//   err  = (1/L) sum_k w_k |X_k - Xhat_k|^2 = ||x - decompress(compress(x))||^2
//   norm = (1/L) sum_k w_k |X_k|^2          = ||x||^2
// with w_k the Parseval weights (spectral.py:109-115; the imaginary parts of
// DC / Nyquist count as the inverse transform ignores them) and Xhat the
// dequantized kept slots of the chunk's message.
__global__ void __launch_bounds__(kDecThreads) k_spectrum_error(const ChunkInfo* chunks, const float2* spectrum,
                                                                 const uint8_t* message, QuantParams q,
                                                                 double2* out) {
  extern __shared__ __align__(16) uint32_t epref[];   // bm_words exclusive popcount prefixes
  __shared__ uint32_t scan[40];
  __shared__ double red[2][kDecThreads / 32];
  const ChunkInfo ci = chunks[blockIdx.x];
  const uint32_t bm_words = (ci.slots + 31) / 32, tid = threadIdx.x;
  const uint8_t* seg = message + ci.seg_off;
  const uint32_t* bm = reinterpret_cast<const uint32_t*>(seg + kSegHeader);
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(seg + ci.code_off);
  const uint32_t per = (bm_words + kDecThreads - 1) / kDecThreads;
  {
    uint32_t local = 0;
    const uint32_t a = tid * per, b = min(bm_words, a + per);
    for (uint32_t w = a; w < b; ++w) local += __popc(bm[w]);
    uint32_t tot;
    uint32_t base = block_exclusive_scan<kDecThreads>(local, scan, tot);
    for (uint32_t w = a; w < b; ++w) {
      epref[w] = base;
      base += __popc(bm[w]);
    }
  }
  __syncthreads();
  const int N = q.n_bits;
  const bool even = (ci.len % 2u) == 0u;
  double e = 0.0, nrm = 0.0;
  for (uint32_t i = tid; i < ci.bins; i += kDecThreads) {
    const float2 X = spectrum[ci.bin_off + i];
    const uint32_t slot = 2 * i, word = slot >> 5, sh = slot & 31u;
    const uint32_t sw = ballot_to_wire(bm[word]);
    const uint32_t bits = (sw >> sh) & 3u;
    float re = 0.f, im = 0.f;
    uint32_t r = epref[word] + __popc(sw & ((1u << sh) - 1u));
    if (bits & 1u) { re = decode_code(q, read_bits(cw, (uint64_t)r * N, N)); ++r; }
    if (bits & 2u) im = decode_code(q, read_bits(cw, (uint64_t)r * N, N));
    const bool edge = i == 0 || (even && i == ci.bins - 1);
    const double w = edge ? 1.0 : 2.0;
    const double dr = (double)X.x - (double)re, di = edge ? 0.0 : (double)X.y - (double)im;
    const double xi = edge ? 0.0 : (double)X.y;
    e += w * (dr * dr + di * di);
    nrm += w * ((double)X.x * X.x + xi * xi);
  }
  for (int d = 16; d > 0; d >>= 1) {
    e += __shfl_down_sync(0xffffffffu, e, d);
    nrm += __shfl_down_sync(0xffffffffu, nrm, d);
  }
  if ((tid & 31) == 0) { red[0][tid >> 5] = e; red[1][tid >> 5] = nrm; }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < kDecThreads / 32; ++k) { a += red[0][k]; b += red[1][k]; }
    out[blockIdx.x] = make_double2(a / (double)ci.len, b / (double)ci.len);
  }
}

fgc_status launch_spectrum_error(const ChunkInfo* d_chunks, uint32_t n_chunks, uint32_t max_slots,
                                 const float2* spectrum, const uint8_t* message, const QuantParams& q, double2* out,
                                 cudaStream_t s) {
  if (!n_chunks) return FGC_OK;
  const size_t smem = ((max_slots + 31) / 32) * 4ull;
  if (smem > 200 * 1024) {
    set_error("chunk too large for the error kernel");
    return FGC_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    FGC_CUDA(cudaFuncSetAttribute(k_spectrum_error, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    attr = true;
  }
  k_spectrum_error<<<n_chunks, kDecThreads, smem, s>>>(d_chunks, spectrum, message, q, out);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_decode_accumulate(const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                    const uint8_t* messages, int W, uint64_t stride, const Weights& wts,
                                    const QuantParams& q, float2* spectrum, uint32_t max_slots, cudaStream_t s) {
  if (!count) return FGC_OK;
  const uint32_t bm_words = (max_slots + 31) / 32;
  const size_t budget = 200 * 1024;
  const size_t gmax = budget / (bm_words * 4ull);
  int G = (int)((size_t)W < gmax ? (size_t)W : gmax);
  if (G < 1) {
    set_error("chunk too large for the decode prefix tables");
    return FGC_ERR_UNSUPPORTED;
  }
  static bool attr = false;
  if (!attr) {
    FGC_CUDA(cudaFuncSetAttribute(k_decode_accumulate<kDecThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)budget));
    FGC_CUDA(cudaFuncSetAttribute(k_decode_accumulate<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)budget));
    attr = true;
  }
  for (int w0 = 0; w0 < W; w0 += G) {
    const size_t smem = (size_t)G * bm_words * 4;
    static const int wide = [] { const char* e = getenv("FGC_WIDE_TAIL"); return e ? atoi(e) : 1; }();
    if (wide && count <= 4)          // a few chunks (a plan's tail class): one wide CTA each
      k_decode_accumulate<1024><<<count, 1024, smem, s>>>(d_chunks, first, messages, W, w0, G, stride, wts, q,
                                                          spectrum);
    else
      k_decode_accumulate<kDecThreads><<<count, kDecThreads, smem, s>>>(d_chunks, first, messages, W, w0, G, stride,
                                                                        wts, q, spectrum);
    FGC_LAUNCHED(1);
  }
  return FGC_OK;
}

}  // namespace fgc
