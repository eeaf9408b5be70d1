// Weighted accumulation of W messages' codes into one chunk's dense
// spectrum by one CTA of TH threads (codec.py:246-270 per message, the
// averaging sum of simulator.py:547 in the frequency domain): the generic
// decode (codec_generic.cu) and the single-CTA tail chain (real_fft.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {

// Messages [w0, w0 + G) of W into spectrum[bin_off .. bin_off + bins)
// (accumulating onto the previous groups' sums when w0 > 0).  pref: shared
// memory for G x bm_words prefixes; scan: >= 40 words.
template <int TH>
__device__ __forceinline__ void decode_accumulate_chunk(const ChunkInfo ci, const uint8_t* messages, int W, int w0,
                                                        int G, uint64_t stride, const Weights& wts,
                                                        const QuantParams& q, float2* spectrum, uint32_t* pref,
                                                        uint32_t* scan) {
  const uint32_t bm_words = (ci.slots + 31) / 32;
  const uint32_t tid = threadIdx.x;
  const int gn = min(G, W - w0);
  // prefix tables: each thread owns a contiguous run of words
  const uint32_t per = (bm_words + TH - 1) / TH;
  for (int g = 0; g < gn; ++g) {
    const uint32_t* bm = reinterpret_cast<const uint32_t*>(messages + (uint64_t)(w0 + g) * stride + ci.seg_off + kSegHeader);
    uint32_t local = 0;
    const uint32_t a = tid * per, b = min(bm_words, a + per);
    for (uint32_t w = a; w < b; ++w) local += __popc(bm[w]);
    uint32_t tot;
    uint32_t base = block_exclusive_scan<TH>(local, scan, tot);
    for (uint32_t w = a; w < b; ++w) {
      pref[g * bm_words + w] = base;
      base += __popc(bm[w]);
    }
  }
  __syncthreads();
  const int N = q.n_bits;
  for (uint32_t i = tid; i < ci.bins; i += TH) {
    float2 acc = make_float2(0.f, 0.f);
    if (w0 > 0) acc = spectrum[ci.bin_off + i];
    const uint32_t slot = 2 * i;
    const uint32_t word = slot >> 5, sh = slot & 31u;
    for (int g = 0; g < gn; ++g) {
      const uint8_t* seg = messages + (uint64_t)(w0 + g) * stride + ci.seg_off;
      const uint32_t* bm = reinterpret_cast<const uint32_t*>(seg + kSegHeader);
      const uint32_t* cw = reinterpret_cast<const uint32_t*>(seg + ci.code_off);
      const uint32_t sw = ballot_to_wire(bm[word]);          // slot order
      const uint32_t bits = (sw >> sh) & 3u;
      if (!bits) continue;
      uint32_t r = pref[g * bm_words + word] + __popc(sw & ((1u << sh) - 1u));
      float re = 0.f, im = 0.f;
      if (bits & 1u) { re = decode_code(q, read_bits(cw, (uint64_t)r * N, N)); ++r; }
      if (bits & 2u) im = decode_code(q, read_bits(cw, (uint64_t)r * N, N));
      const float wt = wts.w[w0 + g];
      acc.x = __fmaf_rn(wt, re, acc.x);
      acc.y = __fmaf_rn(wt, im, acc.y);
    }
    spectrum[ci.bin_off + i] = acc;
  }
}

}  // namespace fgc
