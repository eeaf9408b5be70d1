// Generic count-mode selection + quantize + pack of ONE chunk by one CTA of
// TH threads (default kSelThreads), from coefficients in global memory.  Shared by the
// generic kernel (codec_generic.cu) and the fused compress kernel, which
// hands a degenerate chunk to it in place (fused.cu).
//
//   truncate, count mode    spectral.py:124-156 (stable argsort, k = ceil(theta*bins))
//   _interleave + encode    codec.py:174-180, 197-202; quantizer.py:217-236
//   pack + bitmap bytes     packer.py:41-58, 73-75; quantizer.py:266-273
#pragma once
#include <cuda_runtime.h>
#include <math.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {
namespace sel {
namespace {                         // internal linkage: each including unit has its own copy

constexpr int kSelThreads = 512;
constexpr int kCandCap = 1024;
constexpr uint32_t kHistBins = 2048;

constexpr int kPer = 4;                                   // bins per thread per final-pass tile
static_assert(16 % kPer == 0 || kPer == 16, "a lane group owns whole bitmap words");

template <int TH>
struct SelectSharedT {
  static constexpr uint32_t kTile = kPer * TH;
  static constexpr uint32_t kStageWords = 2 * kTile + 4;  // one tile of codes (<= 2 kTile codes * 32 bits)
  uint32_t hist[kHistBins];
  uint32_t scan[40];
  unsigned long long key[kCandCap];
  uint32_t idx[kCandCap];
  uint32_t stage[kStageWords];
  uint32_t cnt;
  uint32_t found_bucket, found_below;
};
using SelectShared = SelectSharedT<kSelThreads>;

template <typename CT>
struct Coeffs;
template <>
struct Coeffs<float2> {
  const float2* p;
  __device__ __forceinline__ void get(uint64_t i, float& re, float& im, double& dre, double& dim) const {
    const float2 v = p[i];
    re = v.x; im = v.y; dre = v.x; dim = v.y;
  }
};
template <>
struct Coeffs<double2> {
  const double2* p;
  __device__ __forceinline__ void get(uint64_t i, float& re, float& im, double& dre, double& dim) const {
    const double2 v = p[i];
    dre = v.x; dim = v.y; re = (float)v.x; im = (float)v.y;   // float32(coefficient)
  }
};

// Visit every bin of the chunk, each thread kFly bins per round with their
// loads issued together (the passes are latency-bound on these loads otherwise).
constexpr int kFly = 4;
template <int TH, typename CT, typename F>
__device__ __forceinline__ void for_bins(const Coeffs<CT>& cf, uint32_t B, F&& f) {
  for (uint32_t i0 = threadIdx.x; i0 < B; i0 += kFly * TH) {
    float re[kFly], im[kFly];
    double dr[kFly], di[kFly];
#pragma unroll
    for (int u = 0; u < kFly; ++u) {
      const uint32_t i = i0 + u * TH;
      if (i < B) cf.get(i, re[u], im[u], dr[u], di[u]);
    }
#pragma unroll
    for (int u = 0; u < kFly; ++u) {
      const uint32_t i = i0 + u * TH;
      if (i < B) f(i, re[u], im[u], dr[u], di[u]);
    }
  }
}

// Bucket b such that below(b) <= r < below(b) + hist[b]; every thread returns it.
template <int TH>
__device__ void find_bucket(SelectSharedT<TH>& sh, uint32_t r, uint32_t& bucket, uint32_t& below) {
  constexpr uint32_t per = kHistBins / TH;            // 4 (512 threads) or 8 (256)
  uint32_t local = 0;
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) local += sh.hist[threadIdx.x * per + q];
  uint32_t total;
  uint32_t before = block_exclusive_scan<TH>(local, sh.scan, total);
  if (r >= before && r < before + local) {
    uint32_t acc = before;
    for (uint32_t q = 0; q < per; ++q) {
      const uint32_t h = sh.hist[threadIdx.x * per + q];
      if (r < acc + h) {
        sh.found_bucket = threadIdx.x * per + q;
        sh.found_below = acc;
        break;
      }
      acc += h;
    }
  }
  __syncthreads();
  bucket = sh.found_bucket;
  below = sh.found_below;
  __syncthreads();
}

__device__ __forceinline__ bool key_less(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// Bitonic sort of the first M (power of two) entries by (key, idx) or by idx.
template <int TH>
__device__ void bitonic(SelectSharedT<TH>& sh, uint32_t M, bool by_index) {
  for (uint32_t k = 2; k <= M; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < M; t += blockDim.x) {
        const uint32_t u = t ^ j;
        if (u > t) {
          const bool asc = (t & k) == 0;
          bool greater;
          if (by_index) greater = (sh.idx[t] & 0x7FFFFFFFu) > (sh.idx[u] & 0x7FFFFFFFu);
          else greater = key_less(sh.key[u], sh.idx[u], sh.key[t], sh.idx[t]);
          if (greater == asc) {
            unsigned long long tk = sh.key[t]; sh.key[t] = sh.key[u]; sh.key[u] = tk;
            uint32_t ti = sh.idx[t]; sh.idx[t] = sh.idx[u]; sh.idx[u] = ti;
          }
        }
      }
      __syncthreads();
    }
  }
}

enum SelMode : int { kKeepAll = 0, kDropAll = 1, kList = 2, kExact = 3, kMask = 4 };


// Select + pack chunk `ci` whose coefficients start at cf.p.  Every thread of
// the CTA (TH threads) calls it; `sh` is the CTA's scratch.
template <typename CT, int TH = kSelThreads>
__device__ __noinline__ void select_pack_chunk(SelectSharedT<TH>& sh, const ChunkInfo ci, Coeffs<CT> cf, int exact_only,
                                               const QuantParams q, uint8_t* message, uint8_t* kept_mask,
                                               uint32_t* flags, const uint8_t* drop_mask) {
  const uint32_t B = ci.bins;
  const uint32_t kdrop = ci.drop;
  const uint32_t tid = threadIdx.x, lane = tid & 31;

  int mode = kList;
  if (drop_mask) mode = kMask;                  // energy mode: the drop set is given
  else if (kdrop == 0) mode = kKeepAll;
  else if (kdrop >= B) mode = kDropAll;

  float band_lo = 0.f, band_hi = INFINITY;   // proxy band of undecided bins
  bool all_band = false;
  uint32_t need = 0, m = 0;
  unsigned long long Te = 0;                  // exact mode threshold key
  uint32_t tie_cut = 0;

  if (mode == kList) {
    if (exact_only) {
      all_band = true;
    } else {
      const uint32_t r = kdrop - 1;             // rank of the largest dropped bin
      // pass 1: proxy bits [30:20]
      for (uint32_t b = tid; b < kHistBins; b += TH) sh.hist[b] = 0;
      __syncthreads();
      for_bins<TH>(cf, B, [&](uint32_t i, float re, float im, double dr, double di) {
        atomicAdd(&sh.hist[__float_as_uint(proxy_key(re, im)) >> 20], 1u);
      });
      __syncthreads();
      uint32_t b1, below1;
      find_bucket(sh, r, b1, below1);
      // pass 2: proxy bits [19:9] inside bucket b1
      for (uint32_t b = tid; b < kHistBins; b += TH) sh.hist[b] = 0;
      __syncthreads();
      for_bins<TH>(cf, B, [&](uint32_t i, float re, float im, double dr, double di) {
        const uint32_t pb = __float_as_uint(proxy_key(re, im));
        if ((pb >> 20) == b1) atomicAdd(&sh.hist[(pb >> 9) & 0x7FFu], 1u);
      });
      __syncthreads();
      uint32_t b2, below2;
      find_bucket(sh, r - below1, b2, below2);
      const uint32_t lo_pat = (b1 << 20) | (b2 << 9);
      const float lo_f = __uint_as_float(lo_pat);
      const float hi_f = __uint_as_float(lo_pat + 512u);
      if (lo_f < 0x1p-100f || hi_f > 0x1p100f) {
        all_band = true;                          // proxy unreliable: decide exactly
      } else {
        band_lo = lo_f * (1.0f - 0x1p-16f);
        band_hi = hi_f * (1.0f + 0x1p-16f);
      }
    }
    // collect the undecided band; count the certainly-dropped bins below it
    if (tid == 0) sh.cnt = 0;
    __syncthreads();
    uint32_t below_local = 0;
    for_bins<TH>(cf, B, [&](uint32_t i, float re, float im, double dr, double di) {
      const float p = proxy_key(re, im);
      if (!all_band && p < band_lo) {
        ++below_local;
      } else if (all_band || p < band_hi) {
        const uint32_t s = atomicAdd(&sh.cnt, 1u);
        if (s < kCandCap) sh.idx[s] = i;
      }
    });
    const uint32_t below = block_sum<TH>(below_local, sh.scan);
    m = sh.cnt;
    need = kdrop - below;
    if (m <= (uint32_t)kCandCap) {
      uint32_t M = 1;
      while (M < m) M <<= 1;
      for (uint32_t s = tid; s < M; s += TH) {
        if (s < m) {
          float re, im; double dr, di;
          cf.get(sh.idx[s], re, im, dr, di);
          sh.key[s] = (unsigned long long)__double_as_longlong(cabs_key(dr, di));
        } else {
          sh.key[s] = ~0ull;
          sh.idx[s] = 0x7FFFFFFFu;
        }
      }
      __syncthreads();
      bitonic(sh, M, false);
      for (uint32_t s = tid; s < m; s += TH)
        if (s < need) sh.idx[s] |= 0x80000000u;  // mark dropped
      __syncthreads();
      bitonic(sh, M, true);
    } else {
      mode = kExact;
      // radix select over the 63-bit exact key among band bins
      unsigned long long prefix = 0, pmask = 0;
      uint32_t rr = need ? need - 1 : 0, c_less = 0;
      const int shifts[6] = {52, 41, 30, 19, 8, 0};
      const int widths[6] = {11, 11, 11, 11, 11, 8};
      if (need > 0) {
        for (int pass = 0; pass < 6; ++pass) {
          for (uint32_t b = tid; b < kHistBins; b += TH) sh.hist[b] = 0;
          __syncthreads();
          const unsigned long long dm = (1ull << widths[pass]) - 1ull;
          for_bins<TH>(cf, B, [&](uint32_t i, float re, float im, double dr, double di) {
            const float p = proxy_key(re, im);
            if (!(all_band || (p >= band_lo && p < band_hi))) return;
            const unsigned long long key = (unsigned long long)__double_as_longlong(cabs_key(dr, di));
            if ((key & pmask) == prefix) atomicAdd(&sh.hist[(key >> shifts[pass]) & dm], 1u);
          });
          __syncthreads();
          uint32_t bk, bl;
          find_bucket(sh, rr, bk, bl);
          prefix |= (unsigned long long)bk << shifts[pass];
          pmask |= dm << shifts[pass];
          rr -= bl;
          c_less += bl;
        }
        Te = prefix;
        tie_cut = need - c_less;
      }
    }
  }

  // ---- final pass: decide, quantize, bitmap + code stream.  Tiles of
  //      kPer * TH bins, each thread kPer consecutive bins (so its
  //      codes are consecutive in the stream and a lane pair owns one bitmap
  //      word); one block scan per tile places every thread's codes.
  uint32_t* seg = reinterpret_cast<uint32_t*>(message + ci.seg_off);
  uint32_t* bitmap = seg + kSegHeader / 4;
  uint32_t* codes = reinterpret_cast<uint32_t*>(message + ci.seg_off + ci.code_off);
  const uint32_t bm_words = (ci.slots + 31) / 32;
  const int N = q.n_bits;
  uint32_t rank_base = 0;     // codes emitted so far
  uint32_t origin = 0;        // global code word index of stage[0]
  const bool direct = N == 8 || N == 16;         // whole-unit codes: no staging
  const uint32_t cap_units = ci.code_cap * (32u / (uint32_t)(N == 8 ? 8 : 16));
  uint32_t tie_seen = 0;
  bool overflow = false;
  for (uint32_t s = tid; s < SelectSharedT<TH>::kStageWords; s += TH) sh.stage[s] = 0;
  __syncthreads();

  for (uint32_t t0 = 0; t0 < B; t0 += SelectSharedT<TH>::kTile) {
    const uint32_t i0 = t0 + tid * kPer;
    float re[kPer], im[kPer];
    double dr[kPer], di[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      re[u] = im[u] = 0.f;
      dr[u] = di[u] = 0.0;
      if (i0 + u < B) cf.get(i0 + u, re[u], im[u], dr[u], di[u]);
    }
    bool dropped[kPer], is_tie[kPer];
    uint32_t ntie = 0;
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const uint32_t i = i0 + u;
      const bool valid = i < B;
      dropped[u] = false;
      is_tie[u] = false;
      if (mode == kDropAll) {
        dropped[u] = true;
      } else if (mode == kMask) {
        dropped[u] = valid && drop_mask[ci.bin_off + i];
      } else if (mode == kList || mode == kExact) {
        const float p = proxy_key(re[u], im[u]);
        const bool inband = all_band || (p >= band_lo && p < band_hi);
        if (!all_band && p < band_lo) dropped[u] = true;
        else if (inband && valid) {
          if (mode == kList) {
            uint32_t lo = 0, hi = m;                 // binary search by index
            while (lo < hi) {
              const uint32_t mid = (lo + hi) >> 1;
              if ((sh.idx[mid] & 0x7FFFFFFFu) < i) lo = mid + 1; else hi = mid;
            }
            dropped[u] = (lo < m) && ((sh.idx[lo] & 0x7FFFFFFFu) == i) && (sh.idx[lo] & 0x80000000u);
          } else if (need > 0) {
            const unsigned long long key = (unsigned long long)__double_as_longlong(cabs_key(dr[u], di[u]));
            dropped[u] = key < Te;
            is_tie[u] = key == Te;
            ntie += is_tie[u] ? 1u : 0u;
          }
        }
      }
      if (!valid) dropped[u] = true;
    }
    if (mode == kExact) {                        // ties dropped in bin order up to tie_cut
      uint32_t ties_total;
      uint32_t tr = tie_seen + block_exclusive_scan<TH>(ntie, sh.scan, ties_total);
#pragma unroll
      for (int u = 0; u < kPer; ++u)
        if (is_tie[u]) dropped[u] = tr++ < tie_cut;
      tie_seen += ties_total;
    }
    uint32_t cre[kPer], cim[kPer];
    uint32_t cnt = 0, nat = 0;                   // my codes; my 2*kPer slot bits in natural order
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      cre[u] = dropped[u] ? 0u : encode_code(q, re[u]);
      cim[u] = dropped[u] ? 0u : encode_code(q, im[u]);
      if (kept_mask && i0 + u < B) kept_mask[ci.bin_off + i0 + u] = dropped[u] ? 0 : 1;
      cnt += (cre[u] ? 1u : 0u) + (cim[u] ? 1u : 0u);
      nat |= ((cre[u] ? 1u : 0u) | (cim[u] ? 2u : 0u)) << (2 * u);
    }
    // bitmap: 32 slots per word = 32 / (2 kPer) threads per word
    {
      uint32_t w = nat;
#pragma unroll
      for (int o = 1; o < 16 / kPer; o <<= 1) w |= __shfl_down_sync(0xffffffffu, w, o) << (2 * kPer * o);
      if ((lane & (16 / kPer - 1)) == 0) {
        const uint32_t widx = i0 / 16;
        if (widx < bm_words) bitmap[widx] = ballot_to_wire(w);
      }
    }
    uint32_t ttot;
    const uint32_t r0 = rank_base + block_exclusive_scan<TH>(cnt, sh.scan, ttot);
    if (direct) {
      // byte / halfword codes: one writer per unit, straight into the message
      uint32_t rr = r0;
#pragma unroll
      for (int u = 0; u < 2 * kPer; ++u) {
        const uint32_t c = (u & 1) ? cim[u >> 1] : cre[u >> 1];
        if (c) {
          if (rr < cap_units) {
            if (N == 8) reinterpret_cast<uint8_t*>(codes)[rr] = (uint8_t)c;
            else reinterpret_cast<uint16_t*>(codes)[rr] = (uint16_t)c;
          } else {
            overflow = true;
          }
          ++rr;
        }
      }
      rank_base += ttot;
      continue;                                  // (the scan's closing barrier frees sh.scan)
    }
    // stage the codes (LSB-first N-bit fields, bit 0 of stage[0] = word `origin`)
    const uint64_t obit = (uint64_t)origin * 32u;
    FGC_CHECK((uint64_t)(r0 + cnt) * N - obit <= 32ull * SelectSharedT<TH>::kStageWords);
    uint64_t lb = (uint64_t)r0 * N - obit;
#pragma unroll
    for (int u = 0; u < 2 * kPer; ++u) {
      const uint32_t c = (u & 1) ? cim[u >> 1] : cre[u >> 1];
      if (c) {
        const uint32_t o = (uint32_t)(lb & 31u);
        atomicOr(&sh.stage[lb >> 5], c << o);
        if (o + N > 32u) atomicOr(&sh.stage[(lb >> 5) + 1], c >> (32u - o));
        lb += N;
      }
    }
    __syncthreads();
    const uint64_t end_bit = (uint64_t)(rank_base + ttot) * N;
    const uint32_t full_end = (uint32_t)(end_bit >> 5);      // words [origin, full_end) complete
    for (uint32_t w = origin + tid; w < full_end; w += TH) {
      if (w < ci.code_cap) codes[w] = sh.stage[w - origin];
      else overflow = true;
    }
    const uint32_t carry = (full_end >= origin) ? sh.stage[full_end - origin] : 0u;
    __syncthreads();
    for (uint32_t s = tid; s < SelectSharedT<TH>::kStageWords; s += TH) sh.stage[s] = (s == 0) ? carry : 0u;
    origin = full_end;
    rank_base += ttot;
    __syncthreads();
  }
  if (tid == 0) {
    if (direct) {                                // the units after the last code in its word
      const uint32_t per_word = 32u / (uint32_t)N;
      for (uint32_t u = rank_base; u % per_word != 0 && u < cap_units; ++u) {
        if (N == 8) reinterpret_cast<uint8_t*>(codes)[u] = 0;
        else reinterpret_cast<uint16_t*>(codes)[u] = 0;
      }
    } else if ((uint64_t)rank_base * N & 31u) {
      if (origin < ci.code_cap) codes[origin] = sh.stage[0];
      else overflow = true;
    }
    seg[0] = rank_base;
    seg[1] = 0; seg[2] = 0; seg[3] = 0;
  }
  // deterministic padding: bitmap pad words and the unused code capacity
  const uint32_t used = (uint32_t)(((uint64_t)rank_base * N + 31) / 32);
  for (uint32_t w = bm_words + tid; w < (ci.code_off - kSegHeader) / 4; w += TH) bitmap[w] = 0;
  const uint32_t cap_padded = (ci.code_cap + 3u) & ~3u;
  for (uint32_t w = used + tid; w < cap_padded; w += TH) codes[w] = 0;
  // zero the bitmap tail words beyond the last tile (none: tiles cover bins)
  if (overflow) atomicOr(flags, FGC_FLAG_CAPACITY);
}

}  // namespace
}  // namespace sel
}  // namespace fgc
