// Energy-mode drop sets (spectral.py:134-139, _drop_set with mode "energy"):
//
//   energies = bin_weights(L) * |X|**2          (spectral.py:150, Parseval weights)
//   order    = argsort(|X|, stable)
//   budget   = theta**2 * energies.sum()         (numpy pairwise summation)
//   k        = searchsorted(cumsum(energies[order]), budget, side="right")
//   dropped  = order[:k]
//
// Bit-exact with numpy given the same coefficients, one CTA per chunk, no
// library sort:
//   * keys are numpy's SIMD cabs (cabs_key), energies w * key * key in fp64;
//   * energies.sum() replays numpy's pairwise_sum tree exactly: thread 0
//     lays out the leaves (<= 128 values, splits rounded down to multiples of
//     8), the threads sum the leaves in parallel (8 strided accumulators, as
//     numpy's unrolled loop), thread 0 folds them in the tree's order;
//   * the cut is located by a radix select over the keys' high bits with
//     per-bucket fp64 energy sums (two passes of 2048 buckets), which leaves a
//     window of a few bins around the crossing; those are sorted exactly by
//     (key, bin) -- the stable argsort order -- and their prefix sums are
//     formed from an accurate sum of everything below the window;
//   * numpy's cumsum rounds every prefix sequentially; any accurate prefix is
//     within 2 B u S of it (u = 2^-53, S the prefix, B the bins; Higham's
//     bound for non-negative terms), so the cut is exact unless a prefix lies
//     within that distance of the budget -- then (about 1e-7 of chunks, and
//     whenever the window misses the crossing) the chunk is redone by the
//     exact fallback: an in-place bitonic sort of its (key, bin) pairs and the
//     sequential cumulative sum, exactly as numpy rounds it.
#include <cuda_runtime.h>
#include <math.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {
namespace {

constexpr int kET = 512;                       // threads per chunk CTA
constexpr uint32_t kEB = 2048;                 // radix buckets per pass
constexpr uint32_t kTreeDepth = 10;            // parallel pairwise tree depth (else thread 0 alone)
constexpr uint32_t kTreeNodes = (2u << kTreeDepth) - 1;   // heap of levels 0..kTreeDepth
constexpr uint32_t kWin = 1024;                // exact-sort window capacity

__device__ unsigned long long g_energy_fallbacks = 0;   // chunks sent to the exact fallback (diagnostics)

__device__ __forceinline__ double bin_weight(uint32_t b, uint32_t L, uint32_t B) {
  return (b == 0 || ((L % 2u) == 0u && b == B - 1)) ? 1.0 : 2.0;   // bin_weights (spectral.py:109-115)
}

template <class T2>
__device__ __forceinline__ double key_of(const T2* spec, uint64_t i) {
  const T2 x = spec[i];
  return cabs_key((double)x.x, (double)x.y);
}

// numpy's pairwise_sum leaf (loops_utils.h.src): n <= 128 values val(0..n-1)
// (a functor, inlined: the 8 loads of an unrolled step are independent)
template <class V>
__device__ __forceinline__ double leaf_sum(uint32_t n, V val) {
  if (n < 8) {
    double res = 0.0;
    for (uint32_t i = 0; i < n; ++i) res = __dadd_rn(res, val(i));
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = val(j);
  uint32_t i = 8;
  for (; i < n - (n % 8u); i += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = val(i + j);
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], v[j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, val(i));
  return res;
}

// energy of bin off + i from the stored keys (spectral.py:150)
__device__ __forceinline__ double leaf_energy_sum(const double* __restrict__ keys, uint32_t off, uint32_t n,
                                                  uint32_t L, uint32_t B) {
  return leaf_sum(n, [&](uint32_t i) {
    const double k = keys[off + i];
    return bin_weight(off + i, L, B) * __dmul_rn(k, k);
  });
}

// The pairwise tree as an explicit post-order walk by one thread (mode 2:
// sum everything here; used when the tree is deeper than the parallel heap).
__device__ double pairwise_walk(int mode, uint32_t n, uint32_t* loff, uint32_t* lsz, const double* lsum,
                                uint32_t* nleaves, const double* keys, uint32_t L, uint32_t B) {
  struct F { uint32_t off, n; int state; };
  F fs[48];
  double vals[48];
  int fp = 0, vp = 0;
  uint32_t leaf = 0;
  fs[fp++] = {0, n, 0};
  while (fp) {
    F& f = fs[fp - 1];
    if (f.n <= 128) {
      const double res = leaf_energy_sum(keys, f.off, f.n, L, B);
      ++leaf;
      vals[vp++] = res;
      --fp;
      continue;
    }
    uint32_t n2 = f.n / 2;
    n2 -= n2 % 8u;
    if (f.state == 0) {
      f.state = 1;
      fs[fp++] = {f.off, n2, 0};
    } else if (f.state == 1) {
      f.state = 2;
      fs[fp++] = {f.off + n2, f.n - n2, 0};
    } else {
      const double right = vals[--vp];
      const double left = vals[--vp];
      vals[vp++] = __dadd_rn(left, right);
      --fp;
    }
  }
  if (nleaves) *nleaves = leaf;
  return vals[0];
}

struct __align__(16) ESh {
  uint32_t cnt[kEB];
  uint32_t sum[kEB];                 // bucket energies in 2^-31 units of the chunk total (integer adds)
  uint32_t hoff[kTreeNodes];         // numpy's pairwise tree as a heap: node i -> children 2i+1, 2i+2
  uint32_t hn[kTreeNodes];           // node size (0: absent)
  double hval[kTreeNodes];           // node sums
  unsigned long long wkey[kWin];
  uint32_t widx[kWin];
  double scan_d[kET / 32 + 1];
  unsigned long long scan_u[kET / 32 + 1];
  uint32_t scan[40];
  uint32_t wcount, fbin, kcut, fallback, nleaf;
  double total, fbelow_e;
  unsigned long long fbelow_u;
};

// Bucket b whose cumulative energy (over buckets in key order, fixed point)
// first exceeds `budget`: below(b) <= budget < below(b) + sum[b] (the last
// bucket if none); `below` returns the energy before it.
__device__ void energy_bucket(ESh& sh, unsigned long long budget, uint32_t& bucket, unsigned long long& below) {
  constexpr uint32_t per = kEB / kET;          // 4
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  unsigned long long loc = 0;
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) loc += sh.sum[t * per + q];
  unsigned long long x = loc;                  // (u64: a bucket sum is < 2^31, their total < 2^32)
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
    if ((int)lane >= d) x += y;
  }
  if (lane == 31) sh.scan_u[warp] = x;
  if (t == 0) { sh.fbin = kEB - 1; sh.fbelow_u = 0; }
  __syncthreads();
  unsigned long long wb = 0;
  for (uint32_t w = 0; w < warp; ++w) wb += sh.scan_u[w];
  const unsigned long long before = wb + x - loc;
  unsigned long long acc = before;
  bool found = false;
#pragma unroll
  for (uint32_t q = 0; q < per; ++q) {
    const unsigned long long s = sh.sum[t * per + q];
    if (!found && acc + s > budget && sh.cnt[t * per + q]) {
      found = true;
      atomicMin(&sh.fbin, t * per + q);
    }
    acc += s;
  }
  __syncthreads();
  bucket = sh.fbin;
  if (t == bucket / per) {
    unsigned long long a = before;
    for (uint32_t q = 0; q < bucket % per; ++q) a += sh.sum[t * per + q];
    sh.fbelow_u = a;
  }
  __syncthreads();
  below = sh.fbelow_u;
  __syncthreads();
}

// One CTA per chunk: exact pairwise total, radix window, exact window sort,
// the cut, the drop mask.  fb[c] = 1 asks the exact fallback to redo chunk c.
template <class T2>
__global__ void __launch_bounds__(kET) k_energy_select(const ChunkInfo* chunks, uint32_t first, const T2* spectrum,
                                                        double theta, double* keys, uint8_t* drop, uint32_t* fb) {
  extern __shared__ __align__(16) unsigned char esm[];
  ESh& sh = *reinterpret_cast<ESh*>(esm);
  const uint32_t c = blockIdx.x;
  const ChunkInfo ci = chunks[first + c];
  const uint32_t B = ci.bins, L = ci.len, t = threadIdx.x;
  const T2* sp = spectrum + ci.bin_off;
  double* K = keys + ci.bin_off;
  uint8_t* D = drop + ci.bin_off;
  if (t == 0) { sh.wcount = 0; sh.fallback = 0; sh.nleaf = 0; }
  for (uint32_t b0 = t; b0 < B; b0 += 4 * kET) {      // the loads of 4 bins in flight together
    T2 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b0 + u * kET < B) x[u] = sp[b0 + u * kET];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (b0 + u * kET < B) K[b0 + u * kET] = cabs_key((double)x[u].x, (double)x[u].y);
  }
  for (uint32_t b = t; b < kEB; b += kET) { sh.cnt[b] = 0; sh.sum[b] = 0; }
  __syncthreads();
  if (theta == 0.0) {                            // spectral.py:135-136: nothing dropped
    for (uint32_t b = t; b < B; b += kET) D[b] = 0;
    if (t == 0) fb[c] = 0;
    return;
  }
  // ---- exact pairwise total: numpy's tree (split n > 128 at n/2 rounded
  //      down to a multiple of 8) built level by level as a heap, the leaves
  //      summed in parallel, the inner nodes folded bottom-up (left + right)
  if (t == 0) { sh.hoff[0] = 0; sh.hn[0] = B; }
  __syncthreads();
  uint32_t depth = 0;
  bool deeper = B > 128;
  while (deeper && depth < kTreeDepth) {
    const uint32_t l0 = (1u << depth) - 1, cnt = 1u << depth;
    bool split = false;
    for (uint32_t i = t; i < cnt; i += kET) {
      const uint32_t nd = l0 + i, n = sh.hn[nd];
      uint32_t n2 = n / 2;
      n2 -= n2 % 8u;
      const bool inner = n > 128;
      sh.hoff[2 * nd + 1] = sh.hoff[nd];
      sh.hn[2 * nd + 1] = inner ? n2 : 0u;
      sh.hoff[2 * nd + 2] = sh.hoff[nd] + n2;
      sh.hn[2 * nd + 2] = inner ? n - n2 : 0u;
      split |= inner && (n2 > 128 || n - n2 > 128);
    }
    ++depth;
    deeper = __syncthreads_or(split);
  }
  if (!deeper) {
    // The leaves (0 < n <= 128; at most 2^kTreeDepth = kWin of them) are
    // listed in the window index array (free until the window pass), then
    // summed by 8 lanes each: lane j runs numpy's accumulator r[j] over
    // elements j, j+8, ... (its loads issued together), the unrolled loop's
    // final ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) is a 3-step xor shuffle
    // (commutative adds: the same bits), and lane 0 adds the n % 8 tail.
    const uint32_t nodes = (2u << depth) - 1;
    for (uint32_t nd = t; nd < nodes; nd += kET) {
      const uint32_t n = sh.hn[nd];
      if (n && n <= 128) sh.widx[atomicAdd(&sh.nleaf, 1u)] = nd;
    }
    __syncthreads();
    const uint32_t nl = sh.nleaf;
    for (uint32_t base = 0; base < 8u * nl; base += kET) {      // uniform trip count: whole-warp shuffles
      const uint32_t task = base + t, j = t & 7u;
      const bool act = task < 8u * nl;
      const uint32_t nd = act ? sh.widx[task >> 3] : 0u;
      const uint32_t n = act ? sh.hn[nd] : 0u, off = act ? sh.hoff[nd] : 0u;
      const uint32_t m8 = n >= 8u ? n - (n % 8u) : 0u;
      auto val = [&](uint32_t i) {
        const double k = K[off + i];
        return bin_weight(off + i, L, B) * __dmul_rn(k, k);
      };
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = (8u * q + j < m8) ? val(8u * q + j) : 0.0;
      double r = v[0];
#pragma unroll
      for (int q = 1; q < 16; ++q)
        if (8u * q < m8) r = __dadd_rn(r, v[q]);
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
      r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
      if (act && j == 0) {
        double res = m8 ? r : 0.0;
        for (uint32_t i = m8; i < n; ++i) res = __dadd_rn(res, val(i));
        sh.hval[nd] = res;
      }
    }
    __syncthreads();
    for (int l = (int)depth - 1; l >= 0; --l) {
      const uint32_t l0 = (1u << l) - 1, cnt = 1u << l;
      for (uint32_t i = t; i < cnt; i += kET) {
        const uint32_t nd = l0 + i;
        if (sh.hn[nd] > 128) sh.hval[nd] = __dadd_rn(sh.hval[2 * nd + 1], sh.hval[2 * nd + 2]);
      }
      __syncthreads();
    }
    if (t == 0) sh.total = sh.hval[0];
  } else if (t == 0) {
    sh.total = pairwise_walk(2, B, nullptr, nullptr, nullptr, nullptr, K, L, B);
  }
  __syncthreads();
  const double budget = __dmul_rn(__dmul_rn(theta, theta), sh.total);
  // ---- radix window over the keys' high 32 bits: [31:20] exponent+, then
  //      [19:9]; bucket energies in fixed point (units of 2^-31 of the total:
  //      native 32-bit shared-memory atomics, order-free; truncation costs at
  //      most B 2^-31 of the total, below one sub-bucket's energy, and the
  //      window keeps two sub-buckets of margin each side)
  const uint32_t* Kh = reinterpret_cast<const uint32_t*>(K) + 1;   // high word of key b at Kh[2b]
  auto hi32 = [&](uint32_t b) { return Kh[2 * b]; };
  // f(b, hi32(b)) over the chunk's bins, 4 high-word loads in flight per thread
  auto for_hi = [&](auto f) {
    for (uint32_t b0 = t; b0 < B; b0 += 4 * kET) {
      uint32_t h[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) h[u] = (b0 + u * kET < B) ? hi32(b0 + u * kET) : 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (b0 + u * kET < B) f(b0 + u * kET, h[u]);
    }
  };
  const double fscale = sh.total > 0.0 ? 0x1p31 / sh.total : 0.0;
  auto approx_e = [&](uint32_t h, uint32_t b) -> uint32_t {
    const double k = __hiloint2double((int)h, 0);
    return (uint32_t)fmin(bin_weight(b, L, B) * k * k * fscale, 0x1p31);
  };
  const unsigned long long ubudget = (unsigned long long)fmin(budget * fscale, 0x1p62);
  for_hi([&](uint32_t b, uint32_t h) {
    atomicAdd(&sh.cnt[h >> 20], 1u);
    atomicAdd(&sh.sum[h >> 20], approx_e(h, b));
  });
  __syncthreads();
  uint32_t b1;
  unsigned long long e1;
  energy_bucket(sh, ubudget, b1, e1);
  for (uint32_t b = t; b < kEB; b += kET) { sh.cnt[b] = 0; sh.sum[b] = 0; }
  __syncthreads();
  for_hi([&](uint32_t b, uint32_t h) {
    if ((h >> 20) == b1) {
      atomicAdd(&sh.cnt[(h >> 9) & 2047u], 1u);
      atomicAdd(&sh.sum[(h >> 9) & 2047u], approx_e(h, b));
    }
  });
  __syncthreads();
  uint32_t b2;
  unsigned long long e2;
  energy_bucket(sh, ubudget > e1 ? ubudget - e1 : 0ull, b2, e2);
  (void)e2;
  // window: two sub-buckets each side of b2 (the fixed-point sums may put the
  // crossing a bucket off); everything below it is certainly dropped
  const uint32_t base = (b1 << 20) | (b2 << 9);
  const uint32_t wlo = base >= 1024u ? base - 1024u : 0u;
  const uint32_t whi = base + 1536u;
  // Everything below the window is dropped: its mask is written here, and
  // its energy is taken as the total minus the energies at or above the
  // window (a few percent of the bins, the only full keys loaded).  That
  // prefix is as accurate as a direct sum to within the rounding tolerance
  // the cut applies (below), which covers B u S.
  double below = 0.0;                            // (holds the energy at or above the window until reduced)
  uint32_t nbelow = 0;
  for_hi([&](uint32_t b, uint32_t h) {
    D[b] = h < wlo ? 1u : 0u;
    if (h < wlo) {
      ++nbelow;
    } else {
      const double k = K[b];
      below += bin_weight(b, L, B) * __dmul_rn(k, k);
      if (h < whi) {
        const uint32_t s = atomicAdd(&sh.wcount, 1u);
        if (s < kWin) {
          sh.wkey[s] = (unsigned long long)__double_as_longlong(k);
          sh.widx[s] = b;
        }
      }
    }
  });
  // block sums of `below` (fp64) and `nbelow`
  {
    const uint32_t lane = t & 31, warp = t >> 5;
    for (int d = 16; d > 0; d >>= 1) {
      below += __shfl_down_sync(0xffffffffu, below, d);
      nbelow += __shfl_down_sync(0xffffffffu, nbelow, d);
    }
    if (lane == 0) { sh.scan_d[warp] = below; sh.scan[warp] = nbelow; }
    __syncthreads();
    if (t == 0) {
      double s = 0.0;
      uint32_t n = 0;
      for (int w = 0; w < kET / 32; ++w) { s += sh.scan_d[w]; n += sh.scan[w]; }
      sh.fbelow_e = fmax(sh.total - s, 0.0);
      sh.kcut = n;
    }
    __syncthreads();
  }
  const double S0 = sh.fbelow_e;
  const uint32_t n0 = sh.kcut;
  const uint32_t m = sh.wcount;
  if (m > kWin) {
    if (t == 0) sh.fallback = 1;
  } else {
    // exact (key, bin) order of the window: rank by counting (m is small)
    __syncthreads();
    for (uint32_t i = t; i < m; i += kET) {
      const unsigned long long k = sh.wkey[i];
      const uint32_t bi = sh.widx[i];
      uint32_t rank = 0;
      for (uint32_t j = 0; j < m; ++j) {
        const unsigned long long kj = sh.wkey[j];
        rank += (kj < k || (kj == k && sh.widx[j] < bi)) ? 1u : 0u;
      }
      sh.hoff[rank] = bi;                         // window bins in sorted order (the tree heap is free)
    }
    __syncthreads();
    if (t == 0) {
      // prefix sums over the window; tolerance covers numpy's sequential rounding
      const double u = 0x1p-53;
      const double tol = 2.0 * (double)(B + 8) * u * fmax(budget, S0) * 2.0;
      bool ok = S0 <= budget - tol;               // everything below the window is in
      double S = S0;
      uint32_t k = n0;
      bool crossed = false;
      for (uint32_t i = 0; i < m && ok; ++i) {
        const uint32_t bi = sh.hoff[i];
        const double kk = K[bi];
        S += bin_weight(bi, L, B) * __dmul_rn(kk, kk);
        const double tl = 2.0 * (double)(B + 8) * u * fmax(S, budget) * 2.0;
        if (fabs(S - budget) <= tl) ok = false;   // too close to call: the exact fallback decides
        else if (S <= budget) ++k;
        else { crossed = true; break; }
      }
      if (!crossed) ok = false;                   // the window did not reach the budget
      (void)tol;
      sh.fallback = ok ? 0u : 1u;
      sh.kcut = k - n0;                           // dropped window entries
    }
  }
  __syncthreads();
  if (sh.fallback) {
    if (t == 0) {
      fb[c] = 1;
      atomicAdd(&g_energy_fallbacks, 1ull);
    }
    return;
  }
  // ---- the drop mask (below the window: written above): the first kcut
  //      window entries
  const uint32_t kw = sh.kcut;
  for (uint32_t i = t; i < m; i += kET) D[sh.hoff[i]] = i < kw ? 1u : 0u;
  if (t == 0) fb[c] = 0;
}

// Exact fallback for the flagged chunks: in-place bitonic sort of (key, bin)
// over the chunk's bins (virtual +inf entries above B never move down: every
// comparison puts the minimum at the lower index), then numpy's sequential
// cumulative sum in sorted order.
__global__ void __launch_bounds__(1024) k_energy_exact(const ChunkInfo* chunks, uint32_t first, double theta,
                                                        double* keys, uint32_t* idx, uint8_t* drop,
                                                        const uint32_t* fb) {
  const uint32_t c = blockIdx.x;
  if (!fb[c]) return;
  const ChunkInfo ci = chunks[first + c];
  const uint32_t B = ci.bins, L = ci.len, t = threadIdx.x;
  double* K = keys + ci.bin_off;                  // sorted in place (keys are recomputed per call)
  uint32_t* I = idx + ci.bin_off;
  uint8_t* D = drop + ci.bin_off;
  __shared__ double total_s;
  __shared__ uint32_t kcut_s;
  // the total, before the keys are permuted (thread 0, the tree walk)
  if (t == 0) total_s = pairwise_walk(2, B, nullptr, nullptr, nullptr, nullptr, K, L, B);
  for (uint32_t b = t; b < B; b += blockDim.x) I[b] = b;
  __syncthreads();
  uint32_t N2 = 1;
  while (N2 < B) N2 <<= 1;
  auto less = [&](uint32_t a, uint32_t b) {
    const double ka = K[a], kb = K[b];
    return ka < kb || (ka == kb && I[a] < I[b]);
  };
  for (uint32_t k = 2; k <= N2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = t; i < N2; i += blockDim.x) {
        const uint32_t p = (j == (k >> 1)) ? (i ^ (k - 1)) : (i ^ j);   // mirrored first step, then halvers
        if (p > i && p < B && i < B && less(p, i)) {
          const double tk = K[i]; K[i] = K[p]; K[p] = tk;
          const uint32_t ti = I[i]; I[i] = I[p]; I[p] = ti;
        }
      }
      __syncthreads();
    }
  }
  if (t == 0) {
    const double budget = __dmul_rn(__dmul_rn(theta, theta), total_s);
    double run = 0.0;
    uint32_t k = 0;
    for (uint32_t i = 0; i < B && theta != 0.0; ++i) {      // theta == 0 drops nothing (spectral.py:135-136)
      const double kk = K[i];
      run = __dadd_rn(run, bin_weight(I[i], L, B) * __dmul_rn(kk, kk));
      k += run <= budget ? 1u : 0u;
    }
    kcut_s = k;
  }
  __syncthreads();
  for (uint32_t i = t; i < B; i += blockDim.x) D[I[i]] = i < kcut_s ? 1u : 0u;
}

}  // namespace

fgc_status EnergyScratch::ensure(uint64_t bins, uint32_t chunks) {
  if (bins <= cap_bins && chunks <= cap_chunks) return FGC_OK;
  free_all();
  FGC_CUDA(cudaMalloc(&keys, sizeof(double) * bins));
  FGC_CUDA(cudaMalloc(&idx, sizeof(uint32_t) * bins));
  FGC_CUDA(cudaMalloc(&drop, bins));
  FGC_CUDA(cudaMalloc(&kcut, sizeof(uint32_t) * chunks));
  cap_bins = bins;
  cap_chunks = chunks;
  static bool attr = false;
  if (!attr) {
    FGC_CUDA(cudaFuncSetAttribute(k_energy_select<float2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(ESh)));
    FGC_CUDA(cudaFuncSetAttribute(k_energy_select<double2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)sizeof(ESh)));
    attr = true;
  }
  return FGC_OK;
}

void EnergyScratch::free_all() {
  cudaFree(keys); cudaFree(idx); cudaFree(drop); cudaFree(kcut);
  keys = nullptr;
  idx = kcut = nullptr;
  drop = nullptr;
  cap_bins = 0;
  cap_chunks = 0;
}

// Debug knob: force every chunk through the exact fallback (tests).
static bool g_energy_force_exact = false;

// Drop mask (1 = dropped) for chunks [first, first + count) of a chunk-major
// spectrum (float2, or double2 when f64) whose bins start at bin_off(first) = bin0.
fgc_status energy_drop_mask(EnergyScratch& e, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                            uint64_t bin0, uint64_t nbins, uint32_t max_bins, const void* spectrum, int f64,
                            double theta, cudaStream_t s, const uint8_t** drop_out) {
  if (!count) return FGC_OK;
  (void)max_bins;
  FGC_TRY(e.ensure(bin0 + nbins, count));
  if (f64)
    k_energy_select<double2><<<count, kET, sizeof(ESh), s>>>(d_chunks, first, static_cast<const double2*>(spectrum),
                                                             theta, e.keys, e.drop, e.kcut);
  else
    k_energy_select<float2><<<count, kET, sizeof(ESh), s>>>(d_chunks, first, static_cast<const float2*>(spectrum),
                                                            theta, e.keys, e.drop, e.kcut);
  FGC_LAUNCHED(1);
  if (g_energy_force_exact) FGC_CUDA(cudaMemsetAsync(e.kcut, 0x01, sizeof(uint32_t) * count, s));
  k_energy_exact<<<count, 1024, 0, s>>>(d_chunks, first, theta, e.keys, e.idx, e.drop, e.kcut);
  FGC_LAUNCHED(1);
  *drop_out = e.drop;
  return FGC_OK;
}

}  // namespace fgc

extern "C" unsigned long long fgc_debug_energy_fallbacks(void) {
  unsigned long long v = 0;
  cudaMemcpyFromSymbol(&v, fgc::g_energy_fallbacks, sizeof(v));
  return v;
}

extern "C" int fgc_debug_energy_force_exact(int on) {
  fgc::g_energy_force_exact = on != 0;
  return 0;
}
