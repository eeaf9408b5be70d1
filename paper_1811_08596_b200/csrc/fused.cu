// Fused sm_100a kernels for 65536-sample chunks (the codec's default and the
// benchmark's chunk size, codec.py:73).  One chunk per thread-block cluster
// of two CTAs; everything between the HBM read of the gradient and the HBM
// write of the message happens on chip.
//
// compress (k_fused_compress, cluster 2x1x1, 512 threads per CTA)
//   z[n] = x[2n] + i x[2n+1], N = 32768 complex points.  A decimation-in-
//   frequency split gives each CTA an independent 16384-point FFT:
//     CTA 0: a[n] = z[n] + z[n+M]             -> Z[2m]   = FFT_M(a)[m]
//     CTA 1: b[n] = (z[n] - z[n+M]) W_N^n     -> Z[2m+1] = FFT_M(b)[m]
//   (each CTA reads the whole chunk; the second read hits L2).  The real-FFT
//   post-processing pairs Z[k] with Z[N-k]; both stay inside one CTA and, by
//   choosing pass-3 columns (k, 1024-k) / (k, 1023-k), inside one thread.
//   So the 32769 bins X[k] end up in registers: even bins in CTA 0, odd bins
//   in CTA 1.  Count-mode selection (spectral.py:124-156) is a cluster-wide
//   radix select on a float32 proxy of |X|^2 (histograms merged through
//   DSMEM), with numpy's exact float64 cabs key and the stable index
//   tie-break applied to the few bins whose proxy is too close to call.
//   Codes (quantizer.py:217-236) are gathered bin-ordered into two halves,
//   one per CTA (each CTA stores the other's non-zero pairs remotely), and
//   each CTA emits its half of the MSB-first bitmap and of the LSB-first
//   packed code stream (packer.py, quantizer.pack_codes) straight into the
//   device message segment.  Degenerate chunks (all proxies tiny, or > kCand
//   undecided bins) are selected in place by CTA 0 with the generic
//   single-CTA code (select_pack.cuh) from the spectrum written to scratch.
//
// decode (k_fused_decode, 2 CTAs per chunk, 512 threads)
//   Bins are owned in groups {k, M-k, M+k, N-k}; each thread accumulates the
//   weighted non-zero slots of its 32-bin block from the W messages in
//   worker order (single writer per entry: deterministic, identical on every
//   rank).  Each CTA turns its groups into both CTAs' Y values, keeps its own
//   and stores the peer's through DSMEM; one inverse 16384-point FFT per CTA
//   then yields the even (r=0) or odd (r=1) complex samples of the chunk:
//   x[4p+2r], x[4p+2r+1].  In the averaging step the decode is launched as
//   the compress grid's programmatic dependent and waits per chunk for the
//   segment's done tag (and, under the peer exchange, the peers' flags).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdlib.h>

#include <type_traits>

#include "fgc_device.cuh"
#include "fgc_internal.h"
#include "fused_fft.cuh"
#include "select_pack.cuh"

namespace cg = cooperative_groups;

namespace fgc {

struct FusedTables {
  float2* thi = nullptr;     // W_65536^(256 h), h < 256
  float2* tlo = nullptr;     // W_65536^l, l < 256
  float2* t1024 = nullptr;   // W_1024^m, m < 1024
  uint32_t wave = 74;        // clusters resident at once (SMs / 2): the L2 prefetch distance
};

__device__ uint32_t g_fused_dbg = 0;                  // instrumentation knobs (0 in production)
__device__ unsigned long long g_fused_ts[2048 * 16];   // per-CTA phase timestamps (knob 128)

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FGC_TS(k)                                                                        \
  do {                                                                                   \
    if ((dbg & 128u) && threadIdx.x == 0 && blockIdx.x < 2048)                           \
      g_fused_ts[blockIdx.x * 16 + (k)] = globaltimer();                                  \
  } while (0)

namespace {

using namespace ff;

constexpr int kCand = 512;
constexpr uint32_t kBins = kN + 1;                     // 32769
constexpr uint32_t kBmWords = (2 * kBins + 31) / 32;  // 2049
constexpr uint32_t kHalfBins = kN / 2;                 // 16384: pack split point
constexpr uint32_t kStageOff = 16900;                  // u32 offset of the code-stream staging in buf
// emit-phase compaction strips (per warp: 256 bins + 256 float2) above the code half
constexpr uint32_t kEmitStageOff = 16904;
constexpr uint32_t kEmitStageWords = 768;
static_assert(kStageOff > (kHalfBins + kHalfBins / 32) &&
              kStageOff + (32 + (kHalfBins + 1) * 32 + 31) / 32 <= 2 * (kPadded + 64), "staging fits in buf");
static_assert(kEmitStageOff % 2 == 0 && kEmitStageOff >= kHalfBins + kHalfBins / 32 &&
              kEmitStageOff + 16 * kEmitStageWords <= 2 * (kPadded + 64), "emit strips fit in buf");

template <int B, int E, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (B < E) {
    f(std::integral_constant<int, B>{});
    static_for<B + 1, E>(f);
  }
}

__global__ void k_init_tables(float2* thi, float2* tlo, float2* t1024) {
  const int i = threadIdx.x;
  double s, c;
  if (i < 256) {
    sincospi(-2.0 * (double)(256 * i) / 65536.0, &s, &c);
    thi[i] = make_float2((float)c, (float)s);
    sincospi(-2.0 * (double)i / 65536.0, &s, &c);
    tlo[i] = make_float2((float)c, (float)s);
  }
  sincospi(-2.0 * (double)i / 1024.0, &s, &c);
  t1024[i] = make_float2((float)c, (float)s);
}

// ------------------------------------------------------------------ loads

template <class T> struct In;
template <> struct In<float> {
  template <bool HALF>
  __device__ static float2 get(const float* g, uint64_t e, uint32_t& bad) {
    float2 v = __ldg(reinterpret_cast<const float2*>(g + e));
    bad |= (isfinite(v.x) && isfinite(v.y)) ? 0u : FGC_FLAG_NONFINITE;
    if (HALF) {
      v.x = __half2float(__float2half_rn(v.x));
      v.y = __half2float(__float2half_rn(v.y));
      bad |= (isinf(v.x) || isinf(v.y)) ? FGC_FLAG_HALF_OVERFLOW : 0u;
    }
    return v;
  }
};
template <> struct In<double> {
  template <bool HALF>
  __device__ static float2 get(const double* g, uint64_t e, uint32_t& bad) {
    const double2 d = __ldg(reinterpret_cast<const double2*>(g + e));
    if (!isfinite(d.x) || !isfinite(d.y)) { bad |= FGC_FLAG_NONFINITE; return make_float2(0.f, 0.f); }
    float2 v;
    if (HALF) {
      v = make_float2(__half2float(__double2half(d.x)), __half2float(__double2half(d.y)));
      if (isinf(v.x) || isinf(v.y)) bad |= FGC_FLAG_HALF_OVERFLOW;
    } else {
      v = make_float2((float)d.x, (float)d.y);
      if (isinf(v.x) || isinf(v.y)) bad |= FGC_FLAG_F32_RANGE;
    }
    return v;
  }
};

// encode_code specialised for N <= 16 (no passthrough branch)
__device__ __forceinline__ uint32_t enc16(const QuantParams& q, float x) {
  const float a = fabsf(x);
  const bool pos = x > 0.0f;
  const uint32_t off = (__float_as_uint(fminf(a, pos ? q.pos_cap : q.neg_cap)) >> q.shift) - q.pbase + 1u;
  const uint32_t c = pos ? min(off, q.npos) : q.npos + min(off, q.nneg);
  return (a < q.eps) ? 0u : c;
}

// ------------------------------------------------------------------ compress

struct CompressArgs {
  const ChunkInfo* chunks;
  uint32_t first;
  const void* grad;
  QuantParams q;
  uint8_t* message;
  uint32_t* flags;
  const float2* thi;
  const float2* tlo;
  const float2* t1024;
  float2* fb_spec;       // chunk-major spectrum scratch for degenerate (fallback) chunks
  float2* dbg_spec;      // debug hook: write the spectrum and stop
  uint32_t count;        // chunks in this launch
  uint32_t ahead;        // L2 prefetch distance in chunks (one wave)
  PieceCounter pc;       // exchange: per-piece completed-segment counters (optional)
};

struct __align__(16) CompressShared {
  float2 buf[kPadded + 64];          // FFT transposes / 4 sub-histograms / bin-ordered code half + staging
  float2 thi[256], tlo[kTloPadded];   // tlo and t1024 in tpad layout
  float2 t1024[kT1024Padded];
  uint32_t hbm[2048 + 4];            // bitmap words of the whole chunk, this CTA's (parity) bins only, set during
                                     // emit with local atomics; the pack ORs in the peer's words

  uint32_t hist[2048];               // pass-1 histogram of this CTA (read by the peer)
  uint32_t hist2[2048];              // pass-2 histogram of this CTA (read by the peer)
  uint32_t scan[40];
  unsigned long long ckey[kCand];    // CTA 0: undecided bins (exact key, bin), pushed by both CTAs
  uint32_t cidx[kCand];
  unsigned long long lkey[kCand];    // each CTA's own copy of CTA 0's list, sorted locally
  uint32_t lidx[kCand];
  uint32_t ccount;                   // CTA 0: number of undecided bins
  uint32_t below;                    // per CTA: bins certainly dropped
  uint32_t anynz;                    // per CTA: any non-zero coefficient
  uint32_t rcount[2];                // per CTA: its non-zero codes landing in half 0 / half 1
  uint32_t fbin, fbelow;             // merged_bucket result
};

enum : int { kModeKeepAll = 0, kModeDropAll = 1, kModeList = 2, kModeFallback = 3 };

// Bucket holding rank r in the cluster-merged histogram (own + peer).
__device__ void merged_bucket(CompressShared& sh, const uint32_t* own, const uint32_t* peer, uint32_t r,
                              uint32_t& bucket, uint32_t& below) {
  const uint32_t t = threadIdx.x;
  const uint4 a = reinterpret_cast<const uint4*>(own)[t];
  const uint4 b = reinterpret_cast<const uint4*>(peer)[t];
  const uint32_t h[4] = {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w};
  const uint32_t local = h[0] + h[1] + h[2] + h[3];
  uint32_t total;
  const uint32_t before = block_exclusive_scan<kThreads>(local, sh.scan, total);
  if (r >= before && r < before + local) {
    uint32_t acc = before;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (r >= acc && r < acc + h[q]) {
        sh.fbin = 4 * t + q;
        sh.fbelow = acc;
      }
      acc += h[q];
    }
  }
  __syncthreads();
  bucket = sh.fbin;
  below = sh.fbelow;
}

// Rare paths kept out of line so the 32-way unrolled per-bin loops stay small
// (instruction-cache pressure is the fused kernel's first-order stall).
__device__ __noinline__ bool inband_dropped(const CompressShared* sh, uint32_t mcount, uint32_t bin) {
  uint32_t lo = 0, hi = mcount;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if ((sh->lidx[mid] & 0x7FFFFFFFu) < bin) lo = mid + 1; else hi = mid;
  }
  return lo < mcount && (sh->lidx[lo] & 0x7FFFFFFFu) == bin && (sh->lidx[lo] & 0x80000000u);
}

__device__ __noinline__ void push_candidate(CompressShared* sh0, uint32_t bin, float re, float im) {
  const uint32_t s = atomicAdd(&sh0->ccount, 1u);
  FGC_CHECK(bin <= kN);
  if (s < (uint32_t)kCand) {
    sh0->cidx[s] = bin;
    sh0->ckey[s] = (unsigned long long)__double_as_longlong(cabs_key((double)re, (double)im));
  }
}

// CTA 0: sort the undecided bins by (exact key, bin), mark the `need`
// smallest dropped, re-sort by bin for the lookups.
__device__ __noinline__ void resolve_candidates(CompressShared& sh, uint32_t m, uint32_t need) {
  const uint32_t tid = threadIdx.x;
  uint32_t M2 = 1;
  while (M2 < m) M2 <<= 1;
  for (uint32_t s = m + tid; s < M2; s += kThreads) {
    sh.lkey[s] = ~0ull;
    sh.lidx[s] = 0x7FFFFFFFu;
  }
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t k = 2; k <= M2; k <<= 1) {
      for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
        for (uint32_t t = tid; t < M2; t += kThreads) {
          const uint32_t u = t ^ jj;
          if (u > t) {
            const bool asc = (t & k) == 0;
            bool gt;
            if (pass == 0) {
              gt = sh.lkey[t] > sh.lkey[u] ||
                   (sh.lkey[t] == sh.lkey[u] && (sh.lidx[t] & 0x7FFFFFFFu) > (sh.lidx[u] & 0x7FFFFFFFu));
            } else {
              gt = (sh.lidx[t] & 0x7FFFFFFFu) > (sh.lidx[u] & 0x7FFFFFFFu);
            }
            if (gt == asc) {
              const unsigned long long tk = sh.lkey[t]; sh.lkey[t] = sh.lkey[u]; sh.lkey[u] = tk;
              const uint32_t ti = sh.lidx[t]; sh.lidx[t] = sh.lidx[u]; sh.lidx[u] = ti;
            }
          }
        }
        __syncthreads();
      }
    }
    if (pass == 0) {
      for (uint32_t s = tid; s < need && s < m; s += kThreads) sh.lidx[s] |= 0x80000000u;
      __syncthreads();
    }
  }
}

// Kernel pushes (exchange transport 2): store part `part` of `nparts` of
// chunk c's finished segment -- header, bitmap and the codes its nnz says it
// holds, rounded to 16 bytes (what the decode reads) -- into every peer's
// gather buffer, then release the part's tag(s) there at system scope.
__device__ __noinline__ void push_parts(PieceCounter pc, const ChunkInfo ci, const uint8_t* message, uint32_t chunk,
                                        uint32_t N, uint32_t part, uint32_t nparts) {
  const uint8_t* seg = message + ci.seg_off;
  const uint32_t nnz = __ldcg(reinterpret_cast<const uint32_t*>(seg));
  const uint64_t code_bytes = 16ull * (((uint64_t)nnz * N + 127u) / 128u);
  const uint64_t cap = ci.code_off + 4ull * ((ci.code_cap + 3u) & ~3u);
  const uint32_t n4 = (uint32_t)(min((uint64_t)ci.code_off + code_bytes, cap) / 16u);
  const uint32_t lo = part * n4 / nparts, hi = (part + 1) * n4 / nparts;
  const uint4* s4 = reinterpret_cast<const uint4*>(seg);
  for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    const uint4 v = __ldcg(s4 + e);
    for (uint32_t p = 0; p < pc.npeers; ++p) reinterpret_cast<uint4*>(pc.pdst[p] + ci.seg_off)[e] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t p = 0; p < pc.npeers; ++p)
      for (uint32_t j = part; j < part + (nparts == 1 ? 2u : 1u); ++j)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pc.ptag[p] + 2ull * chunk + j), "r"(pc.pval)
                     : "memory");
  }
}

__device__ __forceinline__ void zero_buf(CompressShared& sh, uint32_t words4) {
  uint4* z = reinterpret_cast<uint4*>(sh.buf);
  for (uint32_t e = threadIdx.x; e < words4; e += kThreads) z[e] = make_uint4(0, 0, 0, 0);
}

// PUSH: the kernel-push exchange transport (a separate instantiation, so the
// default kernel carries none of its code: measured 1.5% of compress time)
template <class T, bool DEBUG, bool HALF, bool PUSH = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) k_fused_compress(CompressArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  CompressShared& sh = *reinterpret_cast<CompressShared*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t r = cluster.block_rank();
  const uint32_t tid = threadIdx.x;
  const uint32_t chunk = a.first + blockIdx.x / 2;
  const ChunkInfo ci = a.chunks[chunk];
  CompressShared& sh0 = *cluster.map_shared_rank(&sh, 0);
  CompressShared& shp = *cluster.map_shared_rank(&sh, r ^ 1);
  const QuantParams q = a.q;
  const uint32_t dbg = g_fused_dbg;
  // every CTA of the grid is resident or done from here on: the dependent
  // decode grid may start filling SMs as they free up (it waits per chunk)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const T* g = static_cast<const T*>(a.grad) + ci.in_off;

  if (tid == 0) {
    // stream this CTA's half of the chunk into L2 while the tables load
    const uint32_t half_bytes = (uint32_t)(kL / 2 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(g) + (uint64_t)r * half_bytes;
    for (uint32_t off = 0; off < half_bytes; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }
  if (tid < 256) {
    sh.thi[tid] = a.thi[tid];
    sh.tlo[tpad(tid)] = a.tlo[tid];
  }
  sh.t1024[tpad(tid)] = a.t1024[tid];
  sh.t1024[tpad(tid + 512)] = a.t1024[tid + 512];
  reinterpret_cast<uint4*>(sh.hist2)[tid] = make_uint4(0, 0, 0, 0);
  sh.hbm[tid] = 0u;
  sh.hbm[tid + 512] = 0u;
  sh.hbm[tid + 1024] = 0u;
  sh.hbm[tid + 1536] = 0u;
  if (tid < 4) sh.hbm[2048 + tid] = 0u;
  if (tid == 0) { sh.ccount = 0; sh.below = 0; sh.anynz = 0; sh.rcount[0] = 0; sh.rcount[1] = 0; }
  uint32_t* codes_g = DEBUG ? nullptr : reinterpret_cast<uint32_t*>(a.message + ci.seg_off + ci.code_off);
  __syncthreads();

  FGC_TS(0);
  // ---- 1. load + decimation-in-frequency split (pass-1 input layout)
  float2 v[32];
  {
    uint32_t bad = 0;
    const float2 wi = tw(sh.thi, sh.tlo, 2u * tid);          // W_N^tid
    static_for<0, 32>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const uint32_t n = tid + 512u * j;
      const float2 z0 = In<T>::template get<HALF>(g, 2ull * n, bad);
      const float2 z1 = In<T>::template get<HALF>(g, 2ull * (n + kM), bad);
      if (r == 0) {
        v[j] = make_float2(z0.x + z1.x, z0.y + z1.y);
      } else {                                              // (z0 - z1) W_N^(tid + 512 j)
        v[j] = w64mul<j>(cmul(make_float2(z0.x - z1.x, z0.y - z1.y), wi));
      }
    });
    if (bad && r == 0) atomicOr(a.flags, bad);
  }

  FGC_TS(1);
  if (tid == 0 && blockIdx.x / 2 + a.ahead < a.count) {
    // the chunk the next wave runs here: its HBM read overlaps this wave's compute
    const ChunkInfo cn = a.chunks[chunk + a.ahead];
    const uint32_t half_bytes = (uint32_t)(kL / 2 * sizeof(T));
    const char* base = reinterpret_cast<const char*>(static_cast<const T*>(a.grad) + cn.in_off) + (uint64_t)r * half_bytes;
    for (uint32_t off = 0; off < half_bytes; off += 32768u)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + off), "r"(32768u) : "memory");
  }
  // ---- 2. 16384-point FFT: passes 1, 2 (transposes in smem), pass 3 on two columns
  fft_pass12<false>(v, sh.buf, sh.t1024);
  FGC_TS(2);
  __syncthreads();
  const bool special = (r == 0 && tid == 0);
  const uint32_t ka = tid;
  const uint32_t kb = (r == 0) ? (tid == 0 ? 512u : 1024u - tid) : 1023u - tid;
  float2 va[16], vb[16];
  fft_pass3<false>(ka, sh.buf, va, sh.thi, sh.tlo);
  fft_pass3<false>(kb, sh.buf, vb, sh.thi, sh.tlo);

  // ---- 3. real-FFT post-processing in registers: X[k] = (P + conj Q)/2 - i W_L^k (P - conj Q)/2
  auto r2c = [](float2 P, float2 Q, float2 w) -> float2 {
    const float2 A = make_float2(P.x + Q.x, P.y - Q.y);
    const float2 B = make_float2(P.x - Q.x, P.y + Q.y);
    const float2 t = cmul(w, make_float2(B.y, -B.x));
    return make_float2(0.5f * (A.x + t.x), 0.5f * (A.y + t.y));
  };
  float2 xn = make_float2(0.f, 0.f);      // X[N] (CTA 0, thread 0 only)
  if (!special) {
    // bins: va[j] -> (2ka + r) + 2048 j, vb[j] -> (2kb + r) + 2048 j ; W_L^(2048 j) = W_32^j
    const float2 wA = tw(sh.thi, sh.tlo, 2u * ka + r);
    const float2 wB = tw(sh.thi, sh.tlo, 2u * kb + r);
    static_for<0, 16>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = va[j], Q = vb[15 - j];
      va[j] = r2c(P, Q, w32mul<j>(wA));
      vb[15 - j] = r2c(Q, P, w32mul<15 - j>(wB));
    });
  } else {
    // column 0: pairs j <-> 16-j; self pairs j = 0 (X[0], X[N]) and j = 8 (X[M])
    const float2 a0 = va[0];
    static_for<1, 8>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = va[j], Q = va[16 - j];
      va[j] = r2c(P, Q, w32mul<j>(make_float2(1.f, 0.f)));
      va[16 - j] = r2c(Q, P, w32mul<16 - j>(make_float2(1.f, 0.f)));
    });
    va[8] = r2c(va[8], va[8], w32mul<8>(make_float2(1.f, 0.f)));
    va[0] = make_float2(a0.x + a0.y, 0.f);
    xn = make_float2(a0.x - a0.y, 0.f);
    // column 512: bins 1024 + 2048 j, pairs j <-> 15-j ; W_L^1024 = W_64^1
    const float2 w1 = w64mul<1>(make_float2(1.f, 0.f));
    static_for<0, 8>([&](auto J) {
      constexpr int j = decltype(J)::value;
      const float2 P = vb[j], Q = vb[15 - j];
      vb[j] = r2c(P, Q, w32mul<j>(w1));
      vb[15 - j] = r2c(Q, P, w32mul<15 - j>(w1));
    });
  }
#define BIN_A(j) (2u * (ka + 1024u * (j)) + r)
#define BIN_B(j) (2u * (kb + 1024u * (j)) + r)

  if (DEBUG) {
    float2* out = a.dbg_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      out[BIN_A(j)] = va[j];
      out[BIN_B(j)] = vb[j];
    }
    if (special) out[kN] = xn;
    return;
  }

  FGC_TS(3);
  // ---- 4. count-mode selection, cluster-wide (cluster barriers A-C)
  const uint32_t kdrop = ci.drop;
  int mode = kModeList;
  if (kdrop == 0) mode = kModeKeepAll;
  else if (kdrop >= kBins) mode = kModeDropAll;
  float band_lo = 0.f, band_hi = INFINITY;
  uint32_t mcount = 0;
  __syncthreads();                                // pass-3 reads of buf are done
  if (mode == kModeList) {
    // pass 1: proxy bits [30:20] into four sub-histograms (in buf)
    uint32_t* sub = reinterpret_cast<uint32_t*>(sh.buf) + 2048u * ((tid >> 5) & 3u);
    zero_buf(sh, 2048);
    __syncthreads();
    uint32_t nz = 0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const uint32_t pa = __float_as_uint(proxy_key(va[j].x, va[j].y));
      const uint32_t pb = __float_as_uint(proxy_key(vb[j].x, vb[j].y));
      nz |= __float_as_uint(va[j].x) | __float_as_uint(va[j].y) | __float_as_uint(vb[j].x) |
            __float_as_uint(vb[j].y);
      atomicAdd(&sub[pa >> 20], 1u);
      atomicAdd(&sub[pb >> 20], 1u);
    }
    if (special) {
      nz |= __float_as_uint(xn.x) | __float_as_uint(xn.y);
      atomicAdd(&sub[__float_as_uint(proxy_key(xn.x, xn.y)) >> 20], 1u);
    }
    nz &= 0x7FFFFFFFu;                            // -0.0 is zero
    if (__any_sync(0xffffffffu, nz != 0) && (tid & 31) == 0) atomicOr(&sh.anynz, 1u);
    __syncthreads();
    {
      const uint4* s4 = reinterpret_cast<const uint4*>(sh.buf);
      const uint4 x0 = s4[tid], x1 = s4[512 + tid], x2 = s4[1024 + tid], x3 = s4[1536 + tid];
      reinterpret_cast<uint4*>(sh.hist)[tid] =
          make_uint4(x0.x + x1.x + x2.x + x3.x, x0.y + x1.y + x2.y + x3.y, x0.z + x1.z + x2.z + x3.z,
                     x0.w + x1.w + x2.w + x3.w);
    }
    FGC_TS(7);
    cluster.sync();                               // A: pass-1 histograms visible
    const bool anynz = (sh.anynz | shp.anynz) != 0;
    uint32_t b1, below1;
    merged_bucket(sh, sh.hist, shp.hist, kdrop - 1, b1, below1);
    if (!anynz) {
      mode = kModeDropAll;                        // every coefficient is exactly zero: all codes 0
    } else {
      // pass 2: proxy bits [19:9] of the bins inside bucket b1 (few: direct atomics)
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint32_t pa = __float_as_uint(proxy_key(va[j].x, va[j].y));
        const uint32_t pb = __float_as_uint(proxy_key(vb[j].x, vb[j].y));
        if ((pa >> 20) == b1) atomicAdd(&sh.hist2[(pa >> 9) & 0x7FFu], 1u);
        if ((pb >> 20) == b1) atomicAdd(&sh.hist2[(pb >> 9) & 0x7FFu], 1u);
      }
      if (special) {
        const uint32_t pn = __float_as_uint(proxy_key(xn.x, xn.y));
        if ((pn >> 20) == b1) atomicAdd(&sh.hist2[(pn >> 9) & 0x7FFu], 1u);
      }
      __syncthreads();
    }
    FGC_TS(8);
    cluster.sync();                               // B: pass-2 histograms visible, buf zeroed
    if (mode == kModeList) {
      uint32_t b2, below2;
      merged_bucket(sh, sh.hist2, shp.hist2, kdrop - 1 - below1, b2, below2);
      const uint32_t lo_pat = (b1 << 20) | (b2 << 9);
      const float lo_f = __uint_as_float(lo_pat);
      const float hi_f = __uint_as_float(lo_pat + 512u);
      if (lo_f < 0x1p-100f || hi_f > 0x1p100f) {
        mode = kModeFallback;
      } else {
        band_lo = lo_f * (1.0f - 0x1p-16f);
        band_hi = hi_f * (1.0f + 0x1p-16f);
        // collect undecided bins into CTA 0's list; count the certainly dropped
        uint32_t below_l = 0;
        auto collect = [&](float2 x, uint32_t bin) {
          const float p = proxy_key(x.x, x.y);
          below_l += (p < band_lo) ? 1u : 0u;
          if (p >= band_lo && p < band_hi) push_candidate(&sh0, bin, x.x, x.y);
        };
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          collect(va[j], BIN_A(j));
          collect(vb[j], BIN_B(j));
        }
        if (special) collect(xn, kN);
        const uint32_t bl = block_sum<kThreads>(below_l, sh.scan);
        if (tid == 0) sh.below = bl;
      }
    }
    FGC_TS(9);
    cluster.sync();                               // C: candidates and counts visible
    // Both CTAs copy CTA 0's candidate list and resolve it themselves: the
    // same data and order give the same decision, and no barrier waits for a
    // single resolving CTA.
    {
      const uint32_t m = sh0.ccount;
      const uint32_t below = sh.below + shp.below;
      if (mode == kModeList && (m > (uint32_t)kCand || below > kdrop || below + m < kdrop)) mode = kModeFallback;
      if (mode == kModeList) {
        for (uint32_t s = tid; s < m; s += kThreads) {
          sh.lkey[s] = sh0.ckey[s];
          sh.lidx[s] = sh0.cidx[s];
        }
        __syncthreads();
        resolve_candidates(sh, m, kdrop - below);
        mcount = m;
      }
    }
    FGC_TS(10);
  } else {
    cluster.sync();                               // D': both bitmaps zeroed (peer atomics follow)
  }

  FGC_TS(4);
  if (mode == kModeFallback) {
    float2* out = a.fb_spec + ci.bin_off;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      out[BIN_A(j)] = va[j];
      out[BIN_B(j)] = vb[j];
    }
    if (special) out[kN] = xn;
    __threadfence();
    cluster.sync();          // both halves written; both CTAs finished reading CTA 0's list
    if (r == 1) return;
    // CTA 0 selects and packs the chunk with the generic single-CTA code,
    // its scratch in the (now free) transpose buffer
    static_assert(sizeof(sel::SelectShared) <= sizeof(sh.buf), "select scratch fits in buf");
    sel::select_pack_chunk<float2>(*reinterpret_cast<sel::SelectShared*>(sh.buf), ci,
                                   sel::Coeffs<float2>{a.fb_spec + ci.bin_off}, 0, q, a.message, nullptr, a.flags,
                                   nullptr);
    if (a.pc.cnt || a.pc.done) {
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        if (a.pc.cnt) atomicAdd(&a.pc.cnt[(chunk - a.pc.first) / a.pc.per], 1u);
        if (a.pc.done) release_tag(a.pc.done + chunk, a.pc.tag, a.pc.sys);
      }
      if constexpr (PUSH) push_parts(a.pc, ci, a.message, chunk, (uint32_t)q.n_bits, 0, 1);
    }
    return;
  }

  // ---- 5. codes -> two bin-ordered halves: CTA 0 holds bins [0, 16384),
  //         CTA 1 holds [16384, 32768]; non-zero pairs only (arrays are zeroed).
  float lo_b = band_lo, hi_b = band_hi;           // KeepAll / DropAll as degenerate bands
  if (mode == kModeKeepAll) { lo_b = -1.0f; hi_b = -1.0f; }
  if (mode == kModeDropAll) { lo_b = INFINITY; hi_b = INFINITY; }
  uint32_t* arr_own = reinterpret_cast<uint32_t*>(sh.buf);
  uint32_t* arr_peer = reinterpret_cast<uint32_t*>(shp.buf);
  uint32_t rc0 = 0, rc1 = 0;                      // my non-zero codes per half
  // half d of bin (2k + r) + 2048 j is j >= 8 for both columns (and 1 for bin N):
  // a compile-time choice, so own-half stores stay STS and the peer's go to DSMEM
  auto emit_pair = [&](float2 x, uint32_t bin, auto D) {
    constexpr uint32_t d = decltype(D)::value;
    const float p = proxy_key(x.x, x.y);
    bool keep = p >= lo_b;
    if (keep && p < hi_b) keep = !inband_dropped(&sh, mcount, bin);
    if (keep) {
      const uint32_t cre = enc16(q, x.x), cim = enc16(q, x.y);
      const uint32_t pc = cre | (cim << 16);
      if (pc) {
        const uint32_t c = (cre ? 1u : 0u) + (cim ? 1u : 0u);
        if (d) rc1 += c; else rc0 += c;
        const uint32_t lb = bin - d * kHalfBins;
        FGC_CHECK(lb <= kHalfBins && pad(lb) < kStageOff);
        const uint32_t bits = ((cre ? 1u : 0u) | (cim ? 2u : 0u)) << (2u * (lb & 15u));
        atomicOr(&sh.hbm[(lb >> 4) + d * 1024u], bits);
        if (d == r) arr_own[pad(lb)] = pc;
        else arr_peer[pad(lb)] = pc;
      }
    }
  };
  // keep bits first, branch-free across all 32 values (bit 2j: va[j], 2j+1: vb[j])
  uint32_t keep = 0, band = 0;
  static_for<0, 16>([&](auto J) {
    constexpr int j = decltype(J)::value;
    const float pa = proxy_key(va[j].x, va[j].y), pb = proxy_key(vb[j].x, vb[j].y);
    keep |= ((pa >= hi_b ? 1u : 0u) << (2 * j)) | ((pb >= hi_b ? 1u : 0u) << (2 * j + 1));
    band |= ((pa >= lo_b && pa < hi_b ? 1u : 0u) << (2 * j)) | ((pb >= lo_b && pb < hi_b ? 1u : 0u) << (2 * j + 1));
  });
  while (band) {                                  // undecided bins: the resolved list decides
    const uint32_t b = __ffs(band) - 1u;
    band &= band - 1u;
    const uint32_t bin = 2u * (((b & 1u) ? kb : ka) + 1024u * (b >> 1)) + r;
    if (!inband_dropped(&sh, mcount, bin)) keep |= 1u << b;
  }
  // Only ~1 value in 10 is kept, so encoding every value in every lane would
  // spend most of the phase on dropped bins.  Per round of 4 j (8 values per
  // lane) the warp compacts its kept (bin, value) pairs into a staging strip
  // of the free upper part of buf, then every lane encodes and stores
  // consecutive entries.  Rounds 0-1 land in half 0, rounds 2-3 in half 1.
  {
    const uint32_t lane = tid & 31u;
    uint32_t* wmeta = arr_own + kEmitStageOff + (tid >> 5) * kEmitStageWords;
    float2* wval = reinterpret_cast<float2*>(wmeta + 256);
    static_for<0, 4>([&](auto R) {
      constexpr int j0 = 4 * decltype(R)::value;
      constexpr uint32_t d = j0 >= 8 ? 1u : 0u;
      const uint32_t m8 = (keep >> (2 * j0)) & 0xFFu;
      const uint32_t cnt = __popc(m8);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += t;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      uint32_t pos = incl - cnt;
      static_for<0, 8>([&](auto K) {
        constexpr int k = decltype(K)::value;
        constexpr int j = j0 + k / 2;
        if ((m8 >> k) & 1u) {
          FGC_CHECK(pos < 256u);
          wmeta[pos] = (k & 1) ? BIN_B(j) : BIN_A(j);
          wval[pos] = (k & 1) ? vb[j] : va[j];
          ++pos;
        }
      });
      __syncwarp();
      for (uint32_t e = lane; e < total; e += 32) {
        const uint32_t bin = wmeta[e];
        const float2 x = wval[e];
        const uint32_t cre = enc16(q, x.x), cim = enc16(q, x.y);
        const uint32_t pc = cre | (cim << 16);
        if (pc) {
          const uint32_t c = (cre ? 1u : 0u) + (cim ? 1u : 0u);
          if (d) rc1 += c; else rc0 += c;
          const uint32_t lb = bin - d * kHalfBins;
          FGC_CHECK(lb <= kHalfBins && pad(lb) < kStageOff);
          const uint32_t bits = ((cre ? 1u : 0u) | (cim ? 2u : 0u)) << (2u * (lb & 15u));
          atomicOr(&sh.hbm[(lb >> 4) + d * 1024u], bits);      // local: the pack merges both CTAs' words
          if (d == r) arr_own[pad(lb)] = pc;
          else arr_peer[pad(lb)] = pc;
        }
      }
      __syncwarp();                               // strip reused by the next round
    });
  }
  if (special) emit_pair(xn, kN, std::integral_constant<uint32_t, 1u>{});
#undef BIN_A
#undef BIN_B
  {
    const uint32_t s0 = __reduce_add_sync(0xffffffffu, rc0), s1 = __reduce_add_sync(0xffffffffu, rc1);
    if ((tid & 31) == 0) {
      if (s0) atomicAdd(&sh.rcount[0], s0);
      if (s1) atomicAdd(&sh.rcount[1], s1);
    }
  }
  FGC_TS(11);
  cluster.sync();                                 // E: both halves complete, per-half counts visible
  FGC_TS(5);
  const uint32_t t0 = sh.rcount[0] + shp.rcount[0];            // codes in half 0
  const uint32_t all = t0 + sh.rcount[1] + shp.rcount[1];       // codes in the chunk
  const int N = q.n_bits;
  // byte-aligned half boundary (N = 8, 16, or t0*N % 8 == 0): no cross-CTA fold needed
  const uint64_t s1bits = (uint64_t)t0 * N;
  const bool fold = (s1bits & 7u) != 0;
  // ---- 6. pack: thread t of CTA d owns bins d*16384 + [32t, 32t+32) (+ bin N)
  const uint32_t nb = (r == 1 && tid == kThreads - 1) ? 33u : 32u;
  // the bitmap words of my bins: both CTAs' (disjoint, parity-interleaved)
  // bits; only the set slots of the code arrays are valid
  const uint32_t gw = r * 1024u + 2u * tid;
  const uint32_t w0 = sh.hbm[gw] | shp.hbm[gw], w1 = sh.hbm[gw + 1] | shp.hbm[gw + 1];
  const uint32_t w2 = (nb == 33) ? (sh.hbm[2048] | shp.hbm[2048]) : 0u;
  // Without a fold these were the last remote accesses: arrive now, wait
  // before exiting (a CTA's shared memory must outlive its peer's accesses).
  if (!fold) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  const uint32_t cnt = __popc(w0) + __popc(w1) + __popc(w2);
  uint32_t* seg = reinterpret_cast<uint32_t*>(a.message + ci.seg_off);
  uint32_t* bm = seg + kSegHeader / 4;
  {
    const uint32_t wb = r * (kHalfBins / 16) + 2u * tid;
    bm[wb] = ballot_to_wire(w0);
    bm[wb + 1] = ballot_to_wire(w1);
    if (nb == 33) {
      bm[wb + 2] = ballot_to_wire(w2);
      const uint32_t pad_words = (ci.code_off - kSegHeader) / 4;
      for (uint32_t w = kBmWords; w < pad_words; ++w) bm[w] = 0u;
    }
  }
  uint32_t total;
  const uint32_t base = block_exclusive_scan<kThreads>(cnt, sh.scan, total);
  // This CTA's half of the stream starts at global bit S = (r ? t0 : 0) * N;
  // staged in shared memory: local word k <-> global word (S >> 5) + k.
  const uint64_t S = r ? s1bits : 0ull;
  if ((N == 8 || N == 16) && !(dbg & 32u)) {
    // byte / halfword codes: every code unit has one writer, so the codes go
    // straight to the message (no staging, no zero fill, no copy-out); the
    // half boundary is a unit boundary, and the units after the last code in
    // its word are zeroed explicitly
    const uint32_t* row = arr_own + pad(32u * tid);
    if (N == 8) {
      uint8_t* cg = reinterpret_cast<uint8_t*>(codes_g);
      const uint32_t cap_units = 4u * ci.code_cap;
      uint32_t u = (uint32_t)(S >> 3) + base;
      auto emit = [&](uint64_t m64, const uint32_t* src) {
        while (m64) {
          const uint32_t pos = __ffsll((long long)m64) - 1;
          m64 &= m64 - 1;
          const uint32_t pc = src[pos >> 1];
          if (u < cap_units) cg[u] = (uint8_t)((pos & 1) ? (pc >> 16) : pc);
          ++u;
        }
      };
      emit(((uint64_t)w1 << 32) | w0, row);
      if (w2) emit(w2, arr_own + pad(32u * tid + 32u));
      if (r == 1 && tid == 0)
        for (uint32_t b = all; b < 4u * ((all + 3u) / 4u) && b < cap_units; ++b) cg[b] = 0;
    } else {
      uint16_t* cg = reinterpret_cast<uint16_t*>(codes_g);
      const uint32_t cap_units = 2u * ci.code_cap;
      uint32_t u = (uint32_t)(S >> 4) + base;
      auto emit = [&](uint64_t m64, const uint32_t* src) {
        while (m64) {
          const uint32_t pos = __ffsll((long long)m64) - 1;
          m64 &= m64 - 1;
          const uint32_t pc = src[pos >> 1];
          if (u < cap_units) cg[u] = (uint16_t)((pos & 1) ? (pc >> 16) : pc);
          ++u;
        }
      };
      emit(((uint64_t)w1 << 32) | w0, row);
      if (w2) emit(w2, arr_own + pad(32u * tid + 32u));
      if (r == 1 && tid == 0 && (all & 1u) && all < cap_units) cg[all] = 0;
    }
  } else {
  const uint32_t wstart = (uint32_t)(S >> 5), o = (uint32_t)(S & 31u);
  const uint32_t nwords = (uint32_t)((o + (uint64_t)total * N + 31) / 32);
  uint32_t* stg = arr_own + kStageOff;
  FGC_CHECK(kStageOff + nwords + 1 <= 2 * (kPadded + 64));
  for (uint32_t k = tid; k < nwords; k += kThreads) stg[k] = 0u;
  __syncthreads();
  {
    uint32_t lbit = o + base * (uint32_t)N;               // local bit of my first code
    const uint32_t* row = arr_own + pad(32u * tid);       // my 32 bins (pad(32t + j) = pad(32t) + j)
    uint8_t* stg8 = reinterpret_cast<uint8_t*>(stg);
    // slot s of my bins: bin s / 2, re (s even) / im (s odd); one loop over all 64 slots
    auto emit_slots = [&](uint64_t m64, const uint32_t* src) {
      while (m64) {
        const uint32_t pos = __ffsll((long long)m64) - 1;
        m64 &= m64 - 1;
        const uint32_t pc = src[pos >> 1];
        const uint32_t code = (pos & 1) ? (pc >> 16) : (pc & 0xFFFFu);
        FGC_CHECK((lbit >> 5) < nwords);
        if (N == 8) {
          stg8[lbit >> 3] = (uint8_t)code;                // byte-aligned codes: plain stores
        } else {
          const uint32_t wi = lbit >> 5, sb = lbit & 31u;
          atomicOr(&stg[wi], code << sb);
          if (sb + N > 32u) atomicOr(&stg[wi + 1], code >> (32u - sb));
        }
        lbit += N;
      }
    };
    emit_slots(((uint64_t)w1 << 32) | w0, row);
    if (w2) emit_slots(w2, arr_own + pad(32u * tid + 32u));
  }
  __syncthreads();
  if (fold) {
    // the half boundary splits a byte: CTA 0 folds CTA 1's first word and owns it
    cluster.sync();                               // F: CTA 1's staging complete
    if (r == 0 && tid == 0) stg[s1bits >> 5] |= (reinterpret_cast<const uint32_t*>(shp.buf) + kStageOff)[0];
    __syncthreads();
  }
  // write-out; the word shared by the two halves is written bytewise by each owner
  const uint32_t shared_w = (uint32_t)(s1bits >> 5);
  const bool split = (s1bits & 31u) != 0 && !fold;
  for (uint32_t k = tid; k < nwords; k += kThreads) {
    const uint32_t w = wstart + k;
    if (w >= ci.code_cap) continue;
    if (r == 1 && fold && k == 0) continue;       // folded into CTA 0's copy
    if (split && w == shared_w) {
      uint8_t* p = reinterpret_cast<uint8_t*>(codes_g + w);
      const uint32_t bb = (uint32_t)(s1bits & 31u) >> 3;       // bytes [0, bb) belong to half 0
      const uint32_t val = stg[k];
      for (uint32_t b = (r ? bb : 0u); b < (r ? 4u : bb); ++b) p[b] = (uint8_t)(val >> (8 * b));
      continue;
    }
    codes_g[w] = stg[k];
  }
  }
  const uint32_t used = (uint32_t)(((uint64_t)all * N + 31) / 32);
  const uint32_t cap_padded = (ci.code_cap + 3u) & ~3u;
  if (r == 1)
    for (uint32_t w = used + tid; w < cap_padded; w += kThreads) codes_g[w] = 0u;
  if (r == 0 && tid == 0) {
    seg[0] = all;
    seg[1] = 0; seg[2] = 0; seg[3] = 0;
    if (used > ci.code_cap) atomicOr(a.flags, FGC_FLAG_CAPACITY);
  }
  if (a.pc.cnt || a.pc.done) {
    // the segment is complete once both CTAs' writes are visible device-wide
    __threadfence();
    if (!fold) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // the early arrive's phase
    cluster.sync();                               // (G) every thread of both CTAs has fenced
    if (r == 0 && tid == 0) {
      if (a.pc.cnt) atomicAdd(&a.pc.cnt[(chunk - a.pc.first) / a.pc.per], 1u);
      if (a.pc.done) release_tag(a.pc.done + chunk, a.pc.tag, a.pc.sys);
    }
    if constexpr (PUSH) push_parts(a.pc, ci, a.message, chunk, (uint32_t)N, r, 2);
  } else if (fold) {
    cluster.sync();                               // G: CTA 0 finished reading CTA 1's staging
  } else {
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  FGC_TS(6);
}

// ------------------------------------------------------------------ decode

struct DecodeArgs {
  const ChunkInfo* chunks;
  uint32_t first;
  const uint8_t* messages;
  int W;
  uint64_t stride;
  Weights wts;
  QuantParams q;
  float* out;
  const float2* thi;
  const float2* tlo;
  const float2* t1024;
  const float2* spectrum;     // dense-spectrum mode (debug hook), else null
  uint32_t count;             // chunks in this launch
  uint32_t ahead;             // L2 prefetch distance in chunks (one wave)
  PieceWait pw;               // exchange: wait for the peers' pieces (optional)
};

constexpr int kDecBatch = 4;                           // messages per block scan in the decode
constexpr uint32_t kDecStageWords = 8192;              // code words of a message batch staged in smem

struct __align__(16) DecodeShared {
  float2 x[kPadded + 64];            // this CTA's bins of the weighted spectrum sum, then Y_r / FFT scratch
  float2 thi[256], tlo[kTloPadded];   // tlo and t1024 in tpad layout
  float2 t1024[kT1024Padded];
  uint32_t bm[kDecBatch][2 * kThreads * 2];   // natural-order bitmap words 0..2047 of a message batch
  uint32_t pref[kDecBatch][2 * kThreads];     // codes before each 32-bin block
  uint32_t bmN[kDecBatch];                    // word 2048 (bin N)
  uint32_t soff[kDecBatch];                   // staging offset (words) of each message, ~0u: not staged
  uint32_t scan[4 * (kThreads / 32 + 1)];     // block_exclusive_scan4 scratch
  // packed code streams of the batch's messages (whole chunk segments, each
  // 16-byte aligned), copied once with coalesced loads so the per-lane bit
  // walk refills its window from shared memory instead of L2
  uint4 stage[kDecStageWords / 4 + 2];
};

// decode, one cluster of 2 CTAs per chunk.
//
// The inverse real FFT of X[0..N] (N = 32768, M = N/2) runs as two 16384-
// point FFTs, CTA r transforming Y_r (z[2n + r] = IFFT_M(Y_r)[n]):
//   Y_r[m] = cA(m) X[m] + cA(m+M) X[m+M] + cB(N-m) conj X[N-m] + cB(M-m) conj X[M-m]
//   cA(b) = (1 + i W_L^-b) / 2,  cB(b) = (1 + i W_L^b) / 2, times W_N^-b / W_N^b for r = 1
// (the real-IFFT pre-processing Z[k] = E + i W_L^-k O folded by the DIT
// split).  The four bins {k, M-k, M+k, N-k} feed exactly Y_0 and Y_1 at m = k
// and m = M-k, so chunk bins are owned by groups: CTA 0 owns the groups
// k in [0, 4096) -- 32-bin blocks [0, 4096), [12288, 20480), [28672, 32768] --
// and CTA 1 the groups k in [4096, 8192] -- blocks [4096, 12288), [20480, 28672)
// (group 4096's bins 12288 and 28672 sit in CTA 0 and are read over DSMEM).
//
// Phase 1: thread t owns one 32-bin block; for every message, in worker
// order, it adds weight_w * value of each non-zero slot of its block into its
// own shared-memory entries: single writer, deterministic on every rank.
// Phase 2: each CTA turns its groups into Y_0 and Y_1 values and stores the
// peer's half over DSMEM (64 KB each way), then runs its inverse FFT.
__device__ __forceinline__ uint32_t dec_block(uint32_t r, uint32_t t) {
  if (r == 0) return t < 128 ? t : (t < 384 ? t + 256 : t + 512);
  return t < 256 ? t + 128 : t + 384;
}

// Z[k] = ((X[k] + conj X[N-k]) + i t (X[k] - conj X[N-k])) / 2 with t = W_L^-k:
// the real-IFFT pre-processing (z[n] = x[2n] + i x[2n+1] = IFFT_N(Z)[n]).
__device__ __forceinline__ float2 zval(float2 a, float2 b, float2 t) {
  const float2 s = make_float2(a.x + b.x, a.y - b.y);      // a + conj b
  const float2 d = make_float2(a.x - b.x, a.y + b.y);      // a - conj b
  const float2 u = cmul(t, d);
  return make_float2(0.5f * (s.x - u.y), 0.5f * (s.y + u.x));
}

// Group k -> {Y0[k], Y1[k], Y0[M-k], Y1[M-k]} with Y_r[m] = W_N^-(r m) (Z[m] + (-1)^r Z[m+M]).
// w = W_L^k; W_L^-(k+M) = i conj w, W_L^-(N-k) = -w, W_L^-(M-k) = i w, W_N^-(M-k) = -w^2.
__device__ __forceinline__ void y_group(float2 xk, float2 xMk, float2 xkM, float2 xNk, float2 w, float2 (&y)[4]) {
  const float2 v = conjf2(w);                               // W_L^-k
  const float2 zk = zval(xk, xNk, v);
  const float2 zkM = zval(xkM, xMk, make_float2(-v.y, v.x));
  const float2 zMk = zval(xMk, xkM, make_float2(-w.y, w.x));
  const float2 zNk = zval(xNk, xk, make_float2(-w.x, -w.y));
  const float2 w2 = cmul(w, w);                             // W_N^k
  y[0] = cadd(zk, zkM);
  y[1] = cmul(conjf2(w2), csub(zk, zkM));
  y[2] = cadd(zMk, zNk);
  y[3] = cmul(make_float2(-w2.x, -w2.y), csub(zMk, zNk));
}

// TAGS: the in-kernel exchange transports (per-chunk tag waits, and direct
// reads of the peers' buffers when pw.mtab is set); the default
// instantiation carries none of that code (measured 1.5 us of decode time)
template <bool TAGS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1) k_fused_decode(DecodeArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DecodeShared& sh = *reinterpret_cast<DecodeShared*>(smem_raw);
  cg::cluster_group cluster = cg::this_cluster();
  const uint32_t r = cluster.block_rank();
  const uint32_t chunk = a.first + blockIdx.x / 2;
  const ChunkInfo ci = a.chunks[chunk];
  const uint32_t tid = threadIdx.x;
  if (tid < 256) {
    sh.thi[tid] = a.thi[tid];
    sh.tlo[tpad(tid)] = a.tlo[tid];
  }
  sh.t1024[tpad(tid)] = a.t1024[tid];
  sh.t1024[tpad(tid + 512)] = a.t1024[tid + 512];
  float2* acc = sh.x;
  const uint32_t dbg = g_fused_dbg;
  const uint32_t blk = dec_block(r, tid);                  // my 32-bin block
  const bool binN = (r == 0 && tid == kThreads - 1);       // also owns bin N (local slot 16384)
  float2* mine = acc + pad(32u * tid);                     // pad(32 t + j) = pad(32 t) + j
  if (a.pw.done) {
    // launched as the compress grid's programmatic dependent: wait until this
    // rank's own segment of the chunk is written
    if (tid == 0) {
      const uint32_t* f = a.pw.done + chunk;
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - a.pw.tag) >= 0) break;      // wraparound-safe: tags only grow
        __nanosleep(256);
      }
    }
    __syncthreads();
  }
  if (TAGS && a.pw.dtab) {
    // in-kernel transports: every peer's compress kernel has released this
    // chunk (direct reads: its own tag, remote; kernel pushes: both CTAs'
    // tags, local, set after their stores into our gather buffer)
    const uint32_t ts = a.pw.tstride;
    if (tid < (uint32_t)a.pw.nranks * ts && (int)(tid / ts) != a.pw.me) {
      const uint32_t* f = a.pw.dtab[tid / ts] + chunk * ts + tid % ts;
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - a.pw.target) >= 0) break;
        __nanosleep(128);
      }
    }
    __syncthreads();
  } else if (a.pw.flags) {
    // peer exchange: every peer's copy of this chunk's piece has landed
    if (tid < (uint32_t)a.pw.nranks && (int)tid != a.pw.me) {
      const uint32_t* f = a.pw.flags + tid * a.pw.stride + (chunk - a.pw.first) / a.pw.per;
      for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if ((int32_t)(v - a.pw.target) >= 0) break;
        __nanosleep(128);
      }
    }
    __syncthreads();
  }
  // message w of the step: a peer's own buffer (direct reads) or the gathered stack
  auto mbase = [&](int w) -> const uint8_t* {
    if constexpr (TAGS) {
      if (a.pw.mtab) return a.pw.mtab[w];
    }
    return a.messages + (uint64_t)w * a.stride;
  };
  if (!a.spectrum && tid < (uint32_t)a.W && blockIdx.x / 2 + a.ahead < a.count && !(dbg & 8u) &&
      (!TAGS || !a.pw.mtab || (int)tid == a.pw.me)) {
    // message segments of the chunk the next wave decodes here (CTA r: half of each)
    const ChunkInfo cn = a.chunks[chunk + a.ahead];
    const uint32_t seg = (uint32_t)(cn.code_off + 4ull * ((cn.code_cap + 3u) & ~3u));
    const uint32_t half = ((seg / 2) + 15u) & ~15u;
    const uint32_t lo = r ? half : 0u, bytes = r ? seg - half : half;
    if (bytes)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                   ::"l"(mbase((int)tid) + cn.seg_off + lo), "r"(bytes) : "memory");
  }

  if (a.spectrum) {
    // dense spectrum input (inverse_spectrum / debug hook)
    const float2* X = a.spectrum + ci.bin_off + 32u * blk;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) mine[j] = X[j];
    if (binN) acc[pad(kHalfBins)] = a.spectrum[ci.bin_off + kN];
  } else {
    {
      float4* z = reinterpret_cast<float4*>(acc);
      for (uint32_t e = tid; e < (kPadded + 64) / 2; e += kThreads) z[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const uint32_t N = (uint32_t)a.q.n_bits;
    FGC_TS(0);
    for (int w0 = 0; w0 < a.W; w0 += kDecBatch) {
      const int G = min(kDecBatch, a.W - w0);
      // 1a. every bitmap word of the batch (thread t: blocks 2t, 2t+1), block code prefixes;
      //     the code streams of the messages that fit are staged in smem meanwhile
      uint32_t cnt2[kDecBatch][2];
      {
        // Every load of the batch in flight at once: the segment headers
        // (one latency), then the bitmaps and the staged code streams
        // together (a second).  Issued message by message, each header load
        // serialised the next message's loads behind it.
        const uint8_t* sg[kDecBatch];
        uint32_t nnz[kDecBatch];
#pragma unroll
        for (int i = 0; i < kDecBatch; ++i) {
          sg[i] = mbase(w0 + min(i, G - 1)) + ci.seg_off;
          nnz[i] = (i < G) ? __ldg(reinterpret_cast<const uint32_t*>(sg[i])) : 0u;
        }
        uint4 q4[kDecBatch];
        uint32_t qN[kDecBatch];
#pragma unroll
        for (int i = 0; i < kDecBatch; ++i) {
          q4[i] = (i < G) ? __ldg(reinterpret_cast<const uint4*>(sg[i] + kSegHeader) + tid) : make_uint4(0, 0, 0, 0);
          qN[i] = (i < G && tid == 0) ? __ldg(reinterpret_cast<const uint32_t*>(sg[i] + kSegHeader) + 2 * kThreads * 2)
                                      : 0u;
        }
        // message i's used code words go to stage[off[i], off[i] + s4[i]) (uint4 units) while they fit
        uint32_t off[kDecBatch], s4[kDecBatch];
        uint32_t used_total = 0;
#pragma unroll
        for (int i = 0; i < kDecBatch; ++i) {
          const uint32_t used4 =
              (uint32_t)min((((uint64_t)nnz[i] * N + 127u) >> 7), (uint64_t)((ci.code_cap + 3u) >> 2));
          FGC_CHECK(nnz[i] <= 2u * ci.bins);
          const bool st = i < G && !(dbg & 4u) && 4u * (used_total + used4) <= kDecStageWords;
          off[i] = used_total;
          s4[i] = st ? used4 : 0u;
          if (tid == 0) sh.soff[i] = st ? 4u * used_total : ~0u;
          used_total += s4[i];
        }
        constexpr int kPer = kDecStageWords / 4 / kThreads;
        uint4 tmp[kPer];
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const uint32_t e = tid + u * kThreads;
          if (e < used_total) {
            const uint8_t* src = sg[0];       // the message holding staged word e (static indices only)
            uint32_t o = off[0];
#pragma unroll
            for (int j = 1; j < kDecBatch; ++j)
              if (s4[j] && e >= off[j]) { src = sg[j]; o = off[j]; }
            tmp[u] = __ldg(reinterpret_cast<const uint4*>(src + ci.code_off) + (e - o));
          }
        }
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const uint32_t e = tid + u * kThreads;
          if (e < used_total) sh.stage[e] = tmp[u];
        }
#pragma unroll
        for (int i = 0; i < kDecBatch; ++i) {
          cnt2[i][0] = cnt2[i][1] = 0u;
          if (i < G) {
            const uint4 nat = make_uint4(ballot_to_wire(q4[i].x), ballot_to_wire(q4[i].y), ballot_to_wire(q4[i].z),
                                         ballot_to_wire(q4[i].w));
            reinterpret_cast<uint4*>(sh.bm[i])[tid] = nat;
            cnt2[i][0] = __popc(nat.x) + __popc(nat.y);
            cnt2[i][1] = __popc(nat.z) + __popc(nat.w);
            if (tid == 0) sh.bmN[i] = ballot_to_wire(qN[i]) & 3u;
          }
        }
      }
      uint4 tot;
      const uint4 pre = block_exclusive_scan4<kThreads>(
          make_uint4(cnt2[0][0] + cnt2[0][1], cnt2[1][0] + cnt2[1][1], cnt2[2][0] + cnt2[2][1],
                     cnt2[3][0] + cnt2[3][1]), sh.scan, tot);
      const uint32_t pr[4] = {pre.x, pre.y, pre.z, pre.w};
#pragma unroll
      for (int i = 0; i < kDecBatch; ++i) {
        if (i < G) {
          sh.pref[i][2 * tid] = pr[i];
          sh.pref[i][2 * tid + 1] = pr[i] + cnt2[i][0];
        }
      }
      __syncthreads();
      if (w0 == 0) FGC_TS(7);
      // 1b. my block's slots, message by message in worker order (single
      //     writer per slot: deterministic).  Staged messages read their codes
      //     from shared memory by code index (N = 8 / 16: one byte / halfword
      //     load), the others through a register window over global memory.
      {
        const uint32_t mask = (1u << N) - 1u;
        float* minef = reinterpret_cast<float*>(mine);
        float* nf = reinterpret_cast<float*>(acc + pad(kHalfBins));
        const QuantParams& qq = a.q;
        auto add = [&](float* f, uint32_t pos, uint32_t c, float wt) {
          // decode_code (quantizer.py:239-253) without branches
          const bool neg = c > qq.npos;
          const uint32_t e = qq.pbase + c - 1u - (neg ? qq.npos : 0u);
          const float v = __uint_as_float((e << qq.shift) | (neg ? 0x80000000u : 0u));
          f[pos] += (c ? v : 0.0f) * wt;
        };
#pragma unroll 1
        for (int i = 0; i < G; ++i) {
          const uint32_t m0 = sh.bm[i][2 * blk], m1 = sh.bm[i][2 * blk + 1], m2 = binN ? sh.bmN[i] : 0u;
          if (!(m0 | m1 | m2)) continue;
          const float wt = a.wts.w[w0 + i];
          uint32_t k = sh.pref[i][blk];                       // stream index of my first code
          const uint32_t so = sh.soff[i];
          if (so != ~0u && N == 8) {
            const uint8_t* s8 = reinterpret_cast<const uint8_t*>(sh.stage) + 4u * so;
            auto walk = [&](uint32_t m, float* f) {
              while (m) {
                const uint32_t pos = __ffs(m) - 1;
                m &= m - 1;
                FGC_CHECK(k < 4u * (kDecStageWords - so));
                add(f, pos, s8[k++], wt);
              }
            };
            walk(m0, minef);
            walk(m1, minef + 32);
            walk(m2, nf);
          } else if (so != ~0u && N == 16) {
            const uint16_t* s16 = reinterpret_cast<const uint16_t*>(sh.stage) + 2u * so;
            auto walk = [&](uint32_t m, float* f) {
              while (m) {
                const uint32_t pos = __ffs(m) - 1;
                m &= m - 1;
                FGC_CHECK(k < 2u * (kDecStageWords - so));
                add(f, pos, s16[k++], wt);
              }
            };
            walk(m0, minef);
            walk(m1, minef + 32);
            walk(m2, nf);
          } else if (so != ~0u) {
            const uint32_t* st = reinterpret_cast<const uint32_t*>(sh.stage) + so;
            uint32_t bit = k * N;
            auto walk = [&](uint32_t m, float* f) {
              while (m) {
                const uint32_t pos = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t wi = bit >> 5;
                FGC_CHECK(so + wi + 1 < kDecStageWords + 8);
                add(f, pos, __funnelshift_r(st[wi], st[wi + 1], bit & 31u) & mask, wt);
                bit += N;
              }
            };
            walk(m0, minef);
            walk(m1, minef + 32);
            walk(m2, nf);
          } else {
            // codes from global memory through a 4-word register window
            const uint32_t* cw = reinterpret_cast<const uint32_t*>(mbase(w0 + i) + ci.seg_off + ci.code_off);
            const uint32_t wb = (k * N) >> 5;
            uint32_t A = wb < ci.code_cap ? __ldg(cw + wb) : 0u;
            uint32_t B = wb + 1 < ci.code_cap ? __ldg(cw + wb + 1) : 0u;
            uint32_t C = wb + 2 < ci.code_cap ? __ldg(cw + wb + 2) : 0u;
            uint32_t D = wb + 3 < ci.code_cap ? __ldg(cw + wb + 3) : 0u;
            uint32_t o = (k * N) & 31u, nxt = wb + 4u;
            auto walk = [&](uint32_t m, float* f) {
              while (m) {
                const uint32_t pos = __ffs(m) - 1;
                m &= m - 1;
                const uint32_t c = __funnelshift_r(A, B, o) & mask;
                o += N;
                if (o >= 32u) {
                  o -= 32u;
                  A = B; B = C; C = D;
                  D = nxt < ci.code_cap ? __ldg(cw + nxt) : 0u;
                  ++nxt;
                }
                add(f, pos, c, wt);
              }
            };
            walk(m0, minef);
            walk(m1, minef + 32);
            walk(m2, nf);
          }
        }
      }
      if (w0 == 0) FGC_TS(8);
      __syncthreads();                                      // bm / pref reusable
    }
    FGC_TS(1);
  }
  cluster.sync();                                           // every X entry of the chunk is final
  FGC_TS(2);

  // ---- phase 2: my groups -> Y_0, Y_1 at m = k and m = M - k (registers)
  const float2* peer = cluster.map_shared_rank(acc, r ^ 1);
  float2 ys[8][4];                                          // {Y0[k], Y1[k], Y0[M-k], Y1[M-k]}
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t k = (r ? 4096u : 0u) + tid + 512u * i;
    float2 xk, xMk, xkM, xNk;                               // X[k], X[M-k], X[k+M], X[N-k]
    if (r == 0) {
      xk = acc[pad(k)];
      xMk = acc[pad(8192u - k)];
      xkM = acc[pad(8192u + k)];
      xNk = acc[pad(16384u - k)];
    } else {
      xk = acc[pad(k - 4096u)];
      xkM = acc[pad(k + 4096u)];
      if (k == 4096u) {                                     // bins 12288, 28672 live in CTA 0
        xMk = peer[pad(4096u)];
        xNk = peer[pad(12288u)];
      } else {
        xMk = acc[pad(12288u - k)];
        xNk = acc[pad(20480u - k)];
      }
    }
    if (k == 0) { xk.y = 0.f; xNk.y = 0.f; }                // imag of DC / Nyquist ignored
    y_group(xk, xMk, xkM, xNk, tw(sh.thi, sh.tlo, k), ys[i]);
  }
  // CTA 1's extra group k = 8192 (m = M - m = 8192): bins 8192 (slot 4096) and 24576 (slot 12288)
  float2 y8192_0 = make_float2(0.f, 0.f), y8192_1 = make_float2(0.f, 0.f);
  if (r == 1 && tid == 0) {
    const float2 x8 = acc[pad(4096u)], x24 = acc[pad(12288u)];
    float2 y[4];
    y_group(x8, x8, x24, x24, tw(sh.thi, sh.tlo, 8192u), y);
    y8192_0 = y[0];
    y8192_1 = y[1];
  }
  FGC_TS(3);
  cluster.sync();                                           // all X reads done (both CTAs)
  FGC_TS(4);
  float2* yo = acc;                                         // Y_r in natural m order (FFT input)
  float2* yp = cluster.map_shared_rank(acc, r ^ 1);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t k = (r ? 4096u : 0u) + tid + 512u * i;
    yo[pad(k)] = r ? ys[i][1] : ys[i][0];
    yp[pad(k)] = r ? ys[i][0] : ys[i][1];
    if (k != 0) {
      yo[pad(kHalfBins - k)] = r ? ys[i][3] : ys[i][2];
      yp[pad(kHalfBins - k)] = r ? ys[i][2] : ys[i][3];
    }
  }
  if (r == 1 && tid == 0) {
    yo[pad(8192u)] = y8192_1;
    yp[pad(8192u)] = y8192_0;
  }
  cluster.sync();                                           // Y_r complete in both CTAs
  FGC_TS(9);

  // inverse 16384-point FFT of Y_r, natural-order output
  float2 v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = acc[pad(tid + 512u * j)];
  __syncthreads();
  fft_pass12<true>(v, sh.x, sh.t1024);
  __syncthreads();
  FGC_TS(5);
  const float scale = 1.0f / (float)kN;
  float* out = a.out + ci.in_off;
  float dbg_sum = 0.f;
#pragma unroll
  for (uint32_t c = 0; c < 2; ++c) {                        // (unrolled: the two columns' loads overlap)
    const uint32_t k = tid + 512u * c;
    float2 o[16];
    fft_pass3<true>(k, sh.x, o, sh.thi, sh.tlo);
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      const uint32_t p = k + 1024u * m;
      if (!(dbg & 2u)) *reinterpret_cast<float2*>(out + 4ull * p + 2 * r) = make_float2(o[m].x * scale, o[m].y * scale);
      else dbg_sum += o[m].x + o[m].y;
    }
  }
  if (dbg & 2u) out[tid + 512 * r] = dbg_sum;
  FGC_TS(6);
}

template <class K>
fgc_status set_smem(K kernel, size_t bytes) {
  FGC_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return FGC_OK;
}

}  // namespace

bool fused_available() { return true; }

static uint32_t g_fused_dbg_host = 0;
// the knobs and timestamp buffer for kernels in other translation units
void fused_debug_state(uint32_t& knobs, unsigned long long*& ts) {
  knobs = g_fused_dbg_host;
  void* p = nullptr;
  ts = (knobs && cudaGetSymbolAddress(&p, g_fused_ts) == cudaSuccess) ? static_cast<unsigned long long*>(p) : nullptr;
  if (!ts) knobs = 0;
}

}  // namespace fgc

// Internal instrumentation hooks (not part of the public header).
extern "C" int fgc_debug_set_fused_knobs(uint32_t knobs) {
  fgc::g_fused_dbg_host = knobs;
  return cudaMemcpyToSymbol(fgc::g_fused_dbg, &knobs, sizeof(knobs)) == cudaSuccess ? 0 : 1;
}
extern "C" int fgc_debug_set_compress_kernel(int k);
extern "C" int fgc_debug_fused_timestamps(unsigned long long* host, uint32_t count) {
  if (count > 2048 * 16) count = 2048 * 16;
  return cudaMemcpyFromSymbol(host, fgc::g_fused_ts, count * sizeof(unsigned long long)) == cudaSuccess ? 0 : 1;
}

namespace fgc {

fgc_status fused_tables_init(FusedTables** t, cudaStream_t s) {
  FusedTables* ft = new FusedTables();
  cudaError_t e = cudaMalloc(&ft->thi, 256 * sizeof(float2));
  if (e == cudaSuccess) e = cudaMalloc(&ft->tlo, 256 * sizeof(float2));
  if (e == cudaSuccess) e = cudaMalloc(&ft->t1024, 1024 * sizeof(float2));
  if (e != cudaSuccess) {
    fused_tables_free(ft);
    return cuda_check(e, "cudaMalloc");
  }
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    ft->wave = (uint32_t)(sms / 2);
  }
  k_init_tables<<<1, 1024, 0, s>>>(ft->thi, ft->tlo, ft->t1024);
  FGC_LAUNCHED(1);
  static bool attrs = false;
  if (!attrs) {
    const size_t cs = sizeof(CompressShared);
    FGC_TRY(set_smem(k_fused_compress<float, false, false>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, false, false>, cs));
    FGC_TRY(set_smem(k_fused_compress<float, true, false>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, true, false>, cs));
    FGC_TRY(set_smem(k_fused_compress<float, false, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, false, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<float, true, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, true, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<float, false, false, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, false, false, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<float, false, true, true>, cs));
    FGC_TRY(set_smem(k_fused_compress<double, false, true, true>, cs));
    FGC_TRY(set_smem(k_fused_decode<false>, sizeof(DecodeShared)));
    FGC_TRY(set_smem(k_fused_decode<true>, sizeof(DecodeShared)));
    attrs = true;
  }
  *t = ft;
  return FGC_OK;
}

void fused_tables_free(FusedTables* t) {
  if (!t) return;
  cudaFree(t->thi);
  cudaFree(t->tlo);
  cudaFree(t->t1024);
  delete t;
}

// Which compress kernel runs the 65536-sample chunks: 2 = k_fused_compress
// above (default), 4 = the 4-CTA-cluster kernel of fused4.cu (two CTAs per
// SM; another FFT factorisation, oracle-exact on its own coefficients;
// measured slower: 226 vs 185 us at 25.6M floats, its cluster barriers
// across 4 CTAs on shared SMs stall ~39% of the time), 1 = fused_w.cu (1024
// threads, lane-pair FFT columns; bit-identical; 196 vs 195 us).
// FGC_COMPRESS_KERNEL sets the default; fgc_debug_set_compress_kernel switches it.
static int g_compress_kernel = -1;
static int compress_kernel() {
  if (g_compress_kernel < 0) {
    const char* e = getenv("FGC_COMPRESS_KERNEL");
    g_compress_kernel = (e && e[0] == '4') ? 4 : (e && e[0] == '1') ? 1 : 2;
  }
  return g_compress_kernel;
}

static fgc_status launch_compress_impl(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first,
                                       uint32_t count, const void* grad, int dtype, int half_pass,
                                       const QuantParams& q, uint8_t* message, uint32_t* flags,
                                       float2* fb_spec, float2* dbg, cudaStream_t s, PieceCounter pc) {
  if (!count) return FGC_OK;
  // (the alternative kernels do not implement the kernel-push transport)
  if (compress_kernel() == 4 && !pc.npeers)
    return launch_compress4(t->thi, t->tlo, t->wave, d_chunks, first, count, grad, dtype, half_pass, q, message,
                            flags, fb_spec, dbg, s, pc);
  if (compress_kernel() == 1 && !pc.npeers)
    return launch_compress_w(t->thi, t->tlo, t->t1024, t->wave, d_chunks, first, count, grad, dtype, half_pass, q,
                             message, flags, fb_spec, dbg, s, pc);
  CompressArgs a{d_chunks, first, grad, q, message, flags, t->thi, t->tlo, t->t1024, fb_spec, dbg, count, t->wave,
                 pc};
  const size_t smem = sizeof(CompressShared);
  const dim3 grid(2 * count), block(kThreads);
  const bool f64 = dtype == FGC_DTYPE_F64, h = half_pass != 0;
#define FGC_LAUNCH_FC(T, D, H) k_fused_compress<T, D, H><<<grid, block, smem, s>>>(a)
#define FGC_LAUNCH_FP(T, H) k_fused_compress<T, false, H, true><<<grid, block, smem, s>>>(a)
  if (pc.npeers && !dbg) {
    if (f64) { if (h) FGC_LAUNCH_FP(double, true); else FGC_LAUNCH_FP(double, false); }
    else { if (h) FGC_LAUNCH_FP(float, true); else FGC_LAUNCH_FP(float, false); }
  } else if (dbg) {
    if (f64) { if (h) FGC_LAUNCH_FC(double, true, true); else FGC_LAUNCH_FC(double, true, false); }
    else { if (h) FGC_LAUNCH_FC(float, true, true); else FGC_LAUNCH_FC(float, true, false); }
  } else {
    if (f64) { if (h) FGC_LAUNCH_FC(double, false, true); else FGC_LAUNCH_FC(double, false, false); }
    else { if (h) FGC_LAUNCH_FC(float, false, true); else FGC_LAUNCH_FC(float, false, false); }
  }
#undef FGC_LAUNCH_FC
#undef FGC_LAUNCH_FP
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_fused_compress(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                 const void* grad, int dtype, int half_pass, const QuantParams& q,
                                 uint8_t* message, uint32_t* flags, float2* fb_spec,
                                 cudaStream_t s, PieceCounter pc) {
  if (q.n_bits > 16) {
    set_error("fused kernels take N <= 16");
    return FGC_ERR_UNSUPPORTED;
  }
  return launch_compress_impl(t, d_chunks, first, count, grad, dtype, half_pass, q, message, flags, fb_spec,
                              nullptr, s, pc);
}

fgc_status launch_fused_spectrum(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                 const void* grad, int dtype, int half_pass, float2* spectrum, uint32_t* flags,
                                 cudaStream_t s) {
  QuantParams q{};
  q.n_bits = 8;
  return launch_compress_impl(t, d_chunks, first, count, grad, dtype, half_pass, q, nullptr, flags,
                              nullptr, spectrum, s, PieceCounter());
}

fgc_status launch_fused_decode(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                               const uint8_t* messages, int W, uint64_t stride, const Weights& wts,
                               const QuantParams& q, float* out, cudaStream_t s, PieceWait pw) {
  if (!count) return FGC_OK;
  DecodeArgs a{d_chunks, first, messages, W, stride, wts, q, out, t->thi, t->tlo, t->t1024, nullptr, count, t->wave,
               pw};
  if (pw.done) {
    // programmatic dependent of the compress grid just launched on s: it may
    // start once every compress CTA is resident, and waits per chunk
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * count);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = sizeof(DecodeShared);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (pw.dtab) FGC_CUDA(cudaLaunchKernelEx(&cfg, k_fused_decode<true>, a));
    else FGC_CUDA(cudaLaunchKernelEx(&cfg, k_fused_decode<false>, a));
  } else {
    if (pw.dtab) k_fused_decode<true><<<2 * count, kThreads, sizeof(DecodeShared), s>>>(a);
    else k_fused_decode<false><<<2 * count, kThreads, sizeof(DecodeShared), s>>>(a);
  }
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_fused_inverse(const FusedTables* t, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                                const float2* spectrum, float* out, cudaStream_t s) {
  if (!count) return FGC_OK;
  DecodeArgs a{};
  a.chunks = d_chunks;
  a.first = first;
  a.out = out;
  a.thi = t->thi;
  a.tlo = t->tlo;
  a.t1024 = t->t1024;
  a.spectrum = spectrum;
  a.W = 0;
  k_fused_decode<false><<<2 * count, kThreads, sizeof(DecodeShared), s>>>(a);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

}  // namespace fgc

extern "C" int fgc_debug_set_compress_kernel(int k) {
  fgc::g_compress_kernel = (k == 4 || k == 1) ? k : 2;
  return 0;
}

// Diagnostics: 2-CTA clusters of the fused compress / decode that fit the GPU
// at once (cudaOccupancyMaxActiveClusters; the wave size of the fused grids).
extern "C" int fgc_debug_fused_max_clusters(int which) {
  using namespace fgc;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * 1024);
  cfg.blockDim = dim3(kThreads);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int n = -1;
  cudaError_t e;
  if (which == 0) {
    cfg.dynamicSmemBytes = sizeof(CompressShared);
    e = cudaOccupancyMaxActiveClusters(&n, k_fused_compress<float, false, false>, &cfg);
  } else {
    cfg.dynamicSmemBytes = sizeof(DecodeShared);
    e = cudaOccupancyMaxActiveClusters(&n, k_fused_decode<false>, &cfg);
  }
  return e == cudaSuccess ? n : -(int)e;
}
