// Energy-mode drop sets (spectral.py:134-139, _drop_set with mode "energy"):
//
//   energies = bin_weights(L) * |X|**2          (spectral.py:150, Parseval weights)
//   order    = argsort(|X|, stable)
//   budget   = theta**2 * energies.sum()         (numpy pairwise summation)
//   k        = searchsorted(cumsum(energies[order]), budget, side="right")
//   dropped  = order[:k]
//
// Bit-exact with numpy given the same coefficients: the magnitude key is
// numpy's SIMD cabs (cabs_key), the sum replays numpy's pairwise_sum tree
// (8-way unrolled leaves of <= 128, halving splits rounded to multiples of
// 8), the ordering is a stable segmented radix sort of the fp64 keys (CUB),
// and the cumulative sum is evaluated sequentially in sorted order -- the
// rounding of each prefix matters, so one thread walks each chunk.  The
// resulting drop mask feeds the common quantize + pack kernel.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {
namespace {

// per bin: exact key, weighted energy, original index
template <class T2>
__global__ void k_energy_prep(const ChunkInfo* chunks, uint32_t first, const T2* spectrum, double* keys,
                              uint32_t* idx, double* energy) {
  const ChunkInfo ci = chunks[first + blockIdx.y];
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= ci.bins) return;
  const T2 x = spectrum[ci.bin_off + b];
  const double mag = cabs_key((double)x.x, (double)x.y);
  const bool single = (b == 0) || ((ci.len % 2u) == 0u && b == ci.bins - 1);   // DC / Nyquist weight 1
  keys[ci.bin_off + b] = mag;
  idx[ci.bin_off + b] = b;
  energy[ci.bin_off + b] = (single ? 1.0 : 2.0) * __dmul_rn(mag, mag);
}

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) of a[0, n)
__device__ double pairwise_sum(const double* a, uint32_t n) {
  // the recursion as an explicit post-order walk: a node is a leaf (n <= 128)
  // or left + right with the split rounded down to a multiple of 8
  struct F { uint32_t off, n; int state; };
  F fs[40];
  double vals[40];
  int fp = 0, vp = 0;
  fs[fp++] = {0, n, 0};
  while (fp) {
    F& f = fs[fp - 1];
    if (f.n <= 128) {
      double res;
      if (f.n < 8) {
        res = 0.0;
        for (uint32_t i = 0; i < f.n; ++i) res = __dadd_rn(res, a[f.off + i]);
      } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[f.off + j];
        uint32_t i = 8;
        for (; i < f.n - (f.n % 8u); i += 8)
          for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[f.off + i + j]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < f.n; ++i) res = __dadd_rn(res, a[f.off + i]);
      }
      vals[vp++] = res;
      --fp;
      continue;
    }
    uint32_t n2 = f.n / 2;
    n2 -= n2 % 8u;
    if (f.state == 0) {                 // descend left
      f.state = 1;
      fs[fp++] = {f.off, n2, 0};
    } else if (f.state == 1) {          // descend right
      f.state = 2;
      fs[fp++] = {f.off + n2, f.n - n2, 0};
    } else {                            // combine
      const double right = vals[--vp];
      const double left = vals[--vp];
      vals[vp++] = __dadd_rn(left, right);
      --fp;
    }
  }
  return vals[0];
}

__global__ void k_energy_total(const ChunkInfo* chunks, uint32_t first, uint32_t count, const double* energy,
                               double* total) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  const ChunkInfo ci = chunks[first + c];
  total[c] = pairwise_sum(energy + ci.bin_off, ci.bins);
}

__global__ void k_energy_gather(const ChunkInfo* chunks, uint32_t first, const uint32_t* sidx, const double* energy,
                                double* sorted_e) {
  const ChunkInfo ci = chunks[first + blockIdx.y];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ci.bins) return;
  sorted_e[ci.bin_off + i] = energy[ci.bin_off + sidx[ci.bin_off + i]];
}

// k = #{i : cumsum(sorted energies)[i] <= budget}: one thread per chunk, in order
__global__ void k_energy_cut(const ChunkInfo* chunks, uint32_t first, uint32_t count, const double* sorted_e,
                             const double* total, double theta, uint32_t* kcut) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= count) return;
  const ChunkInfo ci = chunks[first + c];
  if (theta == 0.0) { kcut[c] = 0; return; }          // spectral.py:135-136
  const double budget = __dmul_rn(__dmul_rn(theta, theta), total[c]);
  const double* e = sorted_e + ci.bin_off;
  double run = 0.0;
  uint32_t k = 0;
  const uint32_t n = ci.bins;
  uint32_t i = 0;
  for (; i + 4 <= n; i += 4) {
    const double e0 = e[i], e1 = e[i + 1], e2 = e[i + 2], e3 = e[i + 3];
    run = __dadd_rn(run, e0); k += run <= budget;
    run = __dadd_rn(run, e1); k += run <= budget;
    run = __dadd_rn(run, e2); k += run <= budget;
    run = __dadd_rn(run, e3); k += run <= budget;
  }
  for (; i < n; ++i) { run = __dadd_rn(run, e[i]); k += run <= budget; }
  kcut[c] = k;
}

__global__ void k_energy_mask(const ChunkInfo* chunks, uint32_t first, const uint32_t* sidx, const uint32_t* kcut,
                              uint8_t* drop) {
  const ChunkInfo ci = chunks[first + blockIdx.y];
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ci.bins) return;
  drop[ci.bin_off + sidx[ci.bin_off + i]] = (i < kcut[blockIdx.y]) ? 1u : 0u;
}

__global__ void k_seg_offsets(const ChunkInfo* chunks, uint32_t first, uint32_t count, int* offs) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c > count) return;
  const ChunkInfo ci = chunks[first + (c < count ? c : count - 1)];
  offs[c] = (int)(c < count ? ci.bin_off : ci.bin_off + ci.bins);
}

inline uint32_t cdiv32(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

}  // namespace

fgc_status EnergyScratch::ensure(uint64_t bins, uint32_t chunks) {
  if (bins <= cap_bins && chunks <= cap_chunks) return FGC_OK;
  free_all();
  FGC_CUDA(cudaMalloc(&keys, sizeof(double) * bins));
  FGC_CUDA(cudaMalloc(&keys2, sizeof(double) * bins));
  FGC_CUDA(cudaMalloc(&energy, sizeof(double) * bins));
  FGC_CUDA(cudaMalloc(&sorted_e, sizeof(double) * bins));
  FGC_CUDA(cudaMalloc(&idx, sizeof(uint32_t) * bins));
  FGC_CUDA(cudaMalloc(&idx2, sizeof(uint32_t) * bins));
  FGC_CUDA(cudaMalloc(&drop, bins));
  FGC_CUDA(cudaMalloc(&total, sizeof(double) * chunks));
  FGC_CUDA(cudaMalloc(&kcut, sizeof(uint32_t) * chunks));
  FGC_CUDA(cudaMalloc(&offs, sizeof(int) * (chunks + 1)));
  size_t tb = 0;
  FGC_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tb, keys, keys2, idx, idx2, (int)bins, (int)chunks,
                                                    offs, offs + 1));
  FGC_CUDA(cudaMalloc(&temp, tb));
  temp_bytes = tb;
  cap_bins = bins;
  cap_chunks = chunks;
  return FGC_OK;
}

void EnergyScratch::free_all() {
  cudaFree(keys); cudaFree(keys2); cudaFree(energy); cudaFree(sorted_e);
  cudaFree(idx); cudaFree(idx2); cudaFree(drop); cudaFree(total); cudaFree(kcut); cudaFree(offs); cudaFree(temp);
  keys = keys2 = energy = sorted_e = total = nullptr;
  idx = idx2 = kcut = nullptr;
  drop = nullptr;
  offs = nullptr;
  temp = nullptr;
  cap_bins = 0;
  cap_chunks = 0;
  temp_bytes = 0;
}

// Drop mask (1 = dropped) for chunks [first, first + count) of a chunk-major
// float2 spectrum whose bins start at bin_off(first) = bin0.
fgc_status energy_drop_mask(EnergyScratch& e, const ChunkInfo* d_chunks, uint32_t first, uint32_t count,
                            uint64_t bin0, uint64_t nbins, uint32_t max_bins, const void* spectrum, int f64,
                            double theta, cudaStream_t s, const uint8_t** drop_out) {
  if (!count) return FGC_OK;
  FGC_TRY(e.ensure(bin0 + nbins, count));
  const dim3 grid(cdiv32(max_bins, 256), count);
  if (f64)
    k_energy_prep<double2><<<grid, 256, 0, s>>>(d_chunks, first, static_cast<const double2*>(spectrum), e.keys,
                                                e.idx, e.energy);
  else
    k_energy_prep<float2><<<grid, 256, 0, s>>>(d_chunks, first, static_cast<const float2*>(spectrum), e.keys, e.idx,
                                               e.energy);
  FGC_LAUNCHED(1);
  k_energy_total<<<cdiv32(count, 64), 64, 0, s>>>(d_chunks, first, count, e.energy, e.total);
  FGC_LAUNCHED(1);
  k_seg_offsets<<<cdiv32(count + 1, 128), 128, 0, s>>>(d_chunks, first, count, e.offs);
  FGC_LAUNCHED(1);
  size_t tb = e.temp_bytes;
  // sorted copies land at the same bin offsets (segments are the chunks' bin ranges)
  FGC_CUDA(cub::DeviceSegmentedRadixSort::SortPairs(e.temp, tb, e.keys, e.keys2, e.idx, e.idx2,
                                                    (int)(bin0 + nbins), (int)count, e.offs, e.offs + 1, 0,
                                                    sizeof(double) * 8, s));
  FGC_LAUNCHED(1);
  k_energy_gather<<<grid, 256, 0, s>>>(d_chunks, first, e.idx2, e.energy, e.sorted_e);
  FGC_LAUNCHED(1);
  k_energy_cut<<<cdiv32(count, 32), 32, 0, s>>>(d_chunks, first, count, e.sorted_e, e.total, theta, e.kcut);
  FGC_LAUNCHED(1);
  k_energy_mask<<<grid, 256, 0, s>>>(d_chunks, first, e.idx2, e.kcut, e.drop);
  FGC_LAUNCHED(1);
  *drop_out = e.drop;
  return FGC_OK;
}

}  // namespace fgc
