// FGC1 wire format on the device (codec.serialize / deserialize,
// codec.py:340-441) and conversions between the fixed-capacity device
// message and ChunkPayload arrays (codec.py:112-125).
//
// Device segment: [u32 nnz][12 B 0]
// [bitmap words: wire bytes, MSB-first per byte][pad16][code words, LSB-first].
// The wire chunk is [u32 nnz][ceil(slots/8) bitmap bytes][ceil(nnz*N/8) code
// bytes], concatenated after the 36-byte header.
#include <cuda_runtime.h>

#include "fgc_device.cuh"
#include "fgc_internal.h"

namespace fgc {

namespace {

constexpr int kWireThreads = 256;

struct Header36 {
  uint8_t b[FGC_HEADER_BYTES];
};

__device__ __forceinline__ uint64_t wire_chunk_bytes(const ChunkInfo& ci, uint32_t nnz, int N) {
  return 4ull + (ci.slots + 7) / 8 + ((uint64_t)nnz * N + 7) / 8;
}

__global__ void k_wire_sizes(const ChunkInfo* chunks, uint32_t n, const uint8_t* message, int N, uint64_t* sizes) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const ChunkInfo ci = chunks[c];
  const uint32_t nnz = *reinterpret_cast<const uint32_t*>(message + ci.seg_off);
  sizes[c] = wire_chunk_bytes(ci, nnz, N);
}

// In-place exclusive scan of n uint64 (single CTA, tile-sequential).
__global__ void k_scan_u64(uint64_t* v, uint32_t n, uint64_t* total_out, uint64_t add) {
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t t0 = 0; t0 < n; t0 += blockDim.x) {
    const uint32_t i = t0 + threadIdx.x;
    const uint64_t x = (i < n) ? v[i] : 0;
    uint64_t s = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane == 31) warp_sums[warp] = s;
    __syncthreads();
    if (warp == 0) {
      uint64_t ws = (lane < nw) ? warp_sums[lane] : 0;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, ws, d);
        if (lane >= d) ws += y;
      }
      if (lane < nw) warp_sums[lane] = ws;
    }
    __syncthreads();
    const uint64_t base = carry + (warp ? warp_sums[warp - 1] : 0);
    if (i < n) v[i] = base + s - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[nw - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total_out = carry + add;
}

__global__ void k_wire_copy(const ChunkInfo* chunks, const uint8_t* message, int N, const uint64_t* offsets,
                            Header36 hdr, uint8_t* wire) {
  const uint32_t c = blockIdx.x;
  if (c == 0 && threadIdx.x < FGC_HEADER_BYTES) wire[threadIdx.x] = hdr.b[threadIdx.x];
  const ChunkInfo ci = chunks[c];
  const uint8_t* seg = message + ci.seg_off;
  const uint32_t nnz = *reinterpret_cast<const uint32_t*>(seg);
  const uint64_t bmb = (ci.slots + 7) / 8;
  const uint64_t cb = ((uint64_t)nnz * N + 7) / 8;
  FGC_CHECK(nnz <= ci.slots && (uint64_t)nnz * N <= 32ull * ci.code_cap);
  uint8_t* dst = wire + FGC_HEADER_BYTES + offsets[c];
  const uint64_t total = 4 + bmb + cb;
  for (uint64_t j = threadIdx.x; j < total; j += blockDim.x) {
    uint8_t b;
    if (j < 4) b = seg[j];
    else if (j < 4 + bmb) b = seg[kSegHeader + (j - 4)];
    else b = seg[ci.code_off + (j - 4 - bmb)];
    dst[j] = b;
  }
}

__device__ __forceinline__ uint8_t wire_byte(const uint8_t* p, uint64_t j, uint64_t avail) {
  return j < avail ? p[j] : 0;
}

__global__ void k_unwire(const ChunkInfo* chunks, const uint8_t* wire, const uint64_t* chunk_offsets, int N,
                         uint8_t* message, uint32_t* popcounts) {
  __shared__ uint32_t scan[40];
  const uint32_t c = blockIdx.x;
  const ChunkInfo ci = chunks[c];
  const uint8_t* src = wire + chunk_offsets[c];
  const uint32_t nnz = (uint32_t)src[0] | ((uint32_t)src[1] << 8) | ((uint32_t)src[2] << 16) | ((uint32_t)src[3] << 24);
  uint32_t* seg = reinterpret_cast<uint32_t*>(message + ci.seg_off);
  const uint64_t bmb = (ci.slots + 7) / 8;
  const uint8_t* bsrc = src + 4;
  const uint32_t bm_words = (ci.slots + 31) / 32;
  uint32_t pc = 0;
  for (uint32_t w = threadIdx.x; w < bm_words; w += blockDim.x) {
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) v |= (uint32_t)wire_byte(bsrc, 4ull * w + k, bmb) << (8 * k);
    // keep only bits of real slots (the reference ignores pad bits)
    uint32_t so = ballot_to_wire(v);
    const uint32_t first = w * 32;
    if (first + 32 > ci.slots) so &= (ci.slots - first >= 32) ? ~0u : ((1u << (ci.slots - first)) - 1u);
    pc += __popc(so);
    seg[kSegHeader / 4 + w] = ballot_to_wire(so);
  }
  const uint32_t total = block_sum<kWireThreads>(pc, scan);
  const uint64_t nbits = (uint64_t)nnz * N;
  const uint64_t cbytes = (nbits + 7) / 8;
  const uint8_t* csrc = bsrc + bmb;
  uint32_t* cw = reinterpret_cast<uint32_t*>(message + ci.seg_off + ci.code_off);
  const uint64_t words = (nbits + 31) / 32;
  const uint64_t lim = words < ci.code_cap ? words : ci.code_cap;
  for (uint64_t w = threadIdx.x; w < lim; w += blockDim.x) {
    uint32_t v = 0;
    for (int k = 0; k < 4; ++k) v |= (uint32_t)wire_byte(csrc, 4ull * w + k, cbytes) << (8 * k);
    const uint64_t first = w * 32;
    if (first + 32 > nbits) v &= (1u << (uint32_t)(nbits - first)) - 1u;
    cw[w] = v;
  }
  if (threadIdx.x == 0) {
    seg[0] = nnz;
    seg[1] = seg[2] = seg[3] = 0;
    popcounts[c] = (words > ci.code_cap) ? 0xFFFFFFFFu : total;
  }
}

__global__ void k_message_counts(const ChunkInfo* chunks, uint32_t n, const uint8_t* message, uint32_t* nnz) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  nnz[c] = *reinterpret_cast<const uint32_t*>(message + chunks[c].seg_off);
}

__global__ void k_message_unpack(const ChunkInfo* chunks, const uint8_t* message, int N, const uint64_t* code_offsets,
                                 uint8_t* flags01, uint32_t* codes) {
  const uint32_t c = blockIdx.x;
  const ChunkInfo ci = chunks[c];
  const uint8_t* seg = message + ci.seg_off;
  const uint32_t* bm = reinterpret_cast<const uint32_t*>(seg + kSegHeader);
  const uint32_t* cw = reinterpret_cast<const uint32_t*>(seg + ci.code_off);
  const uint32_t nnz = *reinterpret_cast<const uint32_t*>(seg);
  FGC_CHECK(nnz <= ci.slots && (uint64_t)nnz * N <= 32ull * ci.code_cap);
  for (uint32_t s = threadIdx.x; s < ci.slots; s += blockDim.x) {
    const uint32_t so = ballot_to_wire(bm[s >> 5]);
    flags01[ci.slot_off + s] = (so >> (s & 31)) & 1u;
  }
  uint32_t* out = codes + code_offsets[c];
  for (uint32_t j = threadIdx.x; j < nnz; j += blockDim.x) out[j] = read_bits(cw, (uint64_t)j * N, N);
}

__global__ void k_message_pack(const ChunkInfo* chunks, const uint8_t* flags01, const uint32_t* codes,
                               const uint64_t* code_offsets, int N, uint8_t* message, uint32_t* popcounts,
                               uint32_t* flags) {
  __shared__ uint32_t scan[40];
  const uint32_t c = blockIdx.x;
  const ChunkInfo ci = chunks[c];
  uint32_t* seg = reinterpret_cast<uint32_t*>(message + ci.seg_off);
  const uint32_t bm_words = (ci.slots + 31) / 32;
  uint32_t pc = 0;
  for (uint32_t w = threadIdx.x; w < bm_words; w += blockDim.x) {
    uint32_t so = 0;
    for (uint32_t k = 0; k < 32; ++k) {
      const uint32_t s = w * 32 + k;
      if (s < ci.slots && flags01[ci.slot_off + s]) so |= 1u << k;
    }
    pc += __popc(so);
    seg[kSegHeader / 4 + w] = ballot_to_wire(so);
  }
  const uint32_t total = block_sum<kWireThreads>(pc, scan);
  const uint64_t first = code_offsets[c];
  const uint32_t nnz = (uint32_t)(code_offsets[c + 1] - first);
  const uint64_t nbits = (uint64_t)nnz * N;
  const uint64_t words = (nbits + 31) / 32;
  uint32_t* cw = reinterpret_cast<uint32_t*>(message + ci.seg_off + ci.code_off);
  const uint32_t mask = N == 32 ? ~0u : ((1u << N) - 1u);
  if (words > ci.code_cap) {
    if (threadIdx.x == 0) atomicOr(flags, FGC_FLAG_CAPACITY);
  } else {
    for (uint64_t w = threadIdx.x; w < words; w += blockDim.x) {
      const uint64_t b0 = w * 32, b1 = b0 + 32;
      uint32_t v = 0;
      for (uint64_t j = b0 / N; j < nnz && j * N < b1; ++j) {
        const uint64_t pos = j * N;
        const uint32_t code = codes[first + j] & mask;
        if (pos >= b0) v |= code << (uint32_t)(pos - b0);
        else v |= code >> (uint32_t)(b0 - pos);
      }
      cw[w] = v;
    }
  }
  if (threadIdx.x == 0) {
    seg[0] = nnz;
    seg[1] = seg[2] = seg[3] = 0;
    popcounts[c] = total;
  }
}

inline uint32_t cdiv(uint64_t a, uint32_t b) { return (uint32_t)((a + b - 1) / b); }

}  // namespace

fgc_status launch_serialize(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message, int n_bits,
                            const uint8_t header[FGC_HEADER_BYTES], uint8_t* wire, uint64_t* wire_len,
                            uint64_t* scratch, cudaStream_t s) {
  Header36 h;
  for (int i = 0; i < FGC_HEADER_BYTES; ++i) h.b[i] = header[i];
  k_wire_sizes<<<cdiv(n_chunks, 256), 256, 0, s>>>(d_chunks, n_chunks, message, n_bits, scratch);
  FGC_LAUNCHED(1);
  k_scan_u64<<<1, 1024, 0, s>>>(scratch, n_chunks, wire_len, FGC_HEADER_BYTES);
  FGC_LAUNCHED(1);
  k_wire_copy<<<n_chunks, kWireThreads, 0, s>>>(d_chunks, message, n_bits, scratch, h, wire);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_scan_u64(uint64_t* v, uint32_t n, uint64_t* total, uint64_t add, cudaStream_t s) {
  k_scan_u64<<<1, 1024, 0, s>>>(v, n, total, add);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_deserialize(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* wire,
                              const uint64_t* chunk_offsets, int n_bits, uint8_t* message, uint32_t* popcounts,
                              cudaStream_t s) {
  k_unwire<<<n_chunks, kWireThreads, 0, s>>>(d_chunks, wire, chunk_offsets, n_bits, message, popcounts);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_message_counts(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message,
                                 uint32_t* nnz, cudaStream_t s) {
  k_message_counts<<<cdiv(n_chunks, 256), 256, 0, s>>>(d_chunks, n_chunks, message, nnz);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_message_unpack(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* message, int n_bits,
                                 const uint64_t* code_offsets, uint8_t* flags01, uint32_t* codes, cudaStream_t s) {
  k_message_unpack<<<n_chunks, kWireThreads, 0, s>>>(d_chunks, message, n_bits, code_offsets, flags01, codes);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

fgc_status launch_message_pack(const ChunkInfo* d_chunks, uint32_t n_chunks, const uint8_t* flags01,
                               const uint32_t* codes, const uint64_t* code_offsets, int n_bits, uint8_t* message,
                               uint32_t* popcounts, uint32_t* flags, cudaStream_t s) {
  k_message_pack<<<n_chunks, kWireThreads, 0, s>>>(d_chunks, flags01, codes, code_offsets, n_bits, message,
                                                   popcounts, flags);
  FGC_LAUNCHED(1);
  return FGC_OK;
}

}  // namespace fgc
