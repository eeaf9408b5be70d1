// Plain structs shared by host plan code and device kernels.
#pragma once
#include <stdint.h>

namespace fgc {

// Lattice parameters in the form the kernels consume (quantizer.py:71-151).
struct QuantParams {
  int32_t  n_bits;     // 2..16, or 32 = passthrough (raw f32 bits)
  int32_t  shift;      // 23 - mantissa_bits
  uint32_t pbase;      // bits(eps) >> shift
  uint32_t npos;       // P
  uint32_t nneg;       // Q = 2^N - 1 - P
  float    eps;        // f32(eps)
  float    pos_cap;    // f32(max)
  float    neg_cap;    // f32(-actual_min)
};

// One chunk of the gradient and its device-message segment.
struct ChunkInfo {
  uint64_t in_off;     // first gradient element
  uint64_t seg_off;    // byte offset of the segment in the device message
  uint64_t bin_off;    // first bin in a chunk-major spectrum
  uint64_t slot_off;   // first slot in chunk-major slot arrays
  uint32_t len;        // L
  uint32_t bins;       // L//2 + 1
  uint32_t slots;      // 2 * bins
  uint32_t drop;       // count mode: ceil(theta * bins)  (spectral.py:131)
  uint32_t code_off;   // byte offset of the code words inside the segment
  uint32_t code_cap;   // capacity of the code region in 32-bit words
  uint32_t cls;        // length class index
  uint32_t idx_in_cls; // position within the class batch
};

// Segment layout constants.
constexpr uint32_t kSegHeader = 16;   // u32 nnz + 12 zero bytes; bitmap follows

}  // namespace fgc
