// Stable LSD radix sort of (uint32 key, int32 value) pairs on sm_100a.
// Used by the pushforward to bucket sources by target cell in source order
// (stability is what makes the later per-target fold reproduce the
// reference's sequential scatter order, pushforward.hpp:149-170).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace bfmgpu {

class RadixSorter {
 public:
  RadixSorter() = default;
  ~RadixSorter();
  RadixSorter(const RadixSorter&) = delete;
  RadixSorter& operator=(const RadixSorter&) = delete;
  void init(long n);
  // Sorts keys[0,n) (values = element index when vals_in == nullptr) by the
  // low `bits` key bits, stably. Result pointers valid until the next call.
  // d_n (optional): device-side element count <= n (n sizes the grids).
  void sort(const uint32_t* keys_in, const int* vals_in, long n, int bits, cudaStream_t s,
            LaunchCounter* lc, const uint32_t** keys_out, const int** vals_out, const int* d_n = nullptr);
  // Stable compaction of the pairs (keys_in[i], i) with keys_in[i] != sentinel
  // into the sorter's buffers; returns the device pointer of the kept count.
  const int* compact(const uint32_t* keys_in, long n, uint32_t sentinel, cudaStream_t s, LaunchCounter* lc,
                     const uint32_t** keys_out, const int** vals_out);
  // One-sweep form of compact + sort (+ pack): one histogram kernel over the
  // raw keys (all digit positions at once, sentinel keys skipped), then one
  // scatter kernel per digit whose tiles chain their digit offsets by
  // decoupled look-back; the first pass drops the sentinel keys. Returns the
  // device pointer of the number of sorted pairs.
  const int* sort_onesweep(const uint32_t* keys_in, long n, uint32_t sentinel, int bits, cudaStream_t s,
                           LaunchCounter* lc, const uint32_t** keys_out, const int** vals_out);

 private:
  long cap_ = 0;
  long blocks_ = 0;
  uint32_t* kbuf_[2] = {nullptr, nullptr};
  int* vbuf_[2] = {nullptr, nullptr};
  int* hist_ = nullptr;   // [256 * blocks]
  int* bsum_ = nullptr;   // scan scratch
  int* cnt_ = nullptr;    // [blocks + 2] compaction tile counts -> offsets, total at [blocks]
  unsigned* aux_ = nullptr;  // one-sweep: digit histograms, tile counters, count, look-back words
  long aux_words_ = 0;
};

}  // namespace bfmgpu
