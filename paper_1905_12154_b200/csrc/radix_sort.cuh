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
  void sort(const uint32_t* keys_in, const int* vals_in, long n, int bits, cudaStream_t s,
            LaunchCounter* lc, const uint32_t** keys_out, const int** vals_out);

 private:
  long cap_ = 0;
  long blocks_ = 0;
  uint32_t* kbuf_[2] = {nullptr, nullptr};
  int* vbuf_[2] = {nullptr, nullptr};
  int* hist_ = nullptr;   // [256 * blocks]
  int* bsum_ = nullptr;   // scan scratch
};

}  // namespace bfmgpu
