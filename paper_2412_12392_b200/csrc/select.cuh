// Exact segmented upper-median (rank floor(n/2), std::nth_element semantics)
// of masked fp32 values: three radix passes (12 + 12 + 8 bits) over
// order-preserving keys.  Used for q_min = q_min_fraction * median of valid
// match confidences (tracking.cpp:32-42, backend.cpp:37-46).
#pragma once
#include "pmx_common.cuh"

namespace pmx {

struct SelSeg {
  const float* vals;     // n values
  const uint8_t* valid;  // nullable (all valid)
  int64_t n;
  double* out;           // median (0 when empty), written as double
  double scale;          // out = scale * median
};

// Launch-time scratch: per segment 4096+4096+256 counters + 4 state words.
void segmented_median(Context& ctx, const SelSeg* dev_segs, int nseg, int64_t max_n, DevBuf& scratch);

}  // namespace pmx
