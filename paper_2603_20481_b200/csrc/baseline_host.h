// baseline_host.h -- host half of the baseline detector (csrc/baseline_host.cpp).
#pragma once

#include <cstdint>
#include <vector>

namespace ssb {

struct BaselineRect {
    int t0, t1, f0, f1;  // half-open bins
};

// Greedy seed walk over the kernel sizes in order (cells row-major), box
// growth on the SAT, then merge overlapping boxes and sort by (t0, f0, t1, f1)
// (proj/src/baseline.cpp:126-167).  sat: (rows+1) x (cols+1) doubles; cand:
// n_sizes x rows x ceil(cols/32) words; sizes: n_sizes (kr, kc) pairs.
std::vector<BaselineRect> baseline_greedy(const double* sat, const uint32_t* cand, const int* sizes, int n_sizes,
                                          int rows, int cols, double rate);

} // namespace ssb
