// baseline_host.cpp -- the sequential half of the baseline detector
// (proj/src/baseline.cpp:57-91 expand_box, :126-167 greedy walk and merge),
// fed by the device-built summed-area table and candidate bitmaps
// (csrc/baseline.cu).  Built with -ffp-contract=off; every mean is
// ((a - b) - c) + d over the SAT, divided by the cell count, as the reference.
#include "baseline_host.h"

#include <algorithm>
#include <tuple>

namespace ssb {
namespace {

struct Sat {
    const double* s;
    int rows, cols;
    long long w;
    double sum(int t0, int t1, int f0, int f1) const {
        return s[t1 * w + f1] - s[t0 * w + f1] - s[t1 * w + f0] + s[t0 * w + f0];
    }
    double mean(int t0, int t1, int f0, int f1) const {
        const long long n = static_cast<long long>(t1 - t0) * (f1 - f0);
        return sum(t0, t1, f0, f1) / static_cast<double>(n);
    }
};

// grow one bin per side while the newly exposed strip keeps rate x box mean
BaselineRect grow(BaselineRect b, const Sat& sat, double rate) {
    for (bool again = true; again;) {
        again = false;
        double m = sat.mean(b.t0, b.t1, b.f0, b.f1);
        if (b.t0 > 0 && sat.mean(b.t0 - 1, b.t0, b.f0, b.f1) >= rate * m) {
            --b.t0;
            again = true;
        }
        m = sat.mean(b.t0, b.t1, b.f0, b.f1);
        if (b.t1 < sat.rows && sat.mean(b.t1, b.t1 + 1, b.f0, b.f1) >= rate * m) {
            ++b.t1;
            again = true;
        }
        m = sat.mean(b.t0, b.t1, b.f0, b.f1);
        if (b.f0 > 0 && sat.mean(b.t0, b.t1, b.f0 - 1, b.f0) >= rate * m) {
            --b.f0;
            again = true;
        }
        m = sat.mean(b.t0, b.t1, b.f0, b.f1);
        if (b.f1 < sat.cols && sat.mean(b.t0, b.t1, b.f1, b.f1 + 1) >= rate * m) {
            ++b.f1;
            again = true;
        }
    }
    return b;
}

bool overlap(const BaselineRect& a, const BaselineRect& b) {
    return a.t0 < b.t1 && b.t0 < a.t1 && a.f0 < b.f1 && b.f0 < a.f1;
}

} // namespace

std::vector<BaselineRect> baseline_greedy(const double* sat, const uint32_t* cand, const int* sizes, int n_sizes,
                                          int rows, int cols, double rate) {
    const int W = (cols + 31) / 32;
    const Sat S{sat, rows, cols, cols + 1};
    // covered cells as a bitmap (row-major words): a candidate word is masked
    // with ~covered so covered cells are skipped 32 at a time
    std::vector<uint32_t> covered(static_cast<size_t>(rows) * W, 0u);
    std::vector<BaselineRect> boxes;
    for (int k = 0; k < n_sizes; ++k) {
        const int kr = sizes[2 * k], kc = sizes[2 * k + 1];
        const int rlo = (kr - 1) / 2, rhi = kr / 2, clo = (kc - 1) / 2, chi = kc / 2;
        const uint32_t* ck = cand + static_cast<size_t>(k) * rows * W;
        for (int t = 0; t < rows; ++t) {
            for (int wd = 0; wd < W; ++wd) {
                for (;;) {
                    // re-read: a box found in this word may cover the rest of it
                    const uint32_t live = ck[static_cast<size_t>(t) * W + wd] & ~covered[static_cast<size_t>(t) * W + wd];
                    if (!live) break;
                    const int f = wd * 32 + __builtin_ctz(live);
                    const BaselineRect seed{std::max(0, t - rlo), std::min(rows, t + rhi + 1), std::max(0, f - clo),
                                            std::min(cols, f + chi + 1)};
                    const BaselineRect b = grow(seed, S, rate);
                    boxes.push_back(b);
                    for (int bt = b.t0; bt < b.t1; ++bt) {
                        uint32_t* row = covered.data() + static_cast<size_t>(bt) * W;
                        for (int c = b.f0; c < b.f1;) {
                            const int w0 = c >> 5, lo = c & 31;
                            const int hi = std::min(32, lo + (b.f1 - c));
                            const uint32_t m = (hi == 32 ? ~0u : ((1u << hi) - 1u)) & ~((1u << lo) - 1u);
                            row[w0] |= m;
                            c += hi - lo;
                        }
                    }
                    // the seeding cell itself is always inside its grown box
                }
            }
        }
    }
    // fold overlapping boxes into their bounding rectangle until disjoint:
    // always the first overlapping pair (i, j) in index order
    for (bool merged = true; merged;) {
        merged = false;
        for (size_t i = 0; i < boxes.size() && !merged; ++i) {
            for (size_t j = i + 1; j < boxes.size(); ++j) {
                if (!overlap(boxes[i], boxes[j])) continue;
                BaselineRect& a = boxes[i];
                const BaselineRect& b = boxes[j];
                a = {std::min(a.t0, b.t0), std::max(a.t1, b.t1), std::min(a.f0, b.f0), std::max(a.f1, b.f1)};
                boxes.erase(boxes.begin() + static_cast<std::ptrdiff_t>(j));
                merged = true;
                break;
            }
        }
    }
    std::sort(boxes.begin(), boxes.end(), [](const BaselineRect& a, const BaselineRect& b) {
        return std::tie(a.t0, a.f0, a.t1, a.f1) < std::tie(b.t0, b.f0, b.t1, b.f1);
    });
    return boxes;
}

} // namespace ssb
