// host_consts.cpp -- host-side constants of the detector path.
//
// Compiled with -ffp-contract=off: the only fused operations are the explicit
// std::fma calls, placed exactly where GCC -O3 -march=x86-64-v3/native fuses
// the reference (objdump -l of detector.o: detector.cpp:105, :106, :112;
// DESIGN.md §5).  The weights are therefore bit-identical to the ones the
// reference's savgol_smooth uses (tests compare savgol outputs bit for bit).
#include "internal.h"

#include <cmath>
#include <utility>
#include <vector>

namespace ssb {

// Restates solve_e0 + savgol_weights (proj/src/detector.cpp:84-142):
// normal equations G x = e0 by partial-pivoting elimination, then the
// centre-sample weights c_j = sum_a x_a j^a.
bool savgol_weights_host(int window, int order, std::vector<double>& w) {
    if (window < 5 || window % 2 == 0 || order < 1 || order >= window) return false;
    const int h = (window - 1) / 2;
    const int n = order + 1;
    std::vector<double> g(static_cast<size_t>(n) * n, 0.0), x(static_cast<size_t>(n), 0.0);
    for (int a = 0; a < n; ++a)
        for (int b = 0; b < n; ++b) {
            double acc = 0.0;
            for (int j = -h; j <= h; ++j) acc += std::pow(static_cast<double>(j), static_cast<double>(a + b));
            g[static_cast<size_t>(a) * n + b] = acc;
        }
    x[0] = 1.0;
    for (int col = 0; col < n; ++col) {
        int piv = col;
        for (int r = col + 1; r < n; ++r)
            if (std::fabs(g[static_cast<size_t>(r) * n + col]) > std::fabs(g[static_cast<size_t>(piv) * n + col]))
                piv = r;
        if (piv != col) {
            for (int c = 0; c < n; ++c) std::swap(g[static_cast<size_t>(col) * n + c], g[static_cast<size_t>(piv) * n + c]);
            std::swap(x[static_cast<size_t>(col)], x[static_cast<size_t>(piv)]);
        }
        const double d = g[static_cast<size_t>(col) * n + col];
        if (d == 0.0) return false;
        for (int r = col + 1; r < n; ++r) {
            const double f = g[static_cast<size_t>(r) * n + col] / d;
            if (f == 0.0) continue;
            for (int c = col; c < n; ++c)
                g[static_cast<size_t>(r) * n + c] =
                    std::fma(-f, g[static_cast<size_t>(col) * n + c], g[static_cast<size_t>(r) * n + c]);
            x[static_cast<size_t>(r)] = std::fma(-f, x[static_cast<size_t>(col)], x[static_cast<size_t>(r)]);
        }
    }
    for (int r = n - 1; r >= 0; --r) {
        double acc = x[static_cast<size_t>(r)];
        for (int c = r + 1; c < n; ++c)
            acc = std::fma(-g[static_cast<size_t>(r) * n + c], x[static_cast<size_t>(c)], acc);
        x[static_cast<size_t>(r)] = acc / g[static_cast<size_t>(r) * n + r];
    }
    w.assign(static_cast<size_t>(window), 0.0);
    for (int j = -h; j <= h; ++j) {
        double c = 0.0, jp = 1.0;
        for (int a = 0; a < n; ++a) {
            c = c + x[static_cast<size_t>(a)] * jp;
            jp = jp * j;
        }
        w[static_cast<size_t>(j + h)] = c;
    }
    return true;
}

// glibc's x86_64 ifunc resolver picks the FMA builds of logf/powf when FMA
// and AVX2 are usable; the device floor stage mirrors whichever one the host
// libm (and hence the reference) runs.
bool host_has_fma_avx2() {
#if defined(__x86_64__)
    __builtin_cpu_init();
    return __builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2");
#else
    return true;
#endif
}

} // namespace ssb
