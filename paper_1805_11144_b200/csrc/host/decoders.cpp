// decoders.cpp — the regularised least-squares decoder solve of the reference
// frontend (proj/src/frontend.cpp:56-76, there with Eigen's LLT) without Eigen:
//     (A^T A + m sigma^2 I) D = A^T Y,   sigma = reg * max|A|
// A [m][n] activities, Y [m][d] targets, D [n][d] decoders, all row-major.
// The normal matrix is factored by a right-looking Cholesky (L L^T) in double;
// a non-positive (or NaN) pivot is the singular case the reference reports
// as BuildError.
#include <cmath>
#include <string>
#include <vector>

#include "host_ir.hpp"

namespace nengb {

std::vector<double> solve_decoders(const double* A, int m, int n, const double* Y, int d, double reg) {
    if (m < 1 || n < 1 || d < 1) throw BuildError("solve_decoders: empty system");
    if (!(reg >= 0.0)) throw BuildError("solve_decoders: reg must be non-negative");
    double amax = 0.0;
    for (long long i = 0; i < static_cast<long long>(m) * n; ++i) amax = std::fmax(amax, std::fabs(A[i]));
    const double sigma = reg * amax;
    // G = A^T A + m sigma^2 I (lower triangle), R = A^T Y
    std::vector<double> G(static_cast<size_t>(n) * n, 0.0), R(static_cast<size_t>(n) * d, 0.0);
    for (int s = 0; s < m; ++s) {
        const double* a = A + static_cast<size_t>(s) * n;
        const double* y = Y + static_cast<size_t>(s) * d;
        for (int i = 0; i < n; ++i) {
            const double ai = a[i];
            if (ai == 0.0) continue;
            double* gi = G.data() + static_cast<size_t>(i) * n;
            for (int j = 0; j <= i; ++j) gi[j] += ai * a[j];
            double* ri = R.data() + static_cast<size_t>(i) * d;
            for (int k = 0; k < d; ++k) ri[k] += ai * y[k];
        }
    }
    for (int i = 0; i < n; ++i) G[static_cast<size_t>(i) * n + i] += static_cast<double>(m) * sigma * sigma;
    // in-place Cholesky: L in the lower triangle of G
    for (int j = 0; j < n; ++j) {
        double* gj = G.data() + static_cast<size_t>(j) * n;
        double diag = gj[j];
        for (int k = 0; k < j; ++k) diag -= gj[k] * gj[k];
        if (!(diag > 0.0)) throw BuildError("solve_decoders: singular normal equations (reg too small)");
        const double ljj = std::sqrt(diag);
        gj[j] = ljj;
        for (int i = j + 1; i < n; ++i) {
            double* gi = G.data() + static_cast<size_t>(i) * n;
            double v = gi[j];
            for (int k = 0; k < j; ++k) v -= gi[k] * gj[k];
            gi[j] = v / ljj;
        }
    }
    // L Z = R (forward), L^T D = Z (backward), column by column of the right-hand side
    std::vector<double> D(static_cast<size_t>(n) * d);
    std::vector<double> z(n);
    for (int c = 0; c < d; ++c) {
        for (int i = 0; i < n; ++i) {
            const double* gi = G.data() + static_cast<size_t>(i) * n;
            double v = R[static_cast<size_t>(i) * d + c];
            for (int k = 0; k < i; ++k) v -= gi[k] * z[k];
            z[i] = v / gi[i];
        }
        for (int i = n - 1; i >= 0; --i) {
            double v = z[i];
            for (int k = i + 1; k < n; ++k) v -= G[static_cast<size_t>(k) * n + i] * D[static_cast<size_t>(k) * d + c];
            D[static_cast<size_t>(i) * d + c] = v / G[static_cast<size_t>(i) * n + i];
        }
    }
    return D;
}

}  // namespace nengb
