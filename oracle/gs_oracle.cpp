// ============================================================================
// gs_oracle.cpp -- CPU restatement of the reference hot path.  TEST
// INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py, never by the product.
//
// Restates, function by function, the reference C++ (paths relative to
// /root/reference/proj):
//   fourier.cpp:16-49     transfer_function, haar_fourier, fourier_scaling
//   fourier.cpp:60-120    boundary_fourier_at_zero, fourier_boundary
//   scaling.cpp:42-75     boundary_filters (U = H/sqrt2, V = h/sqrt2)
//   nufft.cpp:74-132      ndft_forward / ndft_adjoint (direct)
//   nufft.cpp:160-365     Kaiser-Bessel NfftPlan (plan, forward, adjoint)
//   nufft.cpp:383-459     uniform_ndft_fft / uniform_ndft_adjoint_fft
//   freq2wave.cpp:15-193  wrap_half_open, detect_uniform, build_axis, freq2wave
//   freq2wave.cpp:215-387 apply_forward / apply_adjoint (1D and 9-block 2D)
//   freq2wave.cpp:389-450 densify
//   solver.cpp:19-91      solve_least_squares (CGNR)
//   patterns.cpp:14-74    gen_grid / gen_jitter / gen_spiral
//   weights.cpp:99-226    voronoi_weights (1D midpoints, 2D half-plane clipping)
//   dyadic.cpp:14-231     integer values, dyadic cascades (interior + edge),
//                         weval_1d / weval_2d (front-end row SURVEY 8(f)4)
// Third-party stand-ins: FFTW (unnormalised c2c, FORWARD = -1) is replaced by
// our own table-twiddle FFT (radix-2; mixed-radix Cooley-Tukey for other
// lengths); Eigen by plain loops.  Results agree with the reference to roundoff.
//
// Parity pinning: tests/test_oracle_known_answers.py checks this file against
// every known-answer relation the reference's own tests hold for this path
// (test_fourier.cpp, test_scaling.cpp, test_nufft.cpp, test_freq2wave.cpp,
// test_solver.cpp, test_patterns.cpp) and against the 60-digit edge-moment
// fixtures (tests/family_fixtures.hpp) for the zero-frequency edge transforms.
// ============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numbers>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

#include "../paper_1607_04091_b200/csrc/family_data.h"

namespace orc {

using cd = std::complex<double>;
using cvec = std::vector<cd>;
constexpr double kTwoPi = 2.0 * std::numbers::pi;
constexpr double kPi = std::numbers::pi;

// error classes, error.hpp:9-41
struct Err : std::runtime_error {
    int code;
    Err(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void shape(const std::string& m) { throw Err(4, m); }
[[noreturn]] void domain(const std::string& m) { throw Err(5, m); }
[[noreturn]] void numerical(const std::string& m) { throw Err(6, m); }

// ---------------------------------------------------------------- families
struct Family {
    int p = 1;
    std::vector<double> taps;  // k = -p+1..p
};
Family make_family(int p) {  // scaling.cpp:29-38
    if (p < 1 || p > 8) domain("unsupported family");
    const gsdata::FamilyData& f = gsdata::kFamilies[p - 1];
    Family fam;
    fam.p = p;
    fam.taps.assign(f.taps, f.taps + 2 * p);
    return fam;
}

struct Boundary {  // scaling.cpp:42-75 + fourier.cpp:74-83
    int p = 0;
    bool left = true;
    std::vector<double> U, V;  // p x p, p x (2p-1), row-major
    std::vector<cd> v_zero;
};

std::vector<double> lu_solve(std::vector<double> A, std::vector<double> b, int n) {
    // partial-pivot LU (Eigen::PartialPivLU, fourier.cpp:64-67)
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int best = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(A[i * n + k]) > std::abs(A[best * n + k])) best = i;
        if (best != k) {
            for (int j = 0; j < n; ++j) std::swap(A[k * n + j], A[best * n + j]);
            std::swap(b[k], b[best]);
        }
        double d = A[k * n + k];
        if (d == 0.0) break;
        for (int i = k + 1; i < n; ++i) {
            double f = A[i * n + k] / d;
            A[i * n + k] = f;
            for (int j = k + 1; j < n; ++j) A[i * n + j] -= f * A[k * n + j];
            b[i] -= f * b[k];
        }
    }
    std::vector<double> x(n);
    for (int i = n - 1; i >= 0; --i) {
        double s = b[i];
        for (int j = i + 1; j < n; ++j) s -= A[i * n + j] * x[j];
        x[i] = s / A[i * n + i];
    }
    return x;
}

Boundary make_boundary(const Family& fam, bool left) {
    if (fam.p == 1) domain("haar has no boundary corrections (p = 1)");
    int p = fam.p;
    const gsdata::FamilyData& f = gsdata::kFamilies[p - 1];
    const double* H = left ? f.left_H : f.right_H;
    const double* h = left ? f.left_h : f.right_h;
    Boundary b;
    b.p = p;
    b.left = left;
    b.U.resize(p * p);
    b.V.resize(p * (2 * p - 1));
    for (int i = 0; i < p * p; ++i) b.U[i] = H[i] / std::sqrt(2.0);
    for (int i = 0; i < p * (2 * p - 1); ++i) b.V[i] = h[i] / std::sqrt(2.0);
    // fixed point (I - U) v = V 1   (fourier.cpp:60-72)
    std::vector<double> lhs(p * p), rhs(p, 0.0);
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j) lhs[i * p + j] = (i == j ? 1.0 : 0.0) - b.U[i * p + j];
    for (int i = 0; i < p; ++i)
        for (int j = 0; j < 2 * p - 1; ++j) rhs[i] += b.V[i * (2 * p - 1) + j];
    std::vector<double> v = lu_solve(lhs, rhs, p);
    double res = 0.0, rn = 0.0;
    for (int i = 0; i < p; ++i) {
        double s = -rhs[i];
        for (int j = 0; j < p; ++j) s += lhs[i * p + j] * v[j];
        res += s * s;
        rn += rhs[i] * rhs[i];
    }
    if (!(std::sqrt(res) <= 1e-10 * (1.0 + std::sqrt(rn))))
        numerical("boundary_fourier_at_zero: singular fixed-point system");
    b.v_zero.assign(v.begin(), v.end());
    return b;
}

// ---------------------------------------------------------------- fourier.cpp
cd transfer_function(const Family& fam, double xi) {  // fourier.cpp:16-24
    cd acc = 0.0;
    int k = -fam.p + 1;
    for (double tap : fam.taps) {
        acc += tap * std::polar(1.0, -kTwoPi * k * xi);
        ++k;
    }
    return acc;
}

cd haar_fourier(double xi) {  // fourier.cpp:26-30
    if (xi == 0.0) return 1.0;
    cd numerator = 1.0 - std::polar(1.0, -kTwoPi * xi);
    return numerator / cd(0.0, kTwoPi * xi);
}

cd fourier_scaling(const Family& fam, double xi, int terms = 48) {  // fourier.cpp:34-49
    if (fam.p == 1) return haar_fourier(xi);
    if (terms < 1) domain("fourier_scaling: terms must be >= 1");
    cd product = 1.0;
    double arg = xi;
    for (int j = 1; j <= terms; ++j) {
        arg *= 0.5;
        cd factor = transfer_function(fam, arg);
        product *= factor;
        if (std::abs(factor - 1.0) < 1e-16) break;
    }
    return product;
}

std::vector<cd> fourier_boundary(const Family& fam, const Boundary& ctx, double xi,
                                 int depth = 30, int terms = 48) {  // fourier.cpp:85-120
    if (depth < 1) domain("fourier_boundary: depth must be >= 1");
    int p = fam.p;
    std::vector<cd> phihat(depth + 1);
    phihat[depth] = fourier_scaling(fam, std::ldexp(xi, -depth), terms);
    for (int l = depth - 1; l >= 1; --l)
        phihat[l] = transfer_function(fam, std::ldexp(xi, -(l + 1))) * phihat[l + 1];
    std::vector<cd> acc = ctx.v_zero, v2(2 * p - 1), nxt(p);
    for (int l = depth - 1; l >= 0; --l) {
        double arg = std::ldexp(xi, -(l + 1));
        cd step = ctx.left ? std::polar(1.0, -kTwoPi * arg) : std::polar(1.0, kTwoPi * arg);
        cd phase = ctx.left ? std::polar(1.0, -kTwoPi * arg * p)
                            : std::polar(1.0, kTwoPi * arg * (p + 1));
        cd amp = phihat[l + 1];
        for (int m = 0; m < 2 * p - 1; ++m) {
            v2[m] = amp * phase;
            phase *= step;
        }
        for (int i = 0; i < p; ++i) {  // acc = U acc + V v2
            cd s = 0.0, t = 0.0;
            for (int j = 0; j < p; ++j) s += ctx.U[i * p + j] * acc[j];
            for (int j = 0; j < 2 * p - 1; ++j) t += ctx.V[i * (2 * p - 1) + j] * v2[j];
            nxt[i] = s + t;
        }
        acc = nxt;
    }
    return acc;
}

// ---------------------------------------------------------------- FFT (FFTW stand-in)
// Unnormalised c2c transform, sign -1 = FFTW_FORWARD, +1 = FFTW_BACKWARD.
// Twiddles come from a per-(length, sign) table (polar once per entry, as a
// planned FFTW does), so the CPU timing is not inflated by sincos per
// butterfly.  Powers of two: iterative radix-2; other lengths: recursive
// mixed-radix Cooley-Tukey over the smallest prime factor (direct DFT for a
// prime length), the same O(n log n) class FFTW's planner reaches.
const cvec& twiddle_table(int n, int sign) {
    thread_local std::vector<std::pair<long long, cvec>> cache;
    const long long key = 2LL * n + (sign > 0);
    for (auto& e : cache)
        if (e.first == key) return e.second;
    cvec t(n);
    for (int k = 0; k < n; ++k) t[k] = std::polar(1.0, sign * kTwoPi * static_cast<double>(k) / n);
    cache.emplace_back(key, std::move(t));
    return cache.back().second;
}

void fft_mixed(const cd* in, size_t stride, cd* out, int n, const cd* tw, int twstep, cd* tmp) {
    if (n == 1) {
        out[0] = in[0];
        return;
    }
    int p = n;
    for (int f = 2; f * f <= n; ++f)
        if (n % f == 0) {
            p = f;
            break;
        }
    const int m = n / p;
    for (int r = 0; r < p; ++r) fft_mixed(in + r * stride, stride * p, out + r * m, m, tw, twstep * p, tmp);
    // X[k + q m] = sum_r w_n^{r (k + q m)} Y_r[k], w_n^j = tw[j * twstep]
    for (int k = 0; k < m; ++k) {
        for (int q = 0; q < p; ++q) {
            const int kk = k + q * m;
            cd acc = out[k];
            for (int r = 1; r < p; ++r)
                acc += out[r * m + k] * tw[(static_cast<long long>(r) * kk % n) * twstep];
            tmp[kk] = acc;
        }
    }
    for (int j = 0; j < n; ++j) out[j] = tmp[j];
}

void fft_inplace(cd* a, int n, int sign) {
    if (n <= 1) return;
    const cvec& tw = twiddle_table(n, sign);
    if ((n & (n - 1)) != 0) {
        cvec in(a, a + n), tmp(n);
        fft_mixed(in.data(), 1, a, n, tw.data(), 1, tmp.data());
        return;
    }
    for (int i = 1, j = 0; i < n; ++i) {
        int bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (int len = 2; len <= n; len <<= 1) {
        const int half = len / 2, stride = n / len;
        for (int i = 0; i < n; i += len) {
            for (int k = 0; k < half; ++k) {
                cd u = a[i + k], v = a[i + k + half] * tw[static_cast<size_t>(k) * stride];
                a[i + k] = u + v;
                a[i + k + half] = u - v;
            }
        }
    }
}

void fft2_inplace(cd* a, int n0, int n1, int sign) {  // row-major, last axis fastest
    for (int r = 0; r < n0; ++r) fft_inplace(a + static_cast<size_t>(r) * n1, n1, sign);
    cvec col(n0);
    for (int c = 0; c < n1; ++c) {
        for (int r = 0; r < n0; ++r) col[r] = a[static_cast<size_t>(r) * n1 + c];
        fft_inplace(col.data(), n0, sign);
        for (int r = 0; r < n0; ++r) a[static_cast<size_t>(r) * n1 + c] = col[r];
    }
}

// ---------------------------------------------------------------- nufft.cpp
void check_points(int dim, const std::vector<double>& pts) {  // nufft.cpp:57-66
    for (double v : pts)
        if (!(v >= -0.5 && v < 0.5)) domain("scaled point outside [-1/2, 1/2)");
    if (pts.empty() || pts.size() % dim != 0) shape("point array size is not a multiple of dim");
}

cvec ndft_forward(int dim, const int N[2], const std::vector<double>& pts, const cvec& grid) {
    check_points(dim, pts);  // nufft.cpp:74-104
    size_t len = static_cast<size_t>(N[0]) * (dim == 2 ? N[1] : 1);
    if (grid.size() != len) shape("grid size mismatch");
    size_t M = pts.size() / dim;
    cvec out(M);
    for (size_t m = 0; m < M; ++m) {
        cd acc = 0.0;
        if (dim == 1) {
            for (int k = -N[0] / 2; k < N[0] / 2; ++k)
                acc += grid[k + N[0] / 2] * std::polar(1.0, -kTwoPi * k * pts[m]);
        } else {
            size_t idx = 0;
            for (int k0 = -N[0] / 2; k0 < N[0] / 2; ++k0) {
                cd ph0 = std::polar(1.0, -kTwoPi * k0 * pts[2 * m]);
                for (int k1 = -N[1] / 2; k1 < N[1] / 2; ++k1, ++idx)
                    acc += grid[idx] * ph0 * std::polar(1.0, -kTwoPi * k1 * pts[2 * m + 1]);
            }
        }
        out[m] = acc;
    }
    return out;
}

cvec ndft_adjoint(int dim, const int N[2], const std::vector<double>& pts, const cvec& y) {
    check_points(dim, pts);  // nufft.cpp:106-132
    size_t M = pts.size() / dim;
    if (y.size() != M) shape("sample count mismatch");
    cvec out(static_cast<size_t>(N[0]) * (dim == 2 ? N[1] : 1), cd(0.0));
    for (size_t m = 0; m < M; ++m) {
        if (dim == 1) {
            for (int k = -N[0] / 2; k < N[0] / 2; ++k)
                out[k + N[0] / 2] += y[m] * std::polar(1.0, kTwoPi * k * pts[m]);
        } else {
            size_t idx = 0;
            for (int k0 = -N[0] / 2; k0 < N[0] / 2; ++k0) {
                cd ph0 = y[m] * std::polar(1.0, kTwoPi * k0 * pts[2 * m]);
                for (int k1 = -N[1] / 2; k1 < N[1] / 2; ++k1, ++idx)
                    out[idx] += ph0 * std::polar(1.0, kTwoPi * k1 * pts[2 * m + 1]);
            }
        }
    }
    return out;
}

double kb_transform(double nu, int w, double beta) {  // nufft.cpp:163-171
    double t = beta * beta - (kTwoPi * w * nu) * (kTwoPi * w * nu);
    if (t > 0) {
        double s = std::sqrt(t);
        return 2.0 * w * std::sinh(s) / s;
    }
    double s = std::sqrt(-t);
    return 2.0 * w * std::sin(s) / s;
}

double kb_kernel(double u, int w, double beta) {  // nufft.cpp:173-177
    double t = 1.0 - (u / w) * (u / w);
    if (t < 0) return 0.0;
    return std::cyl_bessel_i(0.0, beta * std::sqrt(t));
}

double kb_beta(int w, double sigma) {  // nufft.cpp:201-206
    double width = 2.0 * w;
    double t = (width / sigma) * (width / sigma) * (sigma - 0.5) * (sigma - 0.5) - 0.8;
    return std::numbers::pi * std::sqrt(std::max(t, 1.0));
}

struct NfftPlan {  // nufft.cpp:138-233
    int dim = 1;
    int N[2] = {0, 0}, n[2] = {0, 0};
    int w = 6;
    double beta = 0;
    size_t M = 0;
    std::vector<long long> base;
    std::vector<double> weights;
    std::vector<double> deconv[2];

    NfftPlan() = default;
    NfftPlan(int dim_, const int N_[2], const std::vector<double>& pts, double sigma, int w_) {
        if (dim_ != 1 && dim_ != 2) domain("dim must be 1 or 2");
        for (int d = 0; d < dim_; ++d)
            if (N_[d] <= 0 || N_[d] % 2 != 0) domain("transform length must be even");
        if (sigma < 1.25) domain("oversampling factor must be >= 1.25");
        if (w_ < 2) domain("kernel half-width must be >= 2");
        check_points(dim_, pts);
        dim = dim_;
        w = w_;
        M = pts.size() / dim;
        for (int d = 0; d < dim; ++d) {
            N[d] = N_[d];
            n[d] = static_cast<int>(std::ceil(sigma * N[d] / 2.0)) * 2;
        }
        beta = kb_beta(w, sigma);
        int S = 2 * w + 1;
        base.resize(M * dim);
        weights.resize(M * dim * S);
        for (size_t m = 0; m < M; ++m)
            for (int d = 0; d < dim; ++d) {
                double pos = pts[m * dim + d] * n[d];
                long long j0 = std::llround(pos);
                base[m * dim + d] = j0 - w;
                double* wr = &weights[(m * dim + d) * S];
                for (int t = 0; t < S; ++t)
                    wr[t] = kb_kernel(pos - static_cast<double>(j0 - w + t), w, beta);
            }
        for (int d = 0; d < dim; ++d) {
            deconv[d].resize(N[d]);
            for (int k = -N[d] / 2; k < N[d] / 2; ++k)
                deconv[d][k + N[d] / 2] = 1.0 / kb_transform(static_cast<double>(k) / n[d], w, beta);
        }
    }
    size_t grid_size() const { return static_cast<size_t>(N[0]) * (dim == 2 ? N[1] : 1); }
    size_t over_len() const { return static_cast<size_t>(n[0]) * (dim == 2 ? n[1] : 1); }

    cvec forward(const cvec& grid) const {  // nufft.cpp:244-306
        if (grid.size() != grid_size()) shape("grid size mismatch");
        cvec pad(over_len(), cd(0.0));
        if (dim == 1) {
            for (int k = -N[0] / 2; k < N[0] / 2; ++k)
                pad[(k + n[0]) % n[0]] = grid[k + N[0] / 2] * deconv[0][k + N[0] / 2];
            fft_inplace(pad.data(), n[0], -1);
        } else {
            size_t idx = 0;
            for (int k0 = -N[0] / 2; k0 < N[0] / 2; ++k0) {
                size_t row = static_cast<size_t>((k0 + n[0]) % n[0]) * n[1];
                double d0 = deconv[0][k0 + N[0] / 2];
                for (int k1 = -N[1] / 2; k1 < N[1] / 2; ++k1, ++idx)
                    pad[row + (k1 + n[1]) % n[1]] = grid[idx] * (d0 * deconv[1][k1 + N[1] / 2]);
            }
            fft2_inplace(pad.data(), n[0], n[1], -1);
        }
        int S = 2 * w + 1;
        cvec out(M);
        for (size_t m = 0; m < M; ++m) {
            if (dim == 1) {
                long long b = base[m];
                const double* wr = &weights[m * S];
                cd acc = 0.0;
                for (int t = 0; t < S; ++t) {
                    long long j = ((b + t) % n[0] + n[0]) % n[0];
                    acc += wr[t] * pad[j];
                }
                out[m] = acc;
            } else {
                long long b0 = base[2 * m], b1 = base[2 * m + 1];
                const double* w0 = &weights[(2 * m) * S];
                const double* w1 = &weights[(2 * m + 1) * S];
                cd acc = 0.0;
                for (int t0 = 0; t0 < S; ++t0) {
                    long long j0 = ((b0 + t0) % n[0] + n[0]) % n[0];
                    cd rowacc = 0.0;
                    const cd* row = &pad[j0 * n[1]];
                    for (int t1 = 0; t1 < S; ++t1) {
                        long long j1 = ((b1 + t1) % n[1] + n[1]) % n[1];
                        rowacc += w1[t1] * row[j1];
                    }
                    acc += w0[t0] * rowacc;
                }
                out[m] = acc;
            }
        }
        return out;
    }

    cvec adjoint(const cvec& y) const {  // nufft.cpp:308-365
        if (y.size() != M) shape("sample count mismatch");
        int S = 2 * w + 1;
        cvec spread(over_len(), cd(0.0));
        for (size_t m = 0; m < M; ++m) {
            if (dim == 1) {
                long long b = base[m];
                const double* wr = &weights[m * S];
                for (int t = 0; t < S; ++t) {
                    long long j = ((b + t) % n[0] + n[0]) % n[0];
                    spread[j] += wr[t] * y[m];
                }
            } else {
                long long b0 = base[2 * m], b1 = base[2 * m + 1];
                const double* w0 = &weights[(2 * m) * S];
                const double* w1 = &weights[(2 * m + 1) * S];
                for (int t0 = 0; t0 < S; ++t0) {
                    long long j0 = ((b0 + t0) % n[0] + n[0]) % n[0];
                    cd v0 = w0[t0] * y[m];
                    cd* row = &spread[j0 * n[1]];
                    for (int t1 = 0; t1 < S; ++t1) {
                        long long j1 = ((b1 + t1) % n[1] + n[1]) % n[1];
                        row[j1] += w1[t1] * v0;
                    }
                }
            }
        }
        cvec out(grid_size());
        if (dim == 1) {
            fft_inplace(spread.data(), n[0], +1);
            for (int k = -N[0] / 2; k < N[0] / 2; ++k)
                out[k + N[0] / 2] = spread[(k + n[0]) % n[0]] * deconv[0][k + N[0] / 2];
        } else {
            fft2_inplace(spread.data(), n[0], n[1], +1);
            size_t idx = 0;
            for (int k0 = -N[0] / 2; k0 < N[0] / 2; ++k0) {
                size_t row = static_cast<size_t>((k0 + n[0]) % n[0]) * n[1];
                double d0 = deconv[0][k0 + N[0] / 2];
                for (int k1 = -N[1] / 2; k1 < N[1] / 2; ++k1, ++idx)
                    out[idx] = spread[row + (k1 + n[1]) % n[1]] * (d0 * deconv[1][k1 + N[1] / 2]);
            }
        }
        return out;
    }
};

struct UniformSetup { long long inv_eps, q, n2; };
UniformSetup uniform_setup(long long M, double eps, long long N) {  // nufft.cpp:389-400
    if (eps <= 0.0) domain("epsilon must be positive");
    double inv = 1.0 / eps;
    long long inv_eps = std::llround(inv);
    if (inv_eps < 1 || std::abs(inv - static_cast<double>(inv_eps)) > 1e-9)
        domain("1/epsilon must be a positive integer");
    if (M < N) domain("uniform reduction requires M >= N");
    long long per = N * inv_eps;
    long long q = (M + per - 1) / per;
    return {inv_eps, q, q * per};
}

cvec uniform_ndft_fft(const cvec& x, long long M, double eps, long long N) {  // nufft.cpp:404-430
    long long n1 = static_cast<long long>(x.size());
    if (n1 > N) domain("signal length must not exceed N");
    UniformSetup s = uniform_setup(M, eps, N);
    cvec z(s.n2, cd(0.0));
    double phase_step = std::numbers::pi * eps * static_cast<double>(M) / static_cast<double>(N);
    for (long long l = 0; l < n1; ++l)
        z[s.q * l] = x[l] * std::polar(1.0, phase_step * static_cast<double>(l));
    fft_inplace(z.data(), static_cast<int>(s.n2), -1);
    cvec out(M);
    for (long long m = 0; m < M; ++m) {
        double xi = eps / static_cast<double>(N) * (static_cast<double>(m) - static_cast<double>(M) / 2.0);
        out[m] = std::polar(1.0, std::numbers::pi * static_cast<double>(n1) * xi) * z[m];
    }
    return out;
}

cvec uniform_ndft_adjoint_fft(const cvec& y, double eps, long long N) {  // nufft.cpp:432-459
    long long M = static_cast<long long>(y.size());
    UniformSetup s = uniform_setup(M, eps, N);
    cvec pad(s.n2, cd(0.0));
    for (long long m = 0; m < M; ++m) {
        double xi = eps / static_cast<double>(N) * (static_cast<double>(m) - static_cast<double>(M) / 2.0);
        pad[m] = y[m] * std::polar(1.0, -std::numbers::pi * static_cast<double>(N) * xi);
    }
    fft_inplace(pad.data(), static_cast<int>(s.n2), +1);
    double phase_step = std::numbers::pi * eps * static_cast<double>(M) / static_cast<double>(N);
    cvec out(N);
    for (long long l = 0; l < N; ++l)
        out[l] = pad[s.q * l] * std::polar(1.0, -phase_step * static_cast<double>(l));
    return out;
}

// ---------------------------------------------------------------- freq2wave.cpp
double wrap_half_open(double z) {  // freq2wave.cpp:15-19
    double w = z - std::floor(z + 0.5);
    if (w >= 0.5) w -= 1.0;
    return w;
}

bool detect_uniform(const std::vector<double>& zeta, long long n, double* eps_out) {
    size_t M = zeta.size();  // freq2wave.cpp:22-37
    if (M < 2 || static_cast<long long>(M) < n) return false;
    double spacing = zeta[1] - zeta[0];
    if (spacing <= 0.0) return false;
    double eps = spacing * static_cast<double>(n);
    double inv = 1.0 / eps;
    if (std::abs(inv - std::round(inv)) > 1e-9 || std::round(inv) < 1.0) return false;
    double half_m = static_cast<double>(M) / 2.0;
    for (size_t m = 0; m < M; ++m) {
        double expect = eps / static_cast<double>(n) * (static_cast<double>(m) - half_m);
        if (std::abs(zeta[m] - expect) > 1e-12) return false;
    }
    *eps_out = eps;
    return true;
}

struct Op {  // Freq2WaveOp, freq2wave.hpp:32-55
    int dim = 1;
    Family fam;
    int J = 0;
    long long n = 0;
    std::vector<double> coords;
    std::vector<double> sqrt_weights;
    std::vector<double> zeta_x, zeta_y;
    cvec Dx, Dy;
    cvec Lx, Rx, Ly, Ry;  // M x p, column-major (m + c*M)
    NfftPlan plan_x, plan_y, plan_2d;
    bool has_x = false, has_y = false, has_2d = false;
    bool uniform_fast = false;
    double uniform_epsilon = 0.0;
    int depth = 30, terms = 48;
    size_t rows() const { return coords.size() / dim; }
    size_t cols() const { return dim == 1 ? n : n * n; }
    bool weighted() const { return !sqrt_weights.empty(); }
};

void build_axis(const Family& fam, int J, const std::vector<double>& xi, int depth, int terms,
                cvec& D, cvec& L, cvec& R) {  // freq2wave.cpp:45-76
    size_t M = xi.size();
    D.resize(M);
    double amp = std::exp2(-0.5 * J);
    for (size_t m = 0; m < M; ++m) D[m] = amp * fourier_scaling(fam, std::ldexp(xi[m], -J), terms);
    if (fam.p >= 2) {
        int p = fam.p;
        L.assign(M * p, 0.0);
        R.assign(M * p, 0.0);
        Boundary left = make_boundary(fam, true), right = make_boundary(fam, false);
        for (size_t m = 0; m < M; ++m) {
            double scaled = std::ldexp(xi[m], -J);
            std::vector<cd> vl = fourier_boundary(fam, left, scaled, depth, terms);
            std::vector<cd> vr = fourier_boundary(fam, right, scaled, depth, terms);
            cd pl = amp * std::polar(1.0, kPi * xi[m]);
            cd pr = amp * std::polar(1.0, -kPi * xi[m]);
            for (int c = 0; c < p; ++c) {
                L[m + c * M] = pl * vl[c];
                R[m + c * M] = pr * vr[p - 1 - c];
            }
        }
    }
}

Op* freq2wave(int dim, int p, int J, const std::vector<double>& coords, const std::vector<double>& weights,
              bool has_bw, double bw, double sigma, int w, int depth, int terms, bool allow_uniform) {
    Op* op = new Op;  // freq2wave.cpp:86-193
    try {
        op->fam = make_family(p);
        op->dim = dim;
        op->J = J;
        op->coords = coords;
        op->depth = depth;
        op->terms = terms;
        if (dim != 1 && dim != 2) domain("sampling set must be 1D or 2D");
        if (coords.size() / dim == 0) shape("empty sampling set");
        if (J < 0 || J > 24) domain("scale J out of range");
        op->n = 1LL << J;
        if (op->n < 2 * op->fam.p) domain("scale too small: 2^J must be >= 2p");
        for (double v : coords)
            if (!std::isfinite(v)) domain("non-finite frequency");
        size_t M = coords.size() / dim;
        if (!weights.empty()) {
            if (weights.size() != M) shape("weight count does not match sample count");
            op->sqrt_weights.resize(M);
            for (size_t m = 0; m < M; ++m) {
                if (!(weights[m] > 0.0)) domain("weights must be positive");
                op->sqrt_weights[m] = std::sqrt(weights[m]);
            }
        }
        std::vector<double> xi_x(M), xi_y;
        for (size_t m = 0; m < M; ++m) xi_x[m] = coords[m * dim];
        if (dim == 2) {
            xi_y.resize(M);
            for (size_t m = 0; m < M; ++m) xi_y[m] = coords[m * 2 + 1];
        }
        auto check_axis = [&](const std::vector<double>& xi) {
            for (double v : xi) {
                if (has_bw) {
                    if (std::abs(v) > bw) domain("bandwidth exceeded: |xi| > bandwidth");
                } else {
                    double z = std::ldexp(v, -J);
                    if (!(z >= -0.5 && z < 0.5))
                        domain("bandwidth exceeded: scaled point outside [-1/2, 1/2) "
                               "(pass a bandwidth to allow periodized rows)");
                }
            }
        };
        check_axis(xi_x);
        if (dim == 2) check_axis(xi_y);
        op->zeta_x.resize(M);
        for (size_t m = 0; m < M; ++m) op->zeta_x[m] = std::ldexp(xi_x[m], -J);
        if (dim == 2) {
            op->zeta_y.resize(M);
            for (size_t m = 0; m < M; ++m) op->zeta_y[m] = std::ldexp(xi_y[m], -J);
        }
        build_axis(op->fam, J, xi_x, depth, terms, op->Dx, op->Lx, op->Rx);
        if (dim == 2) build_axis(op->fam, J, xi_y, depth, terms, op->Dy, op->Ly, op->Ry);
        if (op->weighted()) {  // freq2wave.cpp:159-168
            int pp = op->fam.p;
            for (size_t m = 0; m < M; ++m) {
                op->Dx[m] *= op->sqrt_weights[m];
                if (pp >= 2)
                    for (int c = 0; c < pp; ++c) {
                        op->Lx[m + c * M] *= op->sqrt_weights[m];
                        op->Rx[m + c * M] *= op->sqrt_weights[m];
                    }
            }
        }
        int nax[2] = {static_cast<int>(op->n), static_cast<int>(op->n)};
        auto wrapped = [](const std::vector<double>& z) {
            std::vector<double> o(z.size());
            for (size_t i = 0; i < z.size(); ++i) o[i] = wrap_half_open(z[i]);
            return o;
        };
        if (dim == 1) {
            if (allow_uniform && detect_uniform(op->zeta_x, op->n, &op->uniform_epsilon)) {
                op->uniform_fast = true;
            } else {
                op->plan_x = NfftPlan(1, nax, wrapped(op->zeta_x), sigma, w);
                op->has_x = true;
            }
        } else {
            std::vector<double> wx = wrapped(op->zeta_x), wy = wrapped(op->zeta_y);
            op->plan_x = NfftPlan(1, nax, wx, sigma, w);
            op->plan_y = NfftPlan(1, nax, wy, sigma, w);
            std::vector<double> pts(2 * M);
            for (size_t m = 0; m < M; ++m) {
                pts[2 * m] = wy[m];
                pts[2 * m + 1] = wx[m];
            }
            op->plan_2d = NfftPlan(2, nax, pts, sigma, w);
            op->has_x = op->has_y = op->has_2d = true;
        }
    } catch (...) {
        delete op;
        throw;
    }
    return op;
}

cvec internal_forward_1d(const Op& op, const cvec& padded) {  // freq2wave.cpp:198-204
    if (op.uniform_fast)
        return uniform_ndft_fft(padded, static_cast<long long>(op.rows()), op.uniform_epsilon, op.n);
    return op.plan_x.forward(padded);
}
cvec internal_adjoint_1d(const Op& op, const cvec& v) {  // freq2wave.cpp:206-211
    if (op.uniform_fast) return uniform_ndft_adjoint_fft(v, op.uniform_epsilon, op.n);
    return op.plan_x.adjoint(v);
}

cvec apply_forward(const Op& op, const cvec& x) {  // freq2wave.cpp:215-303
    if (x.size() != op.cols()) shape("coefficient vector length mismatch");
    size_t M = op.rows();
    size_t n = op.n;
    int p = op.fam.p;
    bool edged = p >= 2;
    cvec out(M, cd(0.0));
    if (op.dim == 1) {
        cvec padded(x);
        if (edged)
            for (int c = 0; c < p; ++c) padded[c] = padded[n - 1 - c] = 0.0;
        cvec internal = internal_forward_1d(op, padded);
        for (size_t m = 0; m < M; ++m) out[m] = op.Dx[m] * internal[m];
        if (edged)
            for (size_t m = 0; m < M; ++m) {
                cd acc = 0.0;
                for (int c = 0; c < p; ++c) acc += op.Lx[m + c * M] * x[c];
                for (int c = 0; c < p; ++c) acc += op.Rx[m + c * M] * x[n - p + c];
                out[m] += acc;
            }
        return out;
    }
    auto X = [&](size_t i, size_t j) { return x[j * n + i]; };  // column-major, i = x index
    {
        cvec padded(x);
        if (edged)
            for (size_t j = 0; j < n; ++j)
                for (size_t i = 0; i < n; ++i)
                    if (i < (size_t)p || i >= n - p || j < (size_t)p || j >= n - p) padded[j * n + i] = 0.0;
        cvec internal = op.plan_2d.forward(padded);
        for (size_t m = 0; m < M; ++m) out[m] += op.Dx[m] * op.Dy[m] * internal[m];
    }
    if (!edged) return out;
    size_t np = n - p;
    auto corner = [&](const cvec& Ax, size_t row0, const cvec& By, size_t col0) {
        for (size_t m = 0; m < M; ++m) {
            cd sum = 0.0;
            for (int j = 0; j < p; ++j) {
                cd t = 0.0;
                for (int i = 0; i < p; ++i) t += Ax[m + i * M] * X(row0 + i, col0 + j);
                sum += t * By[m + j * M];
            }
            out[m] += sum;
        }
    };
    corner(op.Lx, 0, op.Ly, 0);
    corner(op.Lx, 0, op.Ry, np);
    corner(op.Rx, np, op.Ly, 0);
    corner(op.Rx, np, op.Ry, np);
    cvec line(n);
    auto side_x_edge = [&](const cvec& Ax, size_t row0) {
        for (int c = 0; c < p; ++c) {
            std::fill(line.begin(), line.end(), cd(0.0));
            for (size_t j = p; j < np; ++j) line[j] = X(row0 + c, j);
            cvec u = op.plan_y.forward(line);
            for (size_t m = 0; m < M; ++m) out[m] += Ax[m + c * M] * op.Dy[m] * u[m];
        }
    };
    side_x_edge(op.Lx, 0);
    side_x_edge(op.Rx, np);
    auto side_y_edge = [&](const cvec& By, size_t col0) {
        for (int c = 0; c < p; ++c) {
            std::fill(line.begin(), line.end(), cd(0.0));
            for (size_t i = p; i < np; ++i) line[i] = X(i, col0 + c);
            cvec u = op.plan_x.forward(line);
            for (size_t m = 0; m < M; ++m) out[m] += By[m + c * M] * op.Dx[m] * u[m];
        }
    };
    side_y_edge(op.Ly, 0);
    side_y_edge(op.Ry, np);
    return out;
}

cvec apply_adjoint(const Op& op, const cvec& y) {  // freq2wave.cpp:305-387
    if (y.size() != op.rows()) shape("sample vector length mismatch");
    size_t M = op.rows();
    size_t n = op.n;
    int p = op.fam.p;
    bool edged = p >= 2;
    if (op.dim == 1) {
        cvec v(M);
        for (size_t m = 0; m < M; ++m) v[m] = std::conj(op.Dx[m]) * y[m];
        cvec z = internal_adjoint_1d(op, v);
        if (edged) {
            for (int c = 0; c < p; ++c) z[c] = z[n - 1 - c] = 0.0;
            for (int c = 0; c < p; ++c) {
                cd a = 0.0, b = 0.0;
                for (size_t m = 0; m < M; ++m) {
                    a += std::conj(op.Lx[m + c * M]) * y[m];
                    b += std::conj(op.Rx[m + c * M]) * y[m];
                }
                z[c] += a;
                z[n - p + c] += b;
            }
        }
        return z;
    }
    cvec out(op.cols(), cd(0.0));
    auto Z = [&](size_t i, size_t j) -> cd& { return out[j * n + i]; };
    {
        cvec v(M);
        for (size_t m = 0; m < M; ++m) v[m] = std::conj(op.Dx[m] * op.Dy[m]) * y[m];
        cvec w = op.plan_2d.adjoint(v);
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < n; ++i) {
                bool inner = i >= (size_t)p && i < n - p && j >= (size_t)p && j < n - p;
                if (!edged || inner) Z(i, j) = w[j * n + i];
            }
    }
    if (!edged) return out;
    size_t np = n - p;
    auto corner = [&](const cvec& Ax, size_t row0, const cvec& By, size_t col0) {
        for (int i = 0; i < p; ++i)
            for (int j = 0; j < p; ++j) {
                cd acc = 0.0;
                for (size_t m = 0; m < M; ++m)
                    acc += std::conj(Ax[m + i * M]) * (y[m] * std::conj(By[m + j * M]));
                Z(row0 + i, col0 + j) += acc;
            }
    };
    corner(op.Lx, 0, op.Ly, 0);
    corner(op.Lx, 0, op.Ry, np);
    corner(op.Rx, np, op.Ly, 0);
    corner(op.Rx, np, op.Ry, np);
    cvec v(M);
    auto side_x_edge = [&](const cvec& Ax, size_t row0) {
        for (int c = 0; c < p; ++c) {
            for (size_t m = 0; m < M; ++m) v[m] = std::conj(Ax[m + c * M] * op.Dy[m]) * y[m];
            cvec w = op.plan_y.adjoint(v);
            for (size_t j = p; j < np; ++j) Z(row0 + c, j) += w[j];
        }
    };
    side_x_edge(op.Lx, 0);
    side_x_edge(op.Rx, np);
    auto side_y_edge = [&](const cvec& By, size_t col0) {
        for (int c = 0; c < p; ++c) {
            for (size_t m = 0; m < M; ++m) v[m] = std::conj(By[m + c * M] * op.Dx[m]) * y[m];
            cvec w = op.plan_x.adjoint(v);
            for (size_t i = p; i < np; ++i) Z(i, col0 + c) += w[i];
        }
    };
    side_y_edge(op.Ly, 0);
    side_y_edge(op.Ry, np);
    return out;
}

std::vector<cd> dense_axis_row(const Op& op, double xi, const Boundary* left, const Boundary* right) {
    size_t n = op.n;  // freq2wave.cpp:392-416
    int p = op.fam.p;
    double scaled = std::ldexp(xi, -op.J);
    double amp = std::exp2(-0.5 * op.J);
    std::vector<cd> row(n);
    cd interior = amp * fourier_scaling(op.fam, scaled, op.terms);
    for (size_t c = 0; c < n; ++c) {
        long long k = static_cast<long long>(c) - op.n / 2;
        row[c] = interior * std::polar(1.0, -kTwoPi * static_cast<double>(k) * scaled);
    }
    if (p >= 2) {
        std::vector<cd> vl = fourier_boundary(op.fam, *left, scaled, op.depth, op.terms);
        std::vector<cd> vr = fourier_boundary(op.fam, *right, scaled, op.depth, op.terms);
        cd pl = amp * std::polar(1.0, kPi * xi);
        cd pr = amp * std::polar(1.0, -kPi * xi);
        for (int c = 0; c < p; ++c) {
            row[c] = pl * vl[c];
            row[n - p + c] = pr * vr[p - 1 - c];
        }
    }
    return row;
}

// ---------------------------------------------------------------- solver.cpp
double norm2(const cvec& v) {
    double acc = 0.0;
    for (const cd& z : v) acc += std::norm(z);
    return acc;
}

struct SolveResult {
    cvec x;
    int iterations = 0;
    double residual = 0.0;
    std::vector<double> history;
    bool converged = false;
};

SolveResult solve(const Op& op, const cvec& samples, const cvec* x0, int max_iterations, double tol) {
    size_t n = op.cols();  // solver.cpp:19-91
    if (samples.size() != op.rows()) shape("sample vector length mismatch");
    if (tol <= 0) domain("tolerance must be positive");
    int max_iter = max_iterations > 0 ? max_iterations : 2 * static_cast<int>(n);
    cvec b(samples);
    if (op.weighted())
        for (size_t m = 0; m < b.size(); ++m) b[m] *= op.sqrt_weights[m];
    cvec x(n, cd(0.0));
    if (x0) {
        if (x0->size() != n) shape("initial guess length mismatch");
        x = *x0;
    }
    SolveResult st;
    double ref = std::sqrt(norm2(apply_adjoint(op, b)));
    if (ref == 0.0) {
        st.converged = true;
        st.history = {0.0};
        st.x = cvec(n, cd(0.0));
        return st;
    }
    cvec r = b;
    {
        cvec tx = apply_forward(op, x);
        for (size_t m = 0; m < r.size(); ++m) r[m] -= tx[m];
    }
    cvec s = apply_adjoint(op, r);
    double gamma = norm2(s);
    st.history.push_back(std::sqrt(gamma) / ref);
    if (st.history.back() <= tol) {
        st.converged = true;
        st.residual = st.history.back();
        st.x = x;
        return st;
    }
    cvec pv = s, q;
    for (int it = 1; it <= max_iter; ++it) {
        q = apply_forward(op, pv);
        double qq = norm2(q);
        if (qq == 0.0) break;
        double alpha = gamma / qq;
        for (size_t i = 0; i < n; ++i) x[i] += alpha * pv[i];
        for (size_t m = 0; m < r.size(); ++m) r[m] -= alpha * q[m];
        s = apply_adjoint(op, r);
        double gnew = norm2(s);
        st.iterations = it;
        st.history.push_back(std::sqrt(gnew) / ref);
        if (st.history.back() <= tol) {
            st.converged = true;
            break;
        }
        double beta = gnew / gamma;
        gamma = gnew;
        for (size_t i = 0; i < n; ++i) pv[i] = s[i] + beta * pv[i];
    }
    st.residual = st.history.back();
    st.x = x;
    return st;
}

// ---------------------------------------------------------------- patterns.cpp
std::vector<double> gen_grid(long long M, double eps, int dim) {  // patterns.cpp:14-44
    if (M < 1) domain("M must be >= 1");
    if (!(eps > 0)) domain("epsilon must be positive");
    if (dim != 1 && dim != 2) domain("dim must be 1 or 2");
    std::vector<double> axis(M);
    double half = static_cast<double>(M) / 2.0;
    for (long long m = 0; m < M; ++m) axis[m] = eps * (static_cast<double>(m) - half);
    if (dim == 1) return axis;
    std::vector<double> out;
    out.reserve(M * M * 2);
    for (double x : axis)
        for (double y : axis) {
            out.push_back(x);
            out.push_back(y);
        }
    return out;
}

std::vector<double> gen_jitter(long long M, double eps, double eta, uint64_t seed, int dim) {
    if (!(eta >= 0) || eta >= eps / 2) domain("eta must satisfy 0 <= eta < epsilon/2");
    std::vector<double> c = gen_grid(M, eps, dim);  // patterns.cpp:46-56
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> shift(-eta, eta);
    for (double& v : c) v += shift(rng);
    if (dim == 1) std::sort(c.begin(), c.end());
    return c;
}

std::vector<double> gen_spiral(int turns, double ppt, double K) {  // patterns.cpp:58-74
    if (turns < 1) domain("turns must be >= 1");
    if (!(ppt > 0)) domain("points_per_turn must be positive");
    if (!(K > 0)) domain("K must be positive");
    long long count = std::llround(turns * ppt);
    std::vector<double> c;
    c.reserve(count * 2);
    for (long long i = 0; i < count; ++i) {
        double t = static_cast<double>(i) / ppt;
        double radius = K * t / static_cast<double>(turns);
        double angle = 2.0 * std::numbers::pi * t;
        c.push_back(radius * std::cos(angle));
        c.push_back(radius * std::sin(angle));
    }
    return c;
}

// ---------------------------------------------------------------- weights.cpp
struct P2 { double x, y; };
std::vector<P2> clip_half_plane(const std::vector<P2>& poly, P2 mid, P2 a) {  // weights.cpp:20-38
    std::vector<P2> out;
    out.reserve(poly.size() + 2);
    size_t n = poly.size();
    auto sd = [&](const P2& q) { return a.x * (q.x - mid.x) + a.y * (q.y - mid.y); };
    for (size_t i = 0; i < n; ++i) {
        const P2& cur = poly[i];
        const P2& nxt = poly[(i + 1) % n];
        double dc = sd(cur), dn = sd(nxt);
        if (dc <= 0) out.push_back(cur);
        if ((dc < 0 && dn > 0) || (dc > 0 && dn < 0)) {
            double t = dc / (dc - dn);
            out.push_back({cur.x + t * (nxt.x - cur.x), cur.y + t * (nxt.y - cur.y)});
        }
    }
    return out;
}
double polygon_area(const std::vector<P2>& poly) {  // weights.cpp:40-49
    double acc = 0.0;
    size_t n = poly.size();
    for (size_t i = 0; i < n; ++i) acc += poly[i].x * poly[(i + 1) % n].y - poly[(i + 1) % n].x * poly[i].y;
    return 0.5 * std::abs(acc);
}

std::vector<double> voronoi(int dim, const std::vector<double>& c, double K) {  // weights.cpp:95-133
    if (!(K > 0)) domain("K must be positive");
    if (dim == 1) {
        size_t M = c.size();
        if (M == 0) shape("empty point set");
        std::vector<size_t> order(M);
        std::iota(order.begin(), order.end(), 0);
        std::sort(order.begin(), order.end(), [&](size_t a, size_t b) { return c[a] < c[b]; });
        std::vector<double> s(M);
        for (size_t i = 0; i < M; ++i) s[i] = c[order[i]];
        for (size_t i = 1; i < M; ++i)
            if (s[i] == s[i - 1]) domain("degenerate input: duplicate sample points");
        if (s.front() < -K || s.back() > K) domain("point outside the bandwidth region");
        std::vector<double> mu(M);
        for (size_t i = 0; i < M; ++i) {
            double lo = (i == 0) ? -K : 0.5 * (s[i - 1] + s[i]);
            double hi = (i + 1 == M) ? K : 0.5 * (s[i] + s[i + 1]);
            mu[order[i]] = hi - lo;
        }
        return mu;
    }
    size_t M = c.size() / 2;
    if (M == 0) shape("empty point set");
    std::vector<P2> pts(M);
    for (size_t m = 0; m < M; ++m) {
        pts[m] = {c[2 * m], c[2 * m + 1]};
        if (std::abs(pts[m].x) > K || std::abs(pts[m].y) > K) domain("point outside the bandwidth region");
    }
    for (size_t i = 0; i < M; ++i)
        for (size_t j = i + 1; j < M; ++j)
            if (pts[i].x == pts[j].x && pts[i].y == pts[j].y) domain("degenerate input: duplicate sample points");
    std::vector<double> mu(M);
    for (size_t m = 0; m < M; ++m) {
        std::vector<P2> poly = {{-K, -K}, {K, -K}, {K, K}, {-K, K}};
        for (size_t j = 0; j < M; ++j) {
            if (j == m) continue;
            P2 mid = {(pts[m].x + pts[j].x) / 2, (pts[m].y + pts[j].y) / 2};
            P2 a = {pts[j].x - pts[m].x, pts[j].y - pts[m].y};
            poly = clip_half_plane(poly, mid, a);
            if (poly.empty()) break;
        }
        mu[m] = polygon_area(poly);
    }
    return mu;
}


// Same cells as voronoi() (weights.cpp:59-70 clipping, identical clip and
// area code) for point sets too large for the reference's O(M^2) loop: each
// cell is clipped against its neighbours in increasing distance, taken from a
// bucket grid ring by ring, until the next ring lies beyond twice the cell's
// farthest vertex (no further point can cut it).  The clip order differs
// from the reference's index order, so areas agree to roundoff (~1e-16
// relative), not bit for bit.  Threads split the points.  Harness only: the
// CPU legs of bench.py use it so that they never load the product library.
std::vector<double> voronoi_fast_2d(const std::vector<double>& c, double K, int nthreads) {
    if (!(K > 0)) domain("K must be positive");
    const size_t M = c.size() / 2;
    if (M == 0) shape("empty point set");
    for (size_t m = 0; m < M; ++m)
        if (std::abs(c[2 * m]) > K || std::abs(c[2 * m + 1]) > K) domain("point outside the bandwidth region");
    const double h = std::max(2.0 * K / std::max(1.0, std::sqrt((double)M)), 1e-300);
    const int nb = std::max(1, (int)std::ceil(2.0 * K / h));
    auto bucket = [&](double v) { return std::min(nb - 1, std::max(0, (int)std::floor((v + K) / h))); };
    std::vector<int> start(nb * nb + 1, 0), order(M);
    for (size_t m = 0; m < M; ++m) ++start[bucket(c[2 * m + 1]) * nb + bucket(c[2 * m]) + 1];
    for (int i = 0; i < nb * nb; ++i) start[i + 1] += start[i];
    std::vector<int> fill(start.begin(), start.end() - 1);
    for (size_t m = 0; m < M; ++m) order[fill[bucket(c[2 * m + 1]) * nb + bucket(c[2 * m])]++] = (int)m;
    std::vector<double> mu(M);
    std::atomic<int> dup{0};
    auto work = [&](size_t lo, size_t hi) {
        std::vector<std::pair<double, int>> cand;
        for (size_t m = lo; m < hi; ++m) {
            const P2 own = {c[2 * m], c[2 * m + 1]};
            const int bx = bucket(own.x), by = bucket(own.y);
            std::vector<P2> poly = {{-K, -K}, {K, -K}, {K, K}, {-K, K}};
            for (int r = 0;; ++r) {
                // the cell's farthest vertex bounds every cutting neighbour to 2 * rmax
                double rmax = 0.0;
                for (const P2& v : poly) rmax = std::max(rmax, std::hypot(v.x - own.x, v.y - own.y));
                if (r >= 2 && (r - 1) * h > 2.0 * rmax) break;
                if (r > nb) break;
                cand.clear();
                for (int yy = by - r; yy <= by + r; ++yy) {
                    if (yy < 0 || yy >= nb) continue;
                    for (int xx = bx - r; xx <= bx + r; ++xx) {
                        if (xx < 0 || xx >= nb) continue;
                        if (std::max(std::abs(xx - bx), std::abs(yy - by)) != r) continue;
                        const int b = yy * nb + xx;
                        for (int k = start[b]; k < start[b + 1]; ++k) {
                            const int j = order[k];
                            if ((size_t)j == m) continue;
                            const double dx = c[2 * j] - own.x, dy = c[2 * j + 1] - own.y;
                            if (dx == 0.0 && dy == 0.0) dup = 1;
                            cand.push_back({dx * dx + dy * dy, j});
                        }
                    }
                }
                std::sort(cand.begin(), cand.end());
                for (const auto& cj : cand) {
                    const int j = cj.second;
                    P2 mid = {(own.x + c[2 * j]) / 2, (own.y + c[2 * j + 1]) / 2};
                    P2 a = {c[2 * j] - own.x, c[2 * j + 1] - own.y};
                    poly = clip_half_plane(poly, mid, a);
                    if (poly.empty()) break;
                }
                if (poly.empty()) break;
            }
            mu[m] = polygon_area(poly);
        }
    };
    const int T = std::max(1, nthreads);
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(work, M * t / T, M * (t + 1) / T);
    for (auto& t : th) t.join();
    if (dup) domain("degenerate input: duplicate sample points");
    return mu;
}

// ---------------------------------------------------------------- dyadic evaluation (dyadic.cpp)
// Least squares by Householder QR of the (n+1) x n consistent system
// (Eigen colPivHouseholderQr, dyadic.cpp:29): the solution is unique.
std::vector<double> qr_solve(std::vector<double> A, std::vector<double> b, int rows, int cols) {
    for (int k = 0; k < cols; ++k) {
        double nrm = 0.0;
        for (int i = k; i < rows; ++i) nrm += A[i * cols + k] * A[i * cols + k];
        nrm = std::sqrt(nrm);
        if (nrm == 0.0) continue;
        double alpha = A[k * cols + k] > 0 ? -nrm : nrm;
        std::vector<double> v(rows, 0.0);
        for (int i = k; i < rows; ++i) v[i] = A[i * cols + k];
        v[k] -= alpha;
        double vv = 0.0;
        for (int i = k; i < rows; ++i) vv += v[i] * v[i];
        if (vv == 0.0) continue;
        for (int j = k; j < cols; ++j) {
            double d = 0.0;
            for (int i = k; i < rows; ++i) d += v[i] * A[i * cols + j];
            d = 2.0 * d / vv;
            for (int i = k; i < rows; ++i) A[i * cols + j] -= d * v[i];
        }
        double d = 0.0;
        for (int i = k; i < rows; ++i) d += v[i] * b[i];
        d = 2.0 * d / vv;
        for (int i = k; i < rows; ++i) b[i] -= d * v[i];
    }
    std::vector<double> x(cols);
    for (int i = cols - 1; i >= 0; --i) {
        double acc = b[i];
        for (int j = i + 1; j < cols; ++j) acc -= A[i * cols + j] * x[j];
        x[i] = acc / A[i * cols + i];
    }
    return x;
}

// phi at the integers -p+2..p-1: eigenvector of T(n,m) = 2 h(2n - m) for
// eigenvalue 1, sum 1 (dyadic.cpp:14-35)
std::vector<double> integer_values(const Family& fam) {
    int p = fam.p, n = 2 * p - 2;
    auto tap = [&](int k) { return (k < -p + 1 || k > p) ? 0.0 : fam.taps[k + p - 1]; };
    std::vector<double> sys((n + 1) * n, 0.0), rhs(n + 1, 0.0);
    for (int r = 0; r < n; ++r)
        for (int c = 0; c < n; ++c) sys[r * n + c] = 2.0 * tap(2 * (r - p + 2) - (c - p + 2)) - (r == c ? 1.0 : 0.0);
    for (int c = 0; c < n; ++c) sys[n * n + c] = 1.0;
    rhs[n] = 1.0;
    std::vector<double> v = qr_solve(sys, rhs, n + 1, n);
    double res = 0.0;
    for (int r = 0; r <= n; ++r) {
        double acc = -rhs[r];
        for (int c = 0; c < n; ++c) acc += sys[r * n + c] * v[c];
        res += acc * acc;
    }
    if (std::sqrt(res) > 1e-10) numerical("integer value eigenproblem did not solve");
    return v;
}

struct FTable {  // dyadic.hpp:13-25
    int R = 0;
    long long support_begin = 0;
    std::vector<double> values;
    double at(long long num) const {
        long long idx = num - (support_begin << R);
        if (idx < 0 || idx >= (long long)values.size()) return 0.0;
        return values[(size_t)idx];
    }
};

FTable scaling_dyadic(const Family& fam, int R) {  // dyadic.cpp:37-68
    if (R < 0) domain("resolution must be >= 0");
    FTable t;
    t.R = R;
    t.support_begin = -fam.p + 1;
    size_t len = ((size_t)(2 * fam.p - 1) << R) + 1;
    t.values.assign(len, 0.0);
    if (fam.p == 1) {
        for (size_t i = 0; i + 1 < len; ++i) t.values[i] = 1.0;
        return t;
    }
    std::vector<double> iv = integer_values(fam);
    for (size_t k = 0; k < iv.size(); ++k) t.values[(k + 1) << R] = iv[k];
    for (int r = 1; r <= R; ++r) {
        long long step = 1LL << (R - r);
        for (long long i = step; i < (long long)len; i += 2 * step) {
            long long nx = (t.support_begin << R) + i;
            double acc = 0.0;
            for (int k = -fam.p + 1; k <= fam.p; ++k) acc += fam.taps[k + fam.p - 1] * t.at(2 * nx - ((long long)k << R));
            t.values[(size_t)i] = 2.0 * acc;
        }
    }
    return t;
}

std::vector<FTable> boundary_dyadic(const Family& fam, bool left, int R) {  // dyadic.cpp:70-115
    if (fam.p < 2) domain("boundary functions require p >= 2");
    if (R < 0) domain("resolution must be >= 0");
    const int p = fam.p;
    const gsdata::FamilyData& f = gsdata::kFamilies[p - 1];
    const double* H = left ? f.left_H : f.right_H;
    const double* h = left ? f.left_h : f.right_h;
    const double* seed = left ? f.left_seed : f.right_seed;
    FTable interior = scaling_dyadic(fam, R);
    std::vector<FTable> tabs(p);
    for (int k = 0; k < p; ++k) {
        FTable& t = tabs[k];
        t.R = R;
        t.support_begin = left ? 0 : -(p + k);
        t.values.assign(((size_t)(p + k) << R) + 1, 0.0);
        for (int d = 0; d <= p + k; ++d) {
            long long nn = left ? d : -d;
            t.values[(size_t)((nn - t.support_begin) << R)] = seed[k * 2 * p + d];
        }
    }
    const double sqrt2 = std::sqrt(2.0);
    for (int r = 1; r <= R; ++r) {
        long long step = 1LL << (R - r);
        for (int k = 0; k < p; ++k) {
            FTable& t = tabs[k];
            for (long long i = step; i < (long long)t.values.size(); i += 2 * step) {
                long long nx = (t.support_begin << R) + i;
                double acc = 0.0;
                for (int l = 0; l < p; ++l) acc += H[k * p + l] * tabs[l].at(2 * nx);
                for (int m = p; m <= p + 2 * k; ++m) {
                    long long arg = left ? 2 * nx - ((long long)m << R) : 2 * nx + ((long long)(m + 1) << R);
                    acc += h[k * (2 * p - 1) + (m - p)] * interior.at(arg);
                }
                t.values[(size_t)i] = sqrt2 * acc;
            }
        }
    }
    return tabs;
}

// sink(i, w * 2^{J/2} * basis column c at grid point i)  (dyadic.cpp:121-170)
struct Basis {
    const Family& fam;
    int J, R, tabres;
    long long n_grid;
    FTable interior;
    std::vector<FTable> left, right;
    double amplitude;
    Basis(const Family& f, int J_, int R_)
        : fam(f), J(J_), R(R_), tabres(R_ - J_), n_grid(1LL << R_), interior(scaling_dyadic(f, R_ - J_)),
          amplitude(std::exp2(0.5 * J_)) {
        if (f.p >= 2) {
            left = boundary_dyadic(f, true, tabres);
            right = boundary_dyadic(f, false, tabres);
        }
    }
    template <class Sink>
    void column(long long c, double w, Sink&& sink) const {
        long long n = 1LL << J, unit = 1LL << tabres;
        double scale = w * amplitude;
        if (fam.p >= 2 && c < fam.p) {
            const FTable& t = left[(size_t)c];
            long long hi = std::min<long long>(n_grid, (fam.p + c) * unit);
            for (long long i = 0; i <= hi; ++i) sink(i, scale * t.values[(size_t)i]);
        } else if (fam.p >= 2 && c >= n - fam.p) {
            const FTable& t = right[(size_t)(n - 1 - c)];
            long long lo = std::max<long long>(0, n_grid - (fam.p + (n - 1 - c)) * unit);
            for (long long i = lo; i <= n_grid; ++i) sink(i, scale * t.at(i - n_grid));
        } else {
            long long lo = std::max<long long>(0, (c - fam.p + 1) * unit);
            long long hi = std::min<long long>(n_grid, (c + fam.p) * unit);
            for (long long i = lo; i <= hi; ++i) sink(i, scale * interior.at(i - c * unit));
        }
    }
};

void check_weval(const Family& fam, int J, int R, size_t got, size_t want) {  // dyadic.cpp:172-180
    if ((1LL << J) < 2 * fam.p) domain("scale too small: 2^J must be >= 2p");
    if (R < J) domain("resolution too coarse: R must be >= J");
    if (got != want) shape("coefficient vector has wrong length");
}

std::vector<double> weval(int dim, const Family& fam, int J, int R, const std::vector<double>& coeffs) {
    const size_t n = (size_t)1 << J, g = ((size_t)1 << R) + 1;
    check_weval(fam, J, R, coeffs.size(), dim == 1 ? n : n * n);
    Basis basis(fam, J, R);
    if (dim == 1) {  // dyadic.cpp:184-199
        std::vector<double> out(g, 0.0);
        for (size_t c = 0; c < n; ++c) {
            double w = coeffs[c];
            if (w == 0.0) continue;
            basis.column((long long)c, w, [&](long long i, double v) { out[(size_t)i] += v; });
        }
        return out;
    }
    // dyadic.cpp:201-230: out(iy, ix) = sum_j (B X^T)(iy, j) B(ix, j), X(i, j) = coeffs[j n + i]
    std::vector<double> B(g * n, 0.0);
    for (size_t c = 0; c < n; ++c) basis.column((long long)c, 1.0, [&](long long i, double v) { B[(size_t)i * n + c] = v; });
    std::vector<double> Z(g * n, 0.0);
    for (size_t a = 0; a < g; ++a)
        for (size_t i = 0; i < n; ++i) {
            double b = B[a * n + i];
            if (b == 0.0) continue;
            for (size_t j = 0; j < n; ++j) Z[a * n + j] += b * coeffs[i * n + j];
        }
    std::vector<double> out(g * g, 0.0);
    for (size_t a = 0; a < g; ++a)
        for (size_t bx = 0; bx < g; ++bx) {
            double acc = 0.0;
            for (size_t j = 0; j < n; ++j) acc += Z[a * n + j] * B[bx * n + j];
            out[a * g + bx] = acc;
        }
    return out;
}

}  // namespace orc

// ============================================================================
// C ABI for ctypes (tests / bench cpu_baseline).  Complex arrays are
// interleaved (re, im) doubles.  Return 0 or the reference ErrorClass code.
// ============================================================================
namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const orc::Err& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}
orc::cvec cv(const double* a, size_t n) {
    orc::cvec v(n);
    if (n) std::memcpy(static_cast<void*>(v.data()), a, n * sizeof(orc::cd));
    return v;
}
void put(double* dst, const orc::cvec& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(orc::cd));
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

int orc_op_create(int dim, int p, int J, long long M, const double* coords, const double* weights,
                  int has_bw, double bw, double sigma, int w, int depth, int terms, int allow_uniform,
                  void** out) {
    return guard([&] {
        std::vector<double> c(coords, coords + M * dim);
        std::vector<double> wt;
        if (weights) wt.assign(weights, weights + M);
        *out = orc::freq2wave(dim, p, J, c, wt, has_bw != 0, bw, sigma, w, depth, terms, allow_uniform != 0);
    });
}
void orc_op_destroy(void* op) { delete static_cast<orc::Op*>(op); }
int orc_op_info(void* h, long long* rows, long long* cols, int* uniform_fast, double* eps) {
    auto* op = static_cast<orc::Op*>(h);
    *rows = op->rows();
    *cols = op->cols();
    *uniform_fast = op->uniform_fast;
    *eps = op->uniform_epsilon;
    return 0;
}
int orc_forward(void* h, const double* x, double* y) {
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] { put(y, orc::apply_forward(*op, cv(x, op->cols()))); });
}
int orc_adjoint(void* h, const double* y, double* z) {
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] { put(z, orc::apply_adjoint(*op, cv(y, op->rows()))); });
}
int orc_forward_n(void* h, const double* x, long long nx, double* y) {  // shape-checked variant
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] { put(y, orc::apply_forward(*op, cv(x, nx))); });
}
int orc_adjoint_n(void* h, const double* y, long long ny, double* z) {
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] { put(z, orc::apply_adjoint(*op, cv(y, ny))); });
}
int orc_factors(void* h, int axis, double* D, double* L, double* R) {
    auto* op = static_cast<orc::Op*>(h);
    const orc::cvec& d = axis == 0 ? op->Dx : op->Dy;
    const orc::cvec& l = axis == 0 ? op->Lx : op->Ly;
    const orc::cvec& r = axis == 0 ? op->Rx : op->Ry;
    put(D, d);
    if (L) put(L, l);
    if (R) put(R, r);
    return 0;
}
int orc_densify(void* h, long long cap, double* out) {  // row-major M x cols
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] {
        size_t M = op->rows(), nc = op->cols();
        if (M * nc > static_cast<size_t>(cap)) orc::domain("densify: matrix exceeds the entry cap");
        orc::Boundary l, r;
        if (op->fam.p >= 2) {
            l = orc::make_boundary(op->fam, true);
            r = orc::make_boundary(op->fam, false);
        }
        orc::cd* o = reinterpret_cast<orc::cd*>(out);
        for (size_t m = 0; m < M; ++m) {
            double wgt = op->weighted() ? op->sqrt_weights[m] : 1.0;
            auto rx = orc::dense_axis_row(*op, op->coords[m * op->dim], &l, &r);
            if (op->dim == 1) {
                for (size_t c = 0; c < nc; ++c) o[m * nc + c] = wgt * rx[c];
            } else {
                auto ry = orc::dense_axis_row(*op, op->coords[m * 2 + 1], &l, &r);
                size_t n = op->n;
                for (size_t j = 0; j < n; ++j)
                    for (size_t i = 0; i < n; ++i) o[m * nc + j * n + i] = wgt * rx[i] * ry[j];
            }
        }
    });
}
int orc_solve(void* h, const double* b, long long nb, const double* x0, int max_iter, double tol, double* x,
              int* iterations, double* residual, int* converged, double* history, int* history_len) {
    auto* op = static_cast<orc::Op*>(h);
    return guard([&] {
        orc::cvec bb = cv(b, nb);
        orc::cvec xx0;
        if (x0) xx0 = cv(x0, op->cols());
        orc::SolveResult r = orc::solve(*op, bb, x0 ? &xx0 : nullptr, max_iter, tol);
        put(x, r.x);
        *iterations = r.iterations;
        *residual = r.residual;
        *converged = r.converged;
        if (history) std::memcpy(history, r.history.data(), r.history.size() * sizeof(double));
        *history_len = static_cast<int>(r.history.size());
    });
}
int orc_fourier_scaling(int p, double xi, int terms, double* out) {
    return guard([&] {
        orc::cd v = orc::fourier_scaling(orc::make_family(p), xi, terms);
        out[0] = v.real();
        out[1] = v.imag();
    });
}
int orc_fourier_boundary(int p, int left, double xi, int depth, int terms, double* out) {
    return guard([&] {
        orc::Family f = orc::make_family(p);
        orc::Boundary b = orc::make_boundary(f, left != 0);
        put(out, orc::fourier_boundary(f, b, xi, depth, terms));
    });
}
int orc_boundary_at_zero(int p, int left, double* out) {
    return guard([&] {
        orc::Boundary b = orc::make_boundary(orc::make_family(p), left != 0);
        put(out, b.v_zero);
    });
}
int orc_boundary_UV(int p, int left, double* U, double* V) {
    return guard([&] {
        orc::Boundary b = orc::make_boundary(orc::make_family(p), left != 0);
        std::memcpy(U, b.U.data(), b.U.size() * 8);
        std::memcpy(V, b.V.data(), b.V.size() * 8);
    });
}
int orc_family_taps(int p, double* out) {
    return guard([&] {
        orc::Family f = orc::make_family(p);
        std::memcpy(out, f.taps.data(), f.taps.size() * 8);
    });
}
int orc_ndft(int adjoint, int dim, int N0, int N1, long long M, const double* pts, const double* in, double* out) {
    return guard([&] {
        int N[2] = {N0, N1};
        std::vector<double> pp(pts, pts + M * dim);
        size_t len = static_cast<size_t>(N0) * (dim == 2 ? N1 : 1);
        if (adjoint) put(out, orc::ndft_adjoint(dim, N, pp, cv(in, M)));
        else put(out, orc::ndft_forward(dim, N, pp, cv(in, len)));
    });
}
int orc_nfft(int adjoint, int dim, int N0, int N1, long long M, const double* pts, double sigma, int w,
             const double* in, double* out, int* n_over) {
    return guard([&] {
        int N[2] = {N0, N1};
        std::vector<double> pp(pts, pts + M * dim);
        orc::NfftPlan plan(dim, N, pp, sigma, w);
        if (n_over) {
            n_over[0] = plan.n[0];
            n_over[1] = plan.n[1];
        }
        if (!in) return;
        if (adjoint) put(out, plan.adjoint(cv(in, M)));
        else put(out, plan.forward(cv(in, plan.grid_size())));
    });
}
int orc_kb_weights(int dim_unused, long long M, const double* pts, int n_over, double sigma, int w,
                   long long* base, double* weights, double* deconv, int N) {
    (void)dim_unused;
    return guard([&] {
        double beta = orc::kb_beta(w, sigma);
        int S = 2 * w + 1;
        for (long long m = 0; m < M; ++m) {
            double pos = pts[m] * n_over;
            long long j0 = std::llround(pos);
            base[m] = j0 - w;
            for (int t = 0; t < S; ++t) weights[m * S + t] = orc::kb_kernel(pos - static_cast<double>(j0 - w + t), w, beta);
        }
        if (deconv)
            for (int k = -N / 2; k < N / 2; ++k)
                deconv[k + N / 2] = 1.0 / orc::kb_transform(static_cast<double>(k) / n_over, w, beta);
    });
}
int orc_uniform(int adjoint, const double* in, long long n_in, long long M, double eps, long long N, double* out) {
    return guard([&] {
        if (adjoint) put(out, orc::uniform_ndft_adjoint_fft(cv(in, n_in), eps, N));
        else put(out, orc::uniform_ndft_fft(cv(in, n_in), M, eps, N));
    });
}
int orc_gen_grid(long long M, double eps, int dim, double* out) {
    return guard([&] { auto v = orc::gen_grid(M, eps, dim); std::memcpy(out, v.data(), v.size() * 8); });
}
int orc_gen_jitter(long long M, double eps, double eta, unsigned long long seed, int dim, double* out) {
    return guard([&] { auto v = orc::gen_jitter(M, eps, eta, seed, dim); std::memcpy(out, v.data(), v.size() * 8); });
}
int orc_gen_spiral(int turns, double ppt, double K, double* out) {
    return guard([&] { auto v = orc::gen_spiral(turns, ppt, K); std::memcpy(out, v.data(), v.size() * 8); });
}
int orc_voronoi(int dim, long long M, const double* coords, double K, double* mu) {
    return guard([&] {
        std::vector<double> c(coords, coords + M * dim);
        auto v = orc::voronoi(dim, c, K);
        std::memcpy(mu, v.data(), v.size() * 8);
    });
}
int orc_voronoi_fast(int dim, long long M, const double* coords, double K, double* mu, int nthreads) {
    return guard([&] {
        std::vector<double> c(coords, coords + M * dim);
        auto v = dim == 2 ? orc::voronoi_fast_2d(c, K, nthreads) : orc::voronoi(dim, c, K);
        std::memcpy(mu, v.data(), v.size() * 8);
    });
}
// dyadic tables / evaluation (dyadic.cpp); two-call pattern: out == NULL -> sizes only
int orc_scaling_dyadic(int p, int R, double* out, long long* len, long long* support_begin) {
    return guard([&] {
        orc::FTable t = orc::scaling_dyadic(orc::make_family(p), R);
        *len = (long long)t.values.size();
        *support_begin = t.support_begin;
        if (out) std::memcpy(out, t.values.data(), t.values.size() * 8);
    });
}
int orc_boundary_dyadic(int p, int left, int R, int k, double* out, long long* len, long long* support_begin) {
    return guard([&] {
        auto tabs = orc::boundary_dyadic(orc::make_family(p), left != 0, R);
        if (k < 0 || k >= p) orc::domain("edge function index out of range");
        const orc::FTable& t = tabs[(size_t)k];
        *len = (long long)t.values.size();
        *support_begin = t.support_begin;
        if (out) std::memcpy(out, t.values.data(), t.values.size() * 8);
    });
}
int orc_weval(int dim, int p, int J, int R, const double* coeffs, long long ncoeffs, double* out) {
    return guard([&] {
        if (dim != 1 && dim != 2) orc::domain("dim must be 1 or 2");
        std::vector<double> c(coeffs, coeffs + ncoeffs);
        auto v = orc::weval(dim, orc::make_family(p), J, R, c);
        std::memcpy(out, v.data(), v.size() * 8);
    });
}
double orc_wrap_half_open(double z) { return orc::wrap_half_open(z); }

}  // extern "C"
