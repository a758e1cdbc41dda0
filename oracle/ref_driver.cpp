// C entry points over the UNMODIFIED reference library -- TEST INFRASTRUCTURE ONLY.
//
// oracle/Makefile compiles the reference's own sources where they lie
// (/root/reference/proj/src/{scaling,family_tables,fourier,dyadic,nufft,
// freq2wave,weights,solver,patterns}.cpp) against two stand-ins for its
// external libraries -- tests/cpp/shim/Eigen/Dense (Eigen subset) and
// oracle/refshim/fftw3.h (FFTW surface of nufft.cpp:17-55) -- and links this
// file on top into oracle/_ref/libgs_ref.so.  Nothing of the reference is
// copied into the repository.
//
// The symbols are the ones oracle/gs_oracle.cpp exports (same names, same
// argument lists), so oracle/ref.py binds them with the oracle's own ctypes
// front-end: every test can run the restatement and the reference side by
// side.  Each entry point calls the reference's public API only:
//   orc_op_create      gs::freq2wave                      freq2wave.hpp:57
//   orc_forward/adjoint gs::apply_forward / apply_adjoint freq2wave.hpp:61, 64
//   orc_densify        gs::densify                        freq2wave.hpp:68
//   orc_solve          gs::solve_least_squares            solver.hpp:29
//   orc_ndft / orc_nfft / orc_uniform                     nufft.hpp:25-77
//   orc_fourier_* / orc_boundary_* / orc_family_taps      fourier.hpp, scaling.hpp
//   orc_gen_* / orc_voronoi                               patterns.hpp, weights.hpp
//   orc_scaling_dyadic / orc_boundary_dyadic / orc_weval  dyadic.hpp
// Entry points with no public counterpart in the reference (orc_kb_weights,
// orc_wrap_half_open: anonymous-namespace helpers there) report "not exported".
#include <array>
#include <complex>
#include <cstring>
#include <string>
#include <vector>

#include "gs/dyadic.hpp"
#include "gs/error.hpp"
#include "gs/fourier.hpp"
#include "gs/freq2wave.hpp"
#include "gs/nufft.hpp"
#include "gs/patterns.hpp"
#include "gs/scaling.hpp"
#include "gs/solver.hpp"
#include "gs/weights.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const gs::Error& e) {
        g_err = e.what();
        return e.exit_code();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 6;
    }
}

gs::cvec cv(const double* a, size_t n) {
    gs::cvec v(n);
    if (n) std::memcpy(static_cast<void*>(v.data()), a, n * sizeof(gs::cd));
    return v;
}
void put(double* dst, const gs::cvec& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(gs::cd));
}
template <class V>
void put_eigen(double* dst, const V& v) {  // column-major copy of an Eigen complex object
    gs::cd* o = reinterpret_cast<gs::cd*>(dst);
    for (long j = 0; j < v.cols(); ++j)
        for (long i = 0; i < v.rows(); ++i) o[j * v.rows() + i] = v(i, j);
}
gs::Family family_of(int p) {
    if (p < 1 || p > 8) throw gs::DomainError("family: p must be 1..8");
    return static_cast<gs::Family>(p - 1);  // scaling.hpp: haar, db2 .. db8
}
gs::Side side_of(int left) { return left ? gs::Side::left : gs::Side::right; }

}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
const char* orc_backend() { return "reference (unmodified /root/reference/proj/src, Eigen/FFTW stand-ins)"; }

int orc_op_create(int dim, int p, int J, long long M, const double* coords, const double* weights,
                  int has_bw, double bw, double sigma, int w, int depth, int terms, int allow_uniform,
                  void** out) {
    return guard([&] {
        gs::SamplingSet s;
        s.dim = dim;
        s.coords.assign(coords, coords + M * dim);
        gs::Freq2WaveOptions o;
        if (has_bw) o.bandwidth = bw;
        if (weights) o.weights.assign(weights, weights + M);
        o.sigma = sigma;
        o.w = w;
        o.boundary_depth = depth;
        o.product_terms = terms;
        o.allow_uniform_fast_path = allow_uniform != 0;
        *out = new gs::Freq2WaveOp(gs::freq2wave(s, family_of(p), J, o));
    });
}
void orc_op_destroy(void* op) { delete static_cast<gs::Freq2WaveOp*>(op); }
int orc_op_info(void* h, long long* rows, long long* cols, int* uniform_fast, double* eps) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    *rows = static_cast<long long>(op->rows());
    *cols = static_cast<long long>(op->cols());
    *uniform_fast = op->uniform_fast;
    *eps = op->uniform_epsilon;
    return 0;
}
int orc_forward(void* h, const double* x, double* y) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] { put(y, gs::apply_forward(*op, cv(x, op->cols()))); });
}
int orc_adjoint(void* h, const double* y, double* z) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] { put(z, gs::apply_adjoint(*op, cv(y, op->rows()))); });
}
int orc_forward_n(void* h, const double* x, long long nx, double* y) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] { put(y, gs::apply_forward(*op, cv(x, static_cast<size_t>(nx)))); });
}
int orc_adjoint_n(void* h, const double* y, long long ny, double* z) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] { put(z, gs::apply_adjoint(*op, cv(y, static_cast<size_t>(ny)))); });
}
int orc_factors(void* h, int axis, double* D, double* L, double* R) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    put_eigen(D, axis == 0 ? op->Dx : op->Dy);
    if (L) put_eigen(L, axis == 0 ? op->Lx : op->Ly);
    if (R) put_eigen(R, axis == 0 ? op->Rx : op->Ry);
    return 0;
}
int orc_densify(void* h, long long cap, double* out) {  // row-major M x cols
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] {
        Eigen::MatrixXcd m = gs::densify(*op, static_cast<size_t>(cap));
        gs::cd* o = reinterpret_cast<gs::cd*>(out);
        for (long i = 0; i < m.rows(); ++i)
            for (long j = 0; j < m.cols(); ++j) o[i * m.cols() + j] = m(i, j);
    });
}
int orc_solve(void* h, const double* b, long long nb, const double* x0, int max_iter, double tol, double* x,
              int* iterations, double* residual, int* converged, double* history, int* history_len) {
    auto* op = static_cast<gs::Freq2WaveOp*>(h);
    return guard([&] {
        gs::SolveOptions o;
        o.max_iterations = max_iter;
        o.tolerance = tol;
        if (x0) o.initial_guess = cv(x0, op->cols());
        auto [xs, st] = gs::solve_least_squares(*op, cv(b, static_cast<size_t>(nb)), o);
        put(x, xs);
        *iterations = st.iterations;
        *residual = st.residual;
        *converged = st.converged;
        if (history) std::memcpy(history, st.history.data(), st.history.size() * sizeof(double));
        *history_len = static_cast<int>(st.history.size());
    });
}
int orc_fourier_scaling(int p, double xi, int terms, double* out) {
    return guard([&] {
        gs::cd v = gs::fourier_scaling(gs::ScalingFamily::make(family_of(p)), xi, terms);
        out[0] = v.real();
        out[1] = v.imag();
    });
}
int orc_fourier_boundary(int p, int left, double xi, int depth, int terms, double* out) {
    return guard([&] {
        put_eigen(out, gs::fourier_boundary(gs::ScalingFamily::make(family_of(p)), side_of(left), xi, depth, terms));
    });
}
int orc_boundary_at_zero(int p, int left, double* out) {
    return guard([&] {
        put_eigen(out, gs::boundary_fourier_at_zero(gs::ScalingFamily::make(family_of(p)), side_of(left)));
    });
}
int orc_boundary_UV(int p, int left, double* U, double* V) {  // row-major p x p, p x (2p-1)
    return guard([&] {
        const gs::BoundaryFilterSet& bf = gs::boundary_filters(family_of(p), side_of(left));
        for (long i = 0; i < bf.U.rows(); ++i)
            for (long j = 0; j < bf.U.cols(); ++j) U[i * bf.U.cols() + j] = bf.U(i, j);
        for (long i = 0; i < bf.V.rows(); ++i)
            for (long j = 0; j < bf.V.cols(); ++j) V[i * bf.V.cols() + j] = bf.V(i, j);
    });
}
int orc_family_taps(int p, double* out) {
    return guard([&] {
        gs::ScalingFamily f = gs::ScalingFamily::make(family_of(p));
        std::memcpy(out, f.filter.data(), f.filter.size() * 8);
    });
}
int orc_ndft(int adjoint, int dim, int N0, int N1, long long M, const double* pts, const double* in, double* out) {
    return guard([&] {
        std::array<int, 2> N{N0, N1};
        std::vector<double> pp(pts, pts + M * dim);
        size_t len = static_cast<size_t>(N0) * (dim == 2 ? N1 : 1);
        if (adjoint) put(out, gs::ndft_adjoint(dim, N, pp, cv(in, static_cast<size_t>(M))));
        else put(out, gs::ndft_forward(dim, N, pp, cv(in, len)));
    });
}
int orc_nfft(int adjoint, int dim, int N0, int N1, long long M, const double* pts, double sigma, int w,
             const double* in, double* out, int* n_over) {
    return guard([&] {
        std::array<int, 2> N{N0, N1};
        std::vector<double> pp(pts, pts + M * dim);
        gs::NfftPlan plan = gs::plan_nfft(dim, N, pp, sigma, w);
        if (n_over) {
            n_over[0] = plan.oversampled_length(0);
            n_over[1] = dim == 2 ? plan.oversampled_length(1) : 0;
        }
        if (!in) return;
        if (adjoint) put(out, gs::nfft_adjoint(plan, cv(in, static_cast<size_t>(M))));
        else put(out, gs::nfft_forward(plan, cv(in, plan.grid_size())));
    });
}
int orc_kb_weights(int, long long, const double*, int, double, int, long long*, double*, double*, int) {
    g_err = "kb weights: not exported by the reference (anonymous namespace, nufft.cpp:138-171)";
    return 2;
}
int orc_uniform(int adjoint, const double* in, long long n_in, long long M, double eps, long long N, double* out) {
    return guard([&] {
        if (adjoint) put(out, gs::uniform_ndft_adjoint_fft(cv(in, static_cast<size_t>(n_in)), eps, N));
        else put(out, gs::uniform_ndft_fft(cv(in, static_cast<size_t>(n_in)), M, eps, N));
    });
}
int orc_gen_grid(long long M, double eps, int dim, double* out) {
    return guard([&] { auto s = gs::gen_grid(M, eps, dim); std::memcpy(out, s.coords.data(), s.coords.size() * 8); });
}
int orc_gen_jitter(long long M, double eps, double eta, unsigned long long seed, int dim, double* out) {
    return guard([&] {
        auto s = gs::gen_jitter(M, eps, eta, seed, dim);
        std::memcpy(out, s.coords.data(), s.coords.size() * 8);
    });
}
int orc_gen_spiral(int turns, double ppt, double K, double* out) {
    return guard([&] { auto s = gs::gen_spiral(turns, ppt, K); std::memcpy(out, s.coords.data(), s.coords.size() * 8); });
}
int orc_voronoi(int dim, long long M, const double* coords, double K, double* mu) {
    return guard([&] {
        gs::SamplingSet s;
        s.dim = dim;
        s.coords.assign(coords, coords + M * dim);
        auto v = gs::voronoi_weights(s, K);
        std::memcpy(mu, v.mu.data(), v.mu.size() * 8);
    });
}
int orc_voronoi_fast(int dim, long long M, const double* coords, double K, double* mu, int) {
    return orc_voronoi(dim, M, coords, K, mu);  // the reference has one (O(M^2)) routine
}
int orc_scaling_dyadic(int p, int R, double* out, long long* len, long long* support_begin) {
    return guard([&] {
        gs::FunctionTable t = gs::evaluate_scaling_dyadic(gs::ScalingFamily::make(family_of(p)), R);
        *len = static_cast<long long>(t.values.size());
        *support_begin = t.support_begin;
        if (out) std::memcpy(out, t.values.data(), t.values.size() * 8);
    });
}
int orc_boundary_dyadic(int p, int left, int R, int k, double* out, long long* len, long long* support_begin) {
    return guard([&] {
        auto tabs = gs::evaluate_boundary_dyadic(gs::ScalingFamily::make(family_of(p)), side_of(left), R);
        if (k < 0 || k >= static_cast<int>(tabs.size())) throw gs::DomainError("edge function index out of range");
        const gs::FunctionTable& t = tabs[static_cast<size_t>(k)];
        *len = static_cast<long long>(t.values.size());
        *support_begin = t.support_begin;
        if (out) std::memcpy(out, t.values.data(), t.values.size() * 8);
    });
}
int orc_weval(int dim, int p, int J, int R, const double* coeffs, long long ncoeffs, double* out) {
    return guard([&] {
        if (dim != 1 && dim != 2) throw gs::DomainError("dim must be 1 or 2");
        std::vector<double> c(coeffs, coeffs + ncoeffs);
        gs::ScalingFamily f = gs::ScalingFamily::make(family_of(p));
        auto ev = dim == 1 ? gs::weval_1d(c, f, J, R) : gs::weval_2d(c, f, J, R);
        std::memcpy(out, ev.values.data(), ev.values.size() * 8);
    });
}
double orc_wrap_half_open(double z) {  // freq2wave.cpp:15-19 keeps it file-local; not reachable
    (void)z;
    return __builtin_nan("");
}

}  // extern "C"
