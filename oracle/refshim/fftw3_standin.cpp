// FFTW stand-in for the oracle/_ref build (see fftw3.h).  TEST INFRASTRUCTURE ONLY.
//
// Power-of-two lengths: bit-reversal + radix-2 butterflies, twiddles from one
// table computed in long double.  Other lengths: recursive decimation in time
// over the prime factors with table twiddles (O(n * sum of factors)).
// Rank 2 is row-major (n[1] fastest), rows first, then columns through a
// contiguous scratch line.  Execution keeps no shared mutable state, so
// concurrent fftw_execute_dft calls on one plan are safe (as with FFTW's
// new-array interface).
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

namespace {
using cd = std::complex<double>;

struct Axis {
    int n = 1;
    bool pow2 = false;
    std::vector<cd> tw;        // exp(sign * 2 pi i k / n), k < n
    std::vector<int> factors;  // prime factors, ascending
    std::vector<int> rev;      // bit reversal (power of two)
    void init(int len, int sign) {
        n = len;
        tw.resize(static_cast<size_t>(n));
        const long double step = 2.0L * 3.141592653589793238462643383279502884L / n;
        for (int k = 0; k < n; ++k) {
            long double a = step * k;
            tw[static_cast<size_t>(k)] = cd(static_cast<double>(std::cos(a)), static_cast<double>(sign * std::sin(a)));
        }
        pow2 = n > 0 && (n & (n - 1)) == 0;
        if (pow2) {
            rev.resize(static_cast<size_t>(n));
            int bits = 0;
            while ((1 << bits) < n) ++bits;
            for (int i = 0; i < n; ++i) {
                int r = 0;
                for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
                rev[static_cast<size_t>(i)] = r;
            }
        } else {
            int m = n;
            for (int f = 2; f * f <= m; ++f)
                while (m % f == 0) factors.push_back(f), m /= f;
            if (m > 1) factors.push_back(m);
        }
    }
    // out[0..n) = DFT of in[0], in[is], in[2 is] ...  (out contiguous, distinct from in)
    void run(const cd* in, long is, cd* out, cd* scratch) const {
        if (pow2) {
            for (int i = 0; i < n; ++i) out[rev[static_cast<size_t>(i)]] = in[static_cast<long>(i) * is];
            auto mul = [](const cd& a, const cd& b) {  // plain complex product (finite operands)
                return cd(a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real());
            };
            int half = 1;
            if (n >= 2) {  // first stage: twiddle 1
                for (int base = 0; base < n; base += 2) {
                    const cd u = out[base], t = out[base + 1];
                    out[base] = u + t;
                    out[base + 1] = u - t;
                }
                half = 2;
            }
            for (; half < n; half <<= 1) {
                const int stride = n / (2 * half);
                for (int base = 0; base < n; base += 2 * half) {
                    cd* lo = out + base;
                    cd* hi = lo + half;
                    for (int k = 0; k < half; ++k) {
                        const cd t = mul(hi[k], tw[static_cast<size_t>(k * stride)]);
                        const cd u = lo[k];
                        lo[k] = u + t;
                        hi[k] = u - t;
                    }
                }
            }
        } else {
            rec(in, is, out, scratch, n, 0);
        }
    }
    void rec(const cd* in, long is, cd* out, cd* scratch, int len, size_t fi) const {
        if (len == 1) {
            out[0] = in[0];
            return;
        }
        const int r = factors[fi], m = len / r, tstride = n / len;
        for (int q = 0; q < r; ++q) rec(in + q * is, is * r, out + q * m, scratch, m, fi + 1);
        // combine: X[k + j m] = sum_q w_len^{q (k + j m)} Y_q[k]
        for (int k = 0; k < m; ++k) {
            for (int q = 0; q < r; ++q) scratch[q] = out[q * m + k] * tw[static_cast<size_t>((static_cast<long>(q) * k % len) * tstride)];
            for (int j = 0; j < r; ++j) {
                cd acc = scratch[0];
                for (int q = 1; q < r; ++q)
                    acc += scratch[q] * tw[static_cast<size_t>((static_cast<long>(q) * j * m % len) * tstride)];
                scratch[r + j] = acc;
            }
            for (int j = 0; j < r; ++j) out[j * m + k] = scratch[r + j];
        }
    }
};

// Twiddle / bit-reversal tables are kept per (length, sign) for the life of the
// process, as FFTW keeps its own twiddle caches across plans: the reference plans
// the uniform reductions anew on every call (nufft.cpp:410, 440).
std::shared_ptr<const Axis> axis_for(int n, int sign) {
    static std::mutex mu;
    static std::map<std::pair<int, int>, std::shared_ptr<const Axis>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto& slot = cache[{n, sign}];
    if (!slot) {
        auto a = std::make_shared<Axis>();
        a->init(n, sign);
        slot = a;
    }
    return slot;
}
}  // namespace

struct fftw_standin_plan {
    int rank = 1;
    std::shared_ptr<const Axis> ax[2];
};

extern "C" {

fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex*, fftw_complex*, int sign, unsigned) {
    if (rank < 1 || rank > 2) return nullptr;
    auto* p = new fftw_standin_plan;
    p->rank = rank;
    for (int a = 0; a < rank; ++a) p->ax[a] = axis_for(n[a], sign < 0 ? -1 : 1);
    return p;
}

void fftw_execute_dft(const fftw_plan p, fftw_complex* in_, fftw_complex* out_) {
    const cd* in = reinterpret_cast<const cd*>(in_);
    cd* out = reinterpret_cast<cd*>(out_);
    // per-thread work buffers, grown on demand (no allocation per transform)
    thread_local std::vector<cd> line, res, scratch;
    if (p->rank == 1) {
        const int n = p->ax[0]->n;
        if (!p->ax[0]->pow2 && scratch.size() < static_cast<size_t>(2 * n + 2)) scratch.resize(static_cast<size_t>(2 * n + 2));
        if (in == out) {
            if (line.size() < static_cast<size_t>(n)) line.resize(static_cast<size_t>(n));
            std::memcpy(static_cast<void*>(line.data()), static_cast<const void*>(in), sizeof(cd) * static_cast<size_t>(n));
            p->ax[0]->run(line.data(), 1, out, scratch.data());
        } else {
            p->ax[0]->run(in, 1, out, scratch.data());
        }
        return;
    }
    const int n0 = p->ax[0]->n, n1 = p->ax[1]->n;
    const size_t nm = static_cast<size_t>(std::max(n0, n1));
    if (line.size() < nm) line.resize(nm);
    if (res.size() < nm) res.resize(nm);
    if (scratch.size() < 2 * nm + 2) scratch.resize(2 * nm + 2);
    for (int i = 0; i < n0; ++i) {  // rows (contiguous)
        std::memcpy(static_cast<void*>(line.data()), static_cast<const void*>(in + static_cast<size_t>(i) * n1),
                    sizeof(cd) * static_cast<size_t>(n1));
        p->ax[1]->run(line.data(), 1, out + static_cast<size_t>(i) * n1, scratch.data());
    }
    for (int j = 0; j < n1; ++j) {  // columns
        for (int i = 0; i < n0; ++i) line[static_cast<size_t>(i)] = out[static_cast<size_t>(i) * n1 + j];
        p->ax[0]->run(line.data(), 1, res.data(), scratch.data());
        for (int i = 0; i < n0; ++i) out[static_cast<size_t>(i) * n1 + j] = res[static_cast<size_t>(i)];
    }
}

void fftw_destroy_plan(fftw_plan p) { delete p; }

}  // extern "C"
