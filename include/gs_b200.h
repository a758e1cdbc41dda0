/*
 * gs_b200.h -- C-ABI of the B200-native generalized-sampling hot path:
 * the change-of-basis operator T (Fourier samples <- boundary-corrected
 * Daubechies / Haar scaling coefficients), its adjoint T*, and the CGLS
 * least-squares loop that applies them, all resident on one sm_100a GPU.
 *
 * This is the drop-in boundary for the reference C++ API (namespace gs,
 * /root/reference/proj).  Every entry point names the reference interface it
 * replaces.  Plain pointers and sizes only; complex vectors are interleaved
 * (re, im) float64, layout-identical to std::complex<double> / double2.
 * Vector arguments may be host or device pointers (cudaPointerGetAttributes
 * decides); host buffers are staged through pinned memory inside the call.
 *
 * Return codes mirror gs::ErrorClass (include/gs/error.hpp:9-15):
 *   0 ok, 2 usage (null handle / bad argument), 4 shape, 5 domain,
 *   6 numerical, 7 CUDA runtime failure (no GPU, launch error, OOM).
 * The message of the last failure on the calling thread is gs_last_error().
 * A C++ wrapper rethrows the matching gs::Error subclass.
 */
#ifndef GS_B200_H
#define GS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_OK 0
#define GS_ERR_USAGE 2
#define GS_ERR_SHAPE 4
#define GS_ERR_DOMAIN 5
#define GS_ERR_NUMERICAL 6
#define GS_ERR_CUDA 7

/* Route the operator took (freq2wave.cpp:170-191 plus the new exact tensor route). */
#define GS_ROUTE_UNIFORM_1D 1  /* exact zero-embedded DFT (uniform_ndft_fft)       */
#define GS_ROUTE_NFFT_1D 2     /* Kaiser-Bessel gridding NFFT, 1D                   */
#define GS_ROUTE_NFFT_2D 3     /* 2D KB-NFFT + 4p side NFFTs + corners (9 blocks)   */
#define GS_ROUTE_TENSOR_2D 4   /* exact: T = T_x (x) T_y on a uniform tensor grid   */
#define GS_ROUTE_NDFT_1D 5     /* exact: direct NDFT core (ndft_forward, a14), 1D   */

typedef struct gs_op gs_op; /* opaque; replaces gs::Freq2WaveOp (freq2wave.hpp:32-55) */

/* Construction description: gs::freq2wave(SamplingSet, Family, J, Freq2WaveOptions)
 * (freq2wave.hpp:12-24, 57-58).  `batch` >= 1 independent problems of equal
 * shape (dim, family, J, M) share one handle; their coords / weights arrays
 * are concatenated problem-major. */
typedef struct {
  int dim;                 /* 1 or 2 (SamplingSet::dim)                           */
  int family_p;            /* 1 = haar, 2..8 = db2..db8 (Family; p vanishing mom.) */
  int J;                   /* scale, n = 2^J coefficients per axis                 */
  int64_t M;               /* samples per problem                                  */
  int batch;               /* number of independent problems (>= 1)                */
  const double* coords;    /* [batch][M][dim] point-major (x, y) host pointer      */
  const double* weights;   /* [batch][M] Voronoi mu (NOT sqrt), or NULL            */
  double bandwidth;        /* |xi| <= bandwidth accepted; NaN = none               */
  double sigma;            /* NFFT oversampling (default 2)                        */
  int w;                   /* KB half-width (default 6)                            */
  int boundary_depth;      /* default 30                                           */
  int product_terms;       /* default 48                                           */
  int allow_uniform_fast_path; /* default 1                                        */
  int allow_tensor_route;  /* default 0; 1: exact tensor route for uniform 2D grids */
  int device;              /* CUDA ordinal                                         */
  int exact_ndft;          /* default 0; 1: 1D non-uniform samples use the direct  */
                           /* NDFT (exact, O(M N), FP64 pipe) instead of the KB NFFT */
} gs_op_desc;

typedef struct {
  int dim, family_p, J, batch, route;
  int64_t rows;            /* M  (Freq2WaveOp::rows)                               */
  int64_t cols;            /* N_c = n or n^2 (Freq2WaveOp::cols)                   */
  int uniform_fast;        /* Freq2WaveOp::uniform_fast (1D)                        */
  double uniform_epsilon;  /* Freq2WaveOp::uniform_epsilon                         */
  int weighted;            /* Freq2WaveOp::weighted()                              */
  int n_over;              /* NFFT oversampled length per axis (0 on exact routes) */
  int64_t device_bytes;    /* HBM held by the handle                               */
} gs_op_info_t;

typedef struct {
  int iterations;          /* SolveStats::iterations (solver.hpp:16-22)            */
  double residual;         /* SolveStats::residual                                 */
  int converged;           /* SolveStats::converged                                */
} gs_solve_stats;

/* gs::freq2wave (freq2wave.cpp:86-193): validates, builds the factors
 * D, L, R, the KB tables and the sorted sample bins ON THE DEVICE. */
int gs_op_create(const gs_op_desc* desc, gs_op** out);
int gs_op_destroy(gs_op* op);
int gs_op_info(const gs_op* op, gs_op_info_t* info);

/* gs::apply_forward (freq2wave.cpp:215-303): samples[b] = T_b coeffs[b].
 * coeffs [batch][cols], samples [batch][rows]. `stream` is a cudaStream_t or NULL. */
int gs_apply_forward(gs_op* op, const double* coeffs, int64_t coeffs_len,
                     double* samples, void* stream);

/* gs::apply_adjoint (freq2wave.cpp:305-387): coeffs[b] = T_b^* samples[b]. */
int gs_apply_adjoint(gs_op* op, const double* samples, int64_t samples_len,
                     double* coeffs, void* stream);

/* gs::solve_least_squares (solver.cpp:19-91), CGNR resident on the GPU.
 * raw_samples [batch][rows] (weighted ops take RAW data; sqrt(mu) applied here),
 * x0 [batch][cols] or NULL, max_iterations <= 0 -> 2*cols, tolerance > 0.
 * x_out [batch][cols]; stats [batch]; history [batch][max_iter+1] or NULL
 * (entries past stats.iterations are undefined). */
int gs_solve_least_squares(gs_op* op, const double* raw_samples, int64_t samples_len,
                           const double* x0, int max_iterations, double tolerance,
                           double* x_out, gs_solve_stats* stats, double* history,
                           void* stream);

/* Split CGLS for warm restarts and benchmarking (same algorithm as
 * gs_solve_least_squares): begin = preamble (solver.cpp:28-68, 2 adjoints +
 * 1 forward), step = `iterations` loop bodies (solver.cpp:70-88) enqueued on
 * `stream` with no host synchronisation (converged problems freeze on the
 * device), active = host poll of the device flags, finish = x / stats / history.
 * `*out` is write-only (a new session; NULL on failure).  history_capacity
 * >= 1 is the row stride of `history` in gs_cgls_finish; iterations past it
 * overwrite the last slot.
 * Threading: calls on one handle are serialised by the handle, and a handle's
 * workspaces are shared, so use one handle from one stream at a time (one
 * handle per concurrent stream; handles are independent). */
typedef struct gs_cgls_session gs_cgls_session;
int gs_cgls_begin(gs_op* op, const double* raw_samples, int64_t samples_len, const double* x0,
                  double tolerance, int history_capacity, void* stream, gs_cgls_session** out);
int gs_cgls_step(gs_cgls_session* s, int iterations, void* stream);
int gs_cgls_active(gs_cgls_session* s, void* stream, int* any_active);
int gs_cgls_finish(gs_cgls_session* s, double* x_out, gs_solve_stats* stats, double* history,
                   void* stream);
int gs_cgls_destroy(gs_cgls_session* s);

/* Sample-sharded CGLS over several GPUs (the C4 row): each rank
 * builds an operator from ITS contiguous slice of the samples (rows of T);
 * coefficient vectors stay replicated; per iteration the library sums
 * ||q||^2 (B doubles) and the adjoint partials T_g* r_g (B x cols complex)
 * over the ranks with NCCL on `stream` -- no host round trip.  The
 * communicator wraps an NCCL communicator (libnccl.so.2, opened on first
 * use): rank 0 makes a unique id, every rank calls gs_comm_init with it.
 * gs_cgls_step / active / finish / destroy work on sharded sessions too;
 * all ranks must call them in the same order (they stay in lockstep). */
#define GS_COMM_ID_BYTES 128
typedef struct gs_comm gs_comm;
int gs_comm_unique_id(unsigned char* id);
int gs_comm_init(int nranks, int rank, const unsigned char* id, int device, gs_comm** out);
int gs_comm_destroy(gs_comm* comm);
int gs_cgls_begin_sharded(gs_op* op, gs_comm* comm, const double* raw_samples, int64_t samples_len,
                          const double* x0, double tolerance, int history_capacity, void* stream,
                          gs_cgls_session** out);
int gs_solve_least_squares_sharded(gs_op* op, gs_comm* comm, const double* raw_samples, int64_t samples_len,
                                   const double* x0, int max_iterations, double tolerance, double* x_out,
                                   gs_solve_stats* stats, double* history, void* stream);

/* Host copies of the per-axis factors of problem `b` in the reference layout
 * (Freq2WaveOp::Dx/Dy, Lx/Rx/Ly/Ry col-major M x p, freq2wave.hpp:42-43);
 * axis 0 = x, 1 = y.  L, R may be NULL (haar). */
int gs_op_export_factors(gs_op* op, int b, int axis, double* D, double* L, double* R);

/* gs::ndft_forward / gs::ndft_adjoint (nufft.cpp:74-132, nufft.hpp:25-33):
 * the direct O(M prod N) transform on the device (blocked complex-exponential
 * kernel).  N[0] (1D) or N[0], N[1] (2D) modes k = -N/2..N/2-1 per axis, last
 * axis fastest; points [M][dim] scaled to [-1/2, 1/2) (DomainError outside);
 * grid [prod N], samples [M].  Host or device pointers. */
int gs_ndft_forward(int dim, const int* N, const double* points, int64_t M, const double* grid,
                    int64_t grid_len, double* samples, void* stream);
int gs_ndft_adjoint(int dim, const int* N, const double* points, int64_t M, const double* samples,
                    int64_t samples_len, double* grid, void* stream);

/* gs::NfftPlan / plan_nfft / nfft_forward / nfft_adjoint (nufft.hpp:36-70,
 * nufft.cpp:138-365): the Kaiser-Bessel plan on the device at any dim 1/2,
 * even N per axis, sigma >= 1.25 and half-width w >= 2 (general-length FFT
 * engine), same validation and error classes as the reference constructor.
 * points [M][dim] scaled to [-1/2, 1/2); grid [N0 (* N1)], last axis fastest. */
typedef struct gs_nfft_plan gs_nfft_plan;
int gs_nfft_plan_create(int dim, const int* N, const double* points, int64_t M, double sigma, int w,
                        int device, gs_nfft_plan** out);
int gs_nfft_plan_forward(gs_nfft_plan* plan, const double* grid, int64_t grid_len, double* samples,
                         void* stream);
int gs_nfft_plan_adjoint(gs_nfft_plan* plan, const double* samples, int64_t samples_len, double* grid,
                         void* stream);
/* dim, points_count, grid_size, oversampled_length(axis) for axis 0, 1 (NfftPlan accessors) */
int gs_nfft_plan_info(const gs_nfft_plan* plan, int* dim, int64_t* points, int64_t* grid_size, int* n_over);
int gs_nfft_plan_destroy(gs_nfft_plan* plan);

/* gs::uniform_ndft_fft / uniform_ndft_adjoint_fft (nufft.cpp:383-459): the
 * exact NDFT on xi_m = (eps/N)(m - M/2) through one zero-embedded DFT of any
 * length q N / eps.  forward: x [x_len <= N] -> out [M]; adjoint: samples [M]
 * -> out [N]. */
int gs_uniform_ndft_fft(const double* x, int64_t x_len, int64_t M, double epsilon, int64_t N, double* out,
                        void* stream);
int gs_uniform_ndft_adjoint_fft(const double* samples, int64_t M, double epsilon, int64_t N, double* out,
                                void* stream);

/* Family data and transforms (scaling.hpp / fourier.hpp; scaling.cpp:29-75,
 * fourier.cpp:34-130).  taps [2p] (filter_coefficients, k = -p+1..p);
 * boundary filters of one side (left != 0): H [p*p], h [p*(2p-1)] (columns
 * m = p..3p-2), integer values [p*2p], row-major, any pointer may be NULL;
 * v [p] = boundary_fourier_at_zero.  The evaluations run on the device: out
 * [n] complex (scaling) or [n][p] complex (boundary transforms at xi[i]). */
int gs_family_filter(int family_p, double* taps);
int gs_boundary_filter_set(int family_p, int left, double* H, double* h, double* integer_values);
int gs_boundary_at_zero(int family_p, int left, double* v);
int gs_fourier_scaling_eval(int family_p, int64_t n, const double* xi, int terms, double* out, void* stream);
int gs_fourier_boundary_eval(int family_p, int left, int64_t n, const double* xi, int depth, int terms,
                             double* out, void* stream);

/* gs::densify (freq2wave.cpp:389-450): the dense M x cols section assembled
 * on the device from the transform formulas (column-major like
 * Eigen::MatrixXcd); coords [M][dim] natural frequencies, sqrt_weights [M]
 * or NULL; DomainError past entry_cap entries. */
int gs_densify(int dim, int family_p, int J, int64_t M, const double* coords, const double* sqrt_weights,
               int64_t entry_cap, double* out, void* stream);

/* Per-kernel device time of one T + T* pair (no reference counterpart; the
 * measurement hook bench.py uses for the roofline): `reps` pairs on live data
 * (seeded pseudo-random coefficients x, y = T x), CUDA events between
 * consecutive launches on `stream`.  Writes up to max_kernels average
 * durations (ms) and 32-byte kernel names. */
int gs_profile_pair(gs_op* op, int reps, void* stream, int max_kernels, double* ms_out,
                    char* names_out, int* count);

/* 1 when the handle's 2D gridding kernels run the balanced band schedule (the
 * sampling pattern loads the 3-row bands of its tiles unevenly, e.g. a
 * spiral), 0 for the static one; no reference counterpart (diagnostic). */
int gs_op_balanced_schedule(const gs_op* op);

/* Dyadic-grid evaluation (dyadic.hpp:27-64; front-end row SURVEY 8(f)4).
 * Tables of the interior scaling function / of edge function k of one side
 * at resolution R (evaluate_scaling_dyadic, evaluate_boundary_dyadic):
 * values[i] = phi(support_begin + i / 2^R); values == NULL -> sizes only.
 * gs_weval = weval_1d (dim 1, 2^J real coefficients, 2^R + 1 outputs) or
 * weval_2d (dim 2, 4^J coefficients x-fastest, (2^R + 1)^2 outputs, row =
 * y).  Buffers are host or device pointers. */
int gs_scaling_dyadic(int family_p, int R, double* values, int64_t* len, int64_t* support_begin, void* stream);
int gs_boundary_dyadic(int family_p, int left, int R, int k, double* values, int64_t* len, int64_t* support_begin,
                       void* stream);
int gs_weval(int dim, int family_p, int J, int R, const double* coeffs, int64_t coeffs_len, double* out,
             void* stream);

/* Input harness (reference patterns.cpp generators, exact fast Voronoi
 * weights with weights.cpp semantics); host-only, not on the timed path. */
int gs_gen_grid(int64_t M, double eps, int dim, double* out);
int gs_gen_jitter(int64_t M, double eps, double eta, uint64_t seed, int dim, double* out);
int gs_gen_spiral(int turns, double points_per_turn, double K, double* out);
int gs_voronoi_weights(int dim, int64_t M, const double* coords, double K, double* mu, int nthreads);
/* voronoi_weights on the GPU: 2D cells one thread each, the
 * host routine's arithmetic without FMA contraction -> bit-identical mu;
 * dim 1 falls back to the host.  coords / mu host pointers. */
int gs_voronoi_weights_gpu(int dim, int64_t M, const double* coords, double K, double* mu, int device,
                           void* stream);
/* density(samples, K).delta_raw (weights.cpp:135-176; replaces gs::density) */
int gs_density(int dim, int64_t M, const double* coords, double K, double* delta_raw, int nthreads);
/* bench harness right-hand side: n seeded coefficients, interleaved re,im
 * (bench.cpp:30-36 seeded_coefficients) */
int gs_seeded_coefficients(int64_t n, uint64_t seed, double* out);
/* truncated-cosine test signal at 1D frequencies (signals.cpp:27-37) */
int gs_truncated_cosine(int64_t M, const double* xi, double* out);
const char* gs_inputs_last_error(void);

const char* gs_last_error(void);

/* Number of kernels this library has launched so far (process-wide counter). */
long long gs_launch_count(void);

/* Build / capability probe: returns the sm version the library was compiled
 * for (100 for sm_100a) -- loadable without a GPU. */
int gs_build_arch(void);

#ifdef __cplusplus
}
#endif
#endif /* GS_B200_H */
