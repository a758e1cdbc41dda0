// kernels_nfft2d_fast.cuh -- sm_100a fast path of the 2D route for the default
// Kaiser-Bessel window (w = 6, S = 13 taps) and p <= 4 (haar .. db4):
//
//  * samples are bin-sorted by 12x12 grid tile and, inside a tile, by cell
//    (row-major); the work list is (tile, chunk of <= F_CHUNK samples) so dense
//    tiles (the spiral's centre) split across CTAs;
//  * k2f_interp  -- one CTA per chunk stages the tile's (T+12)^2 grid region,
//    its 2 x 2p side-line segments and the 4 p x p corner blocks in shared
//    memory once, then one thread per work unit (a pair of neighbouring
//    samples of one cell row, or a single sample) interpolates from shared
//    memory, loading each row window once for both samples
//    (nufft.cpp:287-303 + freq2wave.cpp:255-301);
//  * k2f_spread  -- output-stationary in registers: lane c < 24 owns grid
//    column c, lanes 24..31 own the 2p y-lines, and warp w owns the band of
//    F_BAND sample rows of the tile, so its accumulators span F_BAND + 12 rows
//    (plus the 2p x-line entries at column c).  Every rank-1 update has a
//    compile-time row offset, the sample pairs are software-pipelined, and the
//    4 warps' bands are folded once per chunk and written with no atomics
//    (transpose of the interpolation, nufft.cpp:324-338 + freq2wave.cpp:332-385).
#pragma once
#include <type_traits>
#include "kernels_nfft.cuh"

#define F_S 13
#define F_T 12
#define F_R 24
#ifndef F_CHUNK
// samples per work item (chunks of a tile are staged in shared memory): one
// sample per grid cell fills a 12 x 12 tile exactly, and 144 keeps a spreading
// CTA's staging under 75 KB so 3 of them fit an SM (C5: 160 -> 144 took the
// spreading from 12.2 to 10.1 ms per 256 problems)
#define F_CHUNK 144
#endif

// cooperative 16-byte copy of [src, src + bytes) global -> shared; the copy starts
// at the aligned address below src, the returned pointer is src's image
// (asynchronous: cp.async 16-B copies, completed by f_stage_wait + __syncthreads)
__device__ __forceinline__ unsigned char* f_stage(unsigned char* dst, const void* src, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src), al = a & ~uintptr_t(15);
  const size_t off = a - al, n = (off + bytes + 15) / 16;
  const char* s = reinterpret_cast<const char*>(al);
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  for (size_t i = threadIdx.x; i < n; i += blockDim.x)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + (unsigned)(16 * i)), "l"(s + 16 * i)
                 : "memory");
  return dst + off;
}
__device__ __forceinline__ void f_stage_wait() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// single asynchronous 8-B / 16-B global -> shared copies (cp.async group; f_stage_wait completes them)
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<unsigned>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { f_stage_wait(); }

// L2 prefetch (cp.async.bulk.prefetch) of [src, src + bytes) rounded out to 16 B
__device__ __forceinline__ void l2_prefetch(const void* src, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src), al = a & ~uintptr_t(15);
  const unsigned n = (unsigned)((a - al + bytes + 15) & ~size_t(15));
  if (n) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(al), "r"(n) : "memory");
}
// Chunks are dispatched in (problem, chunk) order, about F_PF at a time: a CTA
// prefetches into L2 the per-sample streams of the chunk F_PF places after its
// own, so that chunk's TMA staging hits L2 instead of waiting on HBM.
// (measured on C5: +2% for the spreading, -2% for the interpolation, whose
// staging is mostly the L2-resident grid region)
#ifndef F_PF_SPREAD
#define F_PF_SPREAD 296
#endif
#ifndef F_PF_INTERP
#define F_PF_INTERP 0
#endif
template <int RR, int F_PF>
__device__ __forceinline__ void prefetch_chunk_ahead(int prob, int c, int cap, int B, int M, const int* __restrict__ ch_s0,
                                                     const int* __restrict__ ch_s1, const int* __restrict__ base_x,
                                                     const int* __restrict__ base_y, const double* __restrict__ wx_all,
                                                     const double* __restrict__ wy_all, const cplx* __restrict__ recx_all,
                                                     const cplx* __restrict__ recy_all, const cplx* __restrict__ ys) {
  const int64_t lin = (int64_t)prob * cap + c + F_PF;
  if (F_PF <= 0 || lin >= (int64_t)B * cap) return;
  const int p2 = (int)(lin / cap);
  const int a = ch_s0[lin], n = ch_s1[lin] - a;
  if (n <= 0) return;
  const int64_t g = (int64_t)p2 * M + a;
  l2_prefetch(wy_all + g * F_S, sizeof(double) * F_S * n);
  l2_prefetch(wx_all + g * F_S, sizeof(double) * F_S * n);
  l2_prefetch(recx_all + g * RR, sizeof(cplx) * RR * n);
  l2_prefetch(recy_all + g * RR, sizeof(cplx) * RR * n);
  l2_prefetch(base_x + g, sizeof(int) * n);
  l2_prefetch(base_y + g, sizeof(int) * n);
  if (ys) l2_prefetch(ys + g, sizeof(cplx) * n);
}

// TMA bulk staging (cp.async.bulk, one issuing thread, completion on an
// mbarrier): copy [src, src + bytes) rounded out to 16-B boundaries into dst;
// returns src's image in shared memory and adds the copied bytes to *tx.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ unsigned bulk_bytes(const void* src, size_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src), al = a & ~uintptr_t(15);
  return (unsigned)((a - al + bytes + 15) & ~size_t(15));
}
__device__ __forceinline__ unsigned char* bulk_stage(unsigned char* dst, const void* src, size_t bytes, uint64_t* bar) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src), al = a & ~uintptr_t(15);
  const unsigned n = (unsigned)((a - al + bytes + 15) & ~size_t(15));
  if (n)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(al), "r"(n), "r"(smem_u32(bar))
                 : "memory");
  return dst + (a - al);
}

// Row starts of every chunk (built once per operator): byte r of ch_rows[chunk]
// = first sample (relative to the chunk start) whose window row is >= tile
// row r, r = 0..F_T (samples are sorted by cell, row-major, inside a tile).
// Bytes 13-14: the balanced schedule's warps per band (3 bits each, see
// f_band_schedule); bal[0] / bal[1] accumulate the chunks' longest static band
// and longest balanced warp run (in K steps of 4 samples) -- the operator uses
// the balanced kernels when the static bands are measurably uneven.
__global__ void k2f_chunk_rows(const int* __restrict__ ch_tile, const int* __restrict__ ch_s0,
                               const int* __restrict__ ch_s1, const int* __restrict__ ch_count, int64_t nchunks,
                               int cap, int64_t M, int nt, const int* __restrict__ base_y, uint4* __restrict__ ch_rows,
                               unsigned long long* __restrict__ bal) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nchunks) return;
  const int prob = (int)(q / cap), a = ch_s0[q], n = ch_s1[q] - a;
  const bool live = (int)(q - (int64_t)prob * cap) < ch_count[prob];
  const int ty0 = (ch_tile[q] / nt) * F_T;
  const int* by = base_y + (int64_t)prob * M + a;
  unsigned char r8[16] = {0};
  for (int r = 0; r <= F_T; ++r) {
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (by[mid] < ty0 + r) lo = mid + 1;
      else hi = mid;
    }
    r8[r] = (unsigned char)lo;
  }
  // warps per band: one per non-empty band, the spare ones to the band with the most steps per warp
  constexpr int NW = 4, BAND = F_T / NW;
  int steps[NW], nw[NW], used = 0, smax = 0;
  for (int b = 0; b < NW; ++b) {
    steps[b] = (r8[(b + 1) * BAND] - r8[b * BAND] + 3) / 4;
    nw[b] = steps[b] > 0 ? 1 : 0;
    used += nw[b];
    smax = steps[b] > smax ? steps[b] : smax;
  }
  for (int k = used; k < NW && used > 0; ++k) {
    int best = 0, load = -1;
    for (int b = 0; b < NW; ++b) {
      const int l = nw[b] > 0 ? (steps[b] + nw[b] - 1) / nw[b] : -1;
      if (l > load) load = l, best = b;
    }
    ++nw[best];
  }
  if (used == 0)
    for (int b = 0; b < NW; ++b) nw[b] = 1;
  int bmax = 0;
  for (int b = 0; b < NW; ++b) {
    const int l = nw[b] > 0 ? (steps[b] + nw[b] - 1) / nw[b] : 0;
    bmax = l > bmax ? l : bmax;
  }
  const unsigned code = (unsigned)nw[0] | ((unsigned)nw[1] << 3) | ((unsigned)nw[2] << 6) | ((unsigned)nw[3] << 9);
  r8[13] = (unsigned char)(code & 0xffu);
  r8[14] = (unsigned char)(code >> 8);
  ch_rows[q] = *reinterpret_cast<const uint4*>(r8);
  if (live && bal) {
    atomicAdd(bal, (unsigned long long)smax);
    atomicAdd(bal + 1, (unsigned long long)bmax);
  }
}
__device__ __forceinline__ int row_start(const uint4& rw, int r) {
  const unsigned w = r < 4 ? rw.x : (r < 8 ? rw.y : (r < 12 ? rw.z : rw.w));
  return (int)((w >> (8 * (r & 3))) & 0xffu);
}

// Balanced band schedule of the DMMA kernels (template flag BAL).  A tile's
// samples are sorted band-major (NW bands of BAND cell rows); statically warp w
// takes band w, which idles warps whenever a sampling pattern loads the bands
// unevenly (a spiral arm crossing a tile sits in one or two bands: C4's longest
// band holds 1.55x the mean).  In the balanced schedule every non-empty band
// gets one warp and the spare warps go, one at a time, to the band with the
// most K steps per warp (decided once per chunk by k2f_chunk_rows, bytes 13-14
// of ch_rows); a band's warps take equal contiguous runs of its steps (STEP
// samples each).  Any warp's samples still lie in ONE band, so its accumulator
// window (band rows + 12) is unchanged; the chunk fold sums the warp records by
// band.  The operator picks the balanced kernels only when its static bands
// are uneven (gs_capi.cu), so evenly loaded patterns (C5's jittered grid) keep
// the static kernels.  wb[w] = band of warp w; [sa, sb) = this warp's samples.
template <int NW, int BAND, int STEP, bool BAL>
__device__ __forceinline__ void f_band_schedule(const uint4& rw, int warp, int (&wb)[NW], int& sa, int& sb) {
  static_assert(NW == 4, "warps-per-band code of k2f_chunk_rows is for 4 bands");
  sa = sb = 0;
  if (!BAL) {
#pragma unroll
    for (int b = 0; b < NW; ++b) {
      wb[b] = b;
      if (b == warp) sa = row_start(rw, b * BAND), sb = row_start(rw, (b + 1) * BAND);
    }
    return;
  }
  const unsigned code = (rw.w >> 8) & 0xfffu;  // bytes 13-14
  int off = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) wb[w] = w;  // (a live chunk's code always covers all NW warps)
#pragma unroll
  for (int b = 0; b < NW; ++b) {
    const int nwb = (int)((code >> (3 * b)) & 7u);
    const int s0 = row_start(rw, b * BAND), s1 = row_start(rw, (b + 1) * BAND);
#pragma unroll
    for (int w = 0; w < NW; ++w)
      if (w >= off && w < off + nwb) wb[w] = b;
    if (warp >= off && warp < off + nwb) {
      const int steps = (s1 - s0 + STEP - 1) / STEP;
      const int per = (steps + nwb - 1) / nwb * STEP;
      const int a = s0 + (warp - off) * per;
      sa = a < s1 ? a : s1;
      sb = a + per < s1 ? a + per : s1;
    }
    off += nwb;
  }
}

// Debug-only CTA timeline (build with -DF_TIMELINE): per chunk, the SM id and
// SM clock at entry, staging complete, compute complete (tools/timeline.py).
#ifdef F_TIMELINE
#define F_TL_MAX (1 << 16)
__device__ unsigned long long g_tl[F_TL_MAX][5];  // entry, staged, computed, SM id, exit
__device__ __forceinline__ void tl_stamp(int64_t lin, int k) {
  if (threadIdx.x == 0 && lin < F_TL_MAX) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_tl[lin][k] = (unsigned long long)clock64();
    if (k == 0) g_tl[lin][3] = smid;
  }
}
// F_TIMELINE=1 (or bare -DF_TIMELINE): the interpolation records; 2: the spreading
#if F_TIMELINE + 0 == 2
#define F_TLS(k) tl_stamp((int64_t)prob * cap + c, k)
#define F_TLS_SYNC() __syncthreads()
#define F_TL(k)
#define F_TL_SYNC()
#else
#define F_TL(k) tl_stamp(chunk, k)
#define F_TL_SYNC() __syncthreads()
#define F_TLS(k)
#define F_TLS_SYNC()
#endif
#else
#define F_TL(k)
#define F_TL_SYNC()
#define F_TLS(k)
#define F_TLS_SYNC()
#endif

// ------------------------------------------------------------------ interpolation
// Work units of the interpolation: a chunk's samples are walked in sorted order
// and consecutive samples in the same cell row whose columns differ by at most
// F_PD are fused into one unit, so the unit loads each grid row / side-line
// window once (F_W = 13 + F_PD entries) for both samples.  Everything else is a
// single-sample unit (second slot 0xffff).  Built once per operator; units of
// chunk (prob, c) are stored from the chunk's first sample index on.
#define F_PD 3
#define F_W (F_S + F_PD)
// Shared-memory column map of the staged region and x-lines: column c lives at
// f(c) = c + c/2.  Unit windows start at even columns ws in {0, 2, .., 8}, so
// f(ws + j) = f(ws) + f(j) (constant offsets per tap) and f(ws) mod 8 =
// {0, 3, 6, 1, 4} puts the quarter-warp's windows in distinct 16-B bank groups;
// the row stride 39 (= 7 mod 8) keeps the next cell row's windows apart too.
#define F_RS2 39
// interpolation CTA shape (measured on C5: 4 warps x 3 CTAs/SM beat 3 x 4 and
// 2 x 4; the factor records are read through L1, which a larger shared-memory
// carve-out would shrink)
#ifndef F_ITHREADS
#define F_ITHREADS 128
#define F_IBLOCKS 3
#endif
#ifndef F_IUNROLL
#define F_IUNROLL 2  // unroll of the interpolation row / line loops
#endif
__host__ __device__ constexpr int f_col(int c) { return c + (c >> 1); }

__global__ void k2f_build_units(const int* __restrict__ ch_tile, const int* __restrict__ ch_s0,
                                const int* __restrict__ ch_s1, const int* __restrict__ ch_count, int cap, int B, int M, int nt,
                                const int* __restrict__ base_x, const int* __restrict__ base_y,
                                unsigned* __restrict__ units, int* __restrict__ ucount) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)B * cap) return;
  const int prob = (int)(i / cap), c = (int)(i - (int64_t)prob * cap);
  if (c >= ch_count[prob]) {
    ucount[i] = 0;
    return;
  }
  const int s0 = ch_s0[i], s1 = ch_s1[i];
  const int tx0 = (ch_tile[i] % nt) * F_T;
  const int64_t g0 = (int64_t)prob * M;
  unsigned* U = units + g0 + s0;
  int k = 0;
  for (int s = s0; s < s1; ++k) {
    const int by = base_y[g0 + s], bx = base_x[g0 + s];
    // window start of the unit: even column, at most R - W (see f_col)
    const int ws = min((bx - tx0) & ~1, F_R - F_W) + tx0;
    if (s + 1 < s1 && base_y[g0 + s + 1] == by && base_x[g0 + s + 1] >= bx && base_x[g0 + s + 1] - ws <= F_PD) {
      U[k] = (unsigned)(s - s0) | ((unsigned)(s + 1 - s0) << 16);
      s += 2;
    } else {
      U[k] = (unsigned)(s - s0) | (0xffffu << 16);
      s += 1;
    }
  }
  ucount[i] = k;
}

// dynamic shared memory of k2f_interp: the chunk's staged weights and records
template <int P>
struct FInterp {
  static constexpr int RR = 1 + (P >= 2 ? 2 * P : 0);
  static constexpr size_t WY = 0;
  static constexpr size_t WX = WY + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t RX = WX + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t RY = RX + sizeof(cplx) * F_CHUNK * RR + 16;
  static constexpr size_t bytes() { return RX; }  // records are read through L1 (RX, RY: unused)
};

template <int P>
__global__ void __launch_bounds__(F_ITHREADS, F_IBLOCKS) k2f_interp(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0,
                                                     const int* __restrict__ ch_s1, const int* __restrict__ ch_count,
                                                     int cap, const unsigned* __restrict__ units,
                                                     const int* __restrict__ ucount, const int* __restrict__ base_x,
                                                     const int* __restrict__ base_y, const double* __restrict__ wx_all,
                                                     const double* __restrict__ wy_all, const cplx* __restrict__ recx_all,
                                                     const cplx* __restrict__ recy_all, const cplx* __restrict__ G,
                                                     const cplx* __restrict__ lines, const cplx* __restrict__ x,
                                                     const int* __restrict__ out_perm, cplx* __restrict__ y) {
  constexpr int S = F_S, T = F_T, R = F_R, W = F_W, IU = F_IUNROLL;
  constexpr int E = P >= 2 ? 2 * P : 0;
  constexpr int EE = E > 0 ? E : 1;
  constexpr int RR = 1 + E;
  constexpr int NC = P >= 2 ? 4 * P * P : 1;
  constexpr int RS = F_RS2;  // row stride of the column-mapped region (f_col)
  constexpr int LX = f_col(R - 1) + 1;
  __shared__ cplx reg[R * RS];
  __shared__ cplx ly[EE][R];
  __shared__ cplx lx[EE][LX];
  __shared__ cplx cx[NC];
  const int prob = blockIdx.y, c = blockIdx.x;
  if (c >= ch_count[prob]) return;
  const int64_t chunk = (int64_t)prob * cap + c;
  const int tile = ch_tile[chunk], s0 = ch_s0[chunk], s1 = ch_s1[chunk];
  const int ty = tile / Pp.nt, tx = tile - ty * Pp.nt;
  const int n_ov = Pp.n_ov, mask = n_ov - 1, n = Pp.n;
  const cplx* g = G + (int64_t)prob * n_ov * n_ov;
  // asynchronous 16-B copies (cp.async): all of the tile's staging is in flight at once
  auto cp16 = [](cplx* dst, const cplx* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                     static_cast<unsigned>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
  };
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
    const int r = i / R, cc = i - r * R;
    cp16(reg + r * RS + f_col(cc), g + (int64_t)((ty * T + r) & mask) * n_ov + ((tx * T + cc) & mask));
  }
  if (E > 0) {
    const cplx* LY = lines + (int64_t)prob * 2 * E * n_ov;
    const cplx* LX = LY + (int64_t)E * n_ov;
    for (int i = threadIdx.x; i < E * R; i += blockDim.x) {
      const int e = i / R, r = i - e * R;
      cp16(&ly[e][r], LY + (int64_t)e * n_ov + ((ty * T + r) & mask));
      cp16(&lx[e][f_col(r)], LX + (int64_t)e * n_ov + ((tx * T + r) & mask));
    }
    const cplx* X = x + (int64_t)prob * n * n;
    for (int q = threadIdx.x; q < 4 * P * P; q += blockDim.x) {
      const int k = q / (P * P), rem = q - k * P * P, i = rem / P, j = rem - i * P;
      const int row0 = (k < 2) ? 0 : n - P, col0 = (k % 2 == 0) ? 0 : n - P;
      cp16(cx + q, X + (int64_t)(col0 + j) * n + row0 + i);
    }
  }
  // the chunk's window weights (contiguous ranges, staged 16-B aligned-down;
  // layout FInterp<P>)
  const int64_t g0 = (int64_t)prob * Pp.M + s0;
  const int nn = s1 - s0;
  extern __shared__ __align__(16) unsigned char fi_dyn[];
  using FI = FInterp<P>;
  const double* wys = reinterpret_cast<const double*>(f_stage(fi_dyn + FI::WY, wy_all + g0 * S, sizeof(double) * S * nn));
  const double* wxs = reinterpret_cast<const double*>(f_stage(fi_dyn + FI::WX, wx_all + g0 * S, sizeof(double) * S * nn));
  f_stage_wait();
  __syncthreads();
  const unsigned* U = units + g0;
  const int nu = ucount[chunk];
  for (int k = threadIdx.x; k < nu; k += blockDim.x) {
    const unsigned uv = U[k];
    const int la = (int)(uv & 0xffffu), lr = (int)(uv >> 16);
    const bool two = lr != 0xffff;
    const int lb = two ? lr : la;
    const int64_t ga = g0 + la, gb = g0 + lb;
    const int oy = base_y[ga] - ty * T;
    const int oxa = base_x[ga] - tx * T, oxb = base_x[gb] - tx * T;
    const int ws = min(oxa & ~1, R - W);  // shared even column window [ws, ws + W) inside the region
    const int da = oxa - ws, db = oxb - ws;
    // column taps of both samples on the shared window (zero outside each sample's support)
    double wa[W], wb[W];
    const double* wxa = wxs + la * S;
    const double* wxb = wxs + lb * S;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const int ja = j - da, jb = j - db;
      const double va = wxa[ja < 0 ? 0 : (ja >= S ? S - 1 : ja)];
      const double vb = wxb[jb < 0 ? 0 : (jb >= S ? S - 1 : jb)];
      wa[j] = (ja >= 0 && ja < S) ? va : 0.0;
      wb[j] = (two && jb >= 0 && jb < S) ? vb : 0.0;
    }
    const double* wya = wys + la * S;
    const double* wyb = wys + lb * S;
    const cplx* rxa = recx_all + ga * RR;
    const cplx* rxb = recx_all + gb * RR;
    const cplx* rya = recy_all + ga * RR;
    const cplx* ryb = recy_all + gb * RR;
    // out = Dx Dy acc + Dx (b . ux) + a^T (C b + Dy uy): interior (freq2wave.cpp:255),
    // the 4 corner blocks C (260-270) and both side families (272-301), with
    // a = [Lx|Rx](m,:), b = [Ly|Ry](m,:)
    cplx outa, outb;
    {
      cplx acca = mk(0, 0), accb = mk(0, 0);
#pragma unroll IU
      for (int t0 = 0; t0 < S; ++t0) {
        const cplx* row = reg + (oy + t0) * RS + f_col(ws);
        cplx ra[2] = {mk(0, 0), mk(0, 0)}, rb[2] = {mk(0, 0), mk(0, 0)};  // even / odd taps: shorter chains
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const cplx v = row[f_col(j)];
          ra[j & 1] = caxpy(ra[j & 1], wa[j], v);
          rb[j & 1] = caxpy(rb[j & 1], wb[j], v);
        }
        acca = caxpy(acca, wya[t0], cadd(ra[0], ra[1]));
        accb = caxpy(accb, wyb[t0], cadd(rb[0], rb[1]));
      }
      const cplx Dxa = ldg2(rxa), Dxb = ldg2(rxb);
      outa = cmul(cmul(Dxa, ldg2(rya)), acca);
      outb = cmul(cmul(Dxb, ldg2(ryb)), accb);
      if (E > 0) {
        cplx sxa = mk(0, 0), sxb = mk(0, 0);
#pragma unroll IU
        for (int e = 0; e < E; ++e) {
          cplx ua[2] = {mk(0, 0), mk(0, 0)}, ub[2] = {mk(0, 0), mk(0, 0)};
#pragma unroll
          for (int j = 0; j < W; ++j) {
            const cplx v = lx[e][f_col(ws) + f_col(j)];
            ua[j & 1] = caxpy(ua[j & 1], wa[j], v);
            ub[j & 1] = caxpy(ub[j & 1], wb[j], v);
          }
          sxa = cadd(sxa, cmul(ldg2(rya + 1 + e), cadd(ua[0], ua[1])));
          sxb = cadd(sxb, cmul(ldg2(ryb + 1 + e), cadd(ub[0], ub[1])));
        }
        outa = cadd(outa, cmul(Dxa, sxa));
        outb = cadd(outb, cmul(Dxb, sxb));
      }
    }
    if (E > 0) {
      // side y-lines: Dy sum_i a_i uy_i, both samples sharing the line loads
      // (freq2wave.cpp:287-301)
      double ta[S], tb[S];
#pragma unroll
      for (int t = 0; t < S; ++t) {
        ta[t] = wya[t];
        tb[t] = wyb[t];
      }
      cplx sya = mk(0, 0), syb = mk(0, 0);
#pragma unroll IU
      for (int i = 0; i < E; ++i) {
        cplx ua[2] = {mk(0, 0), mk(0, 0)}, ub[2] = {mk(0, 0), mk(0, 0)};
#pragma unroll
        for (int t = 0; t < S; ++t) {
          const cplx v = ly[i][oy + t];
          ua[t & 1] = caxpy(ua[t & 1], ta[t], v);
          ub[t & 1] = caxpy(ub[t & 1], tb[t], v);
        }
        sya = cadd(sya, cmul(ldg2(rxa + 1 + i), cadd(ua[0], ua[1])));
        syb = cadd(syb, cmul(ldg2(rxb + 1 + i), cadd(ub[0], ub[1])));
      }
      outa = cadd(outa, cmul(ldg2(rya), sya));
      outb = cadd(outb, cmul(ldg2(ryb), syb));
      // corners a^T C b of both samples, each C entry loaded once (freq2wave.cpp:260-270)
      cplx bva[EE], bvb[EE];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        bva[e] = ldg2(rya + 1 + e);
        bvb[e] = ldg2(ryb + 1 + e);
      }
      cplx oa = mk(0, 0), ob = mk(0, 0);
#pragma unroll 1
      for (int i = 0; i < E; ++i) {
        const int hi = i < P ? 0 : 1, ii = i - hi * P;
        cplx va = mk(0, 0), vb = mk(0, 0);
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int hj = j < P ? 0 : 1, jj = j - hj * P;
          const cplx cc = cx[(2 * hi + hj) * P * P + ii * P + jj];
          va = cadd(va, cmul(cc, bva[j]));
          vb = cadd(vb, cmul(cc, bvb[j]));
        }
        oa = cadd(oa, cmul(ldg2(rxa + 1 + i), va));
        ob = cadd(ob, cmul(ldg2(rxb + 1 + i), vb));
      }
      outa = cadd(outa, oa);
      outb = cadd(outb, ob);
    }
    const int64_t base = (int64_t)prob * Pp.M;
    y[base + (out_perm ? (int64_t)out_perm[ga] : (int64_t)(s0 + la))] = outa;
    if (two) y[base + (out_perm ? (int64_t)out_perm[gb] : (int64_t)(s0 + lb))] = outb;
  }
}

// ------------------------------------------------------------------ spreading
#ifndef F_WARPS
#define F_WARPS 4
#endif
#define F_BAND (F_T / F_WARPS)   // sample rows of a tile per warp
#define F_AR (F_BAND - 1 + F_S)  // accumulator rows a warp's band touches

// compile-time loop: f(integral_constant<int, K>) for K in [K0, N)
template <int K0, int N, class Fn>
__device__ __forceinline__ void f_static_for(Fn&& f) {
  if constexpr (K0 < N) {
    f(std::integral_constant<int, K0>{});
    f_static_for<K0 + 1, N>(f);
  }
}

template <int P>
struct FSpread {
  static constexpr int E = P >= 2 ? 2 * P : 0;
  static constexpr int EE = E > 0 ? E : 1;
  static constexpr int RR = 1 + E;
  static constexpr int NCE = P >= 2 ? 4 * P * P : 0;
  static constexpr int NCU = NCE > 0 ? (NCE + 31) / 32 : 1;
  // per-warp fold record: band region + band of the y-lines + x-lines
  static constexpr int PER_WARP = F_AR * F_R + E * F_AR + E * F_R;
  // staged chunk (structure of arrays, in sample order)
  // each staged array gets 16 B of slack: copies start at the 16-B-aligned address below
  static constexpr size_t STG_WY = 0;
  static constexpr size_t STG_WX = STG_WY + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t STG_RX = STG_WX + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t STG_RY = STG_RX + sizeof(cplx) * F_CHUNK * RR + 16;
  static constexpr size_t STG_YS = STG_RY + sizeof(cplx) * F_CHUNK * RR + 16;
  static constexpr size_t STG_OX = STG_YS + sizeof(cplx) * F_CHUNK;
  static constexpr size_t STG_BY = STG_OX + sizeof(int) * F_CHUNK + 16;  // raw window origins (DMMA kernel)
  static constexpr size_t STG_END = STG_BY + sizeof(int) * F_CHUNK + 16;
  static constexpr size_t FOLD = sizeof(cplx) * (F_WARPS * PER_WARP + F_WARPS * (NCE > 0 ? NCE : 1));
  static constexpr size_t MAIN = (STG_END > FOLD ? STG_END : FOLD);  // fold buffer aliases the staging
  struct Scratch {  // derived per-sample values of one sample pair, shared inside a warp
    cplx d[2][32];
    double2 wy[16];  // row taps of the two samples, packed (wy_a[t], wy_b[t])
  };
  // two scratch buffers per warp: the next pair is derived while the current one updates
  static constexpr size_t bytes() { return (MAIN + 15) / 16 * 16 + sizeof(Scratch) * 2 * F_WARPS; }
};

// acc[OY + t] += w[t].x u0 + w[t].y u1, t < 13 (w = the two samples' row taps,
// packed pairwise), with OY a compile-time row offset inside the warp's band
template <int OY>
__device__ __forceinline__ void f_upd(cplx (&acc)[F_AR], cplx u0, cplx u1, const double2* w) {
#pragma unroll
  for (int t = 0; t < F_S; ++t) {
    const double2 ww = w[t];
    acc[OY + t].x = fma(ww.y, u1.x, fma(ww.x, u0.x, acc[OY + t].x));
    acc[OY + t].y = fma(ww.y, u1.y, fma(ww.x, u0.y, acc[OY + t].y));
  }
}


// Warp w owns the F_BAND sample rows [w F_BAND, (w+1) F_BAND) of the tile, so its
// register accumulators span only F_AR rows and every row offset is a
// compile-time constant (one specialised loop per band row, no dispatch).  Pairs
// of samples are software-pipelined: the next pair's derived values are loaded
// and multiplied while the current pair's rank-1 updates issue.
template <int P>
__global__ void __launch_bounds__(32 * F_WARPS, 2)
k2f_spread(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0, const int* __restrict__ ch_s1,
           const int* __restrict__ ch_count, int cap, const int* __restrict__ base_x, const int* __restrict__ base_y,
           const double* __restrict__ wx_all, const double* __restrict__ wy_all, const cplx* __restrict__ recx_all,
           const cplx* __restrict__ recy_all, const cplx* __restrict__ yin, const int* __restrict__ in_perm,
           cplx* __restrict__ TB, cplx* __restrict__ TL, cplx* __restrict__ TC) {
  using F = FSpread<P>;
  using Scr = typename F::Scratch;
  constexpr int S = F_S, T = F_T, R = F_R, AR = F_AR, BAND = F_BAND, E = F::E, EE = F::EE, RR = F::RR,
                NCE = F::NCE, NCU = F::NCU;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  cplx* s_ys = reinterpret_cast<cplx*>(fsm_raw + F::STG_YS);
  int* s_ox = reinterpret_cast<int*>(fsm_raw + F::STG_OX);
  Scr* scr_all = reinterpret_cast<Scr*>(fsm_raw + (F::MAIN + 15) / 16 * 16);
  __shared__ int rs[T + 1];
  const int prob = blockIdx.y, c = blockIdx.x;
  if (c >= ch_count[prob]) return;
  const int tile = ch_tile[prob * cap + c], s0 = ch_s0[prob * cap + c], s1 = ch_s1[prob * cap + c];
  const int n = s1 - s0;
  const int ty = tile / Pp.nt, tx = tile - ty * Pp.nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t g0 = (int64_t)prob * Pp.M + s0;
  // ---- stage the chunk: weights, factor records, samples, column offsets
  const double* s_wy = reinterpret_cast<const double*>(f_stage(fsm_raw + F::STG_WY, wy_all + g0 * S, sizeof(double) * S * n));
  const double* s_wx = reinterpret_cast<const double*>(f_stage(fsm_raw + F::STG_WX, wx_all + g0 * S, sizeof(double) * S * n));
  const cplx* s_rx = reinterpret_cast<const cplx*>(f_stage(fsm_raw + F::STG_RX, recx_all + g0 * RR, sizeof(cplx) * RR * n));
  const cplx* s_ry = reinterpret_cast<const cplx*>(f_stage(fsm_raw + F::STG_RY, recy_all + g0 * RR, sizeof(cplx) * RR * n));
  __shared__ unsigned char s_oy[F_CHUNK];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t gs = g0 + i;
    s_ys[i] = ldg2(yin + (int64_t)prob * Pp.M + (in_perm ? (int64_t)in_perm[gs] : (int64_t)(s0 + i)));
    s_ox[i] = base_x[gs] - tx * T;
    s_oy[i] = (unsigned char)(base_y[gs] - ty * T);
  }
  f_stage_wait();
  __syncthreads();
  if (threadIdx.x <= T) {  // row starts (samples are sorted by cell, row-major, in a tile)
    const int key = threadIdx.x;
    int lo = 0, hi = n;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if ((int)s_oy[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    rs[threadIdx.x] = lo;
  }
  __syncthreads();
  Scr* cur = scr_all + 2 * warp;
  Scr* nxt = cur + 1;
  cplx acc[AR];
  cplx accx[EE];
  cplx cacc[NCU];
  int cqa[NCU], cqb[NCU];
#pragma unroll
  for (int r = 0; r < AR; ++r) acc[r] = mk(0, 0);
#pragma unroll
  for (int e = 0; e < EE; ++e) accx[e] = mk(0, 0);
#pragma unroll
  for (int uu = 0; uu < NCU; ++uu) {
    cacc[uu] = mk(0, 0);
    const int q = lane + 32 * uu;
    const int k = P >= 2 ? q / (P * P) : 0, rem = q - k * P * P, i = P >= 2 ? rem / P : 0, j = rem - i * P;
    cqa[uu] = ((k < 2) ? 0 : P) + i;          // index into ca[] (Lx | Rx columns)
    cqb[uu] = 1 + ((k % 2 == 0) ? 0 : P) + j;  // record index of the (Ly | Ry) column
  }
  const int ly = E > 0 ? ((lane >= R && lane - R < E) ? lane - R : 0) : 0;  // y-line lane
  // lane roles of the derived values: A from ry (lanes 0..7) or rx, record index
  // 1 + e (clamped to the family) or 0 (lane >= 24); B = Dx | 1 | Dy
  const int role_e = E > 0 ? ((lane & 7) < E ? (lane & 7) : E - 1) : 0;
  const bool role_a_y = lane < 8;
  const int role_idx = (lane < 24 && E > 0) ? 1 + role_e : 0;
  const int role_b = lane < 8 ? 0 : (lane < 16 ? 1 : 2);
  const cplx* base_a = (role_a_y ? s_ry : s_rx) + role_idx;  // per-lane record columns (branch-free loads)
  const cplx* base_b = role_b == 2 ? s_ry : s_rx;
  const bool b_one = role_b == 1;
  // derived per-sample values of the pair (i0, i1), one per lane, z = conj(A B) ys:
  //   lanes 0..7  vx_e = conj(By(m,e) Dx) y   (side_y_edge, freq2wave.cpp:376)
  //   lanes 8..15 ca_i = conj(Ax(m,i)) y      (corner rows, freq2wave.cpp:351)
  //   lanes 16..23 vy_e = conj(Ax(m,e) Dy) y  (side_x_edge, freq2wave.cpp:363)
  //   lane 24      v2  = conj(Dx Dy) y        (interior,    freq2wave.cpp:335)
  // plus this lane's column tap w1 of each sample and the pair's packed row taps.
  // The second amplitude is scaled by kb (0 for the odd tail, whose second slot
  // repeats the first sample).
  auto load_pair = [&](int i0, int i1, double kb, cplx (&dv)[2], double2& wyp, double (&w1)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = k ? i1 : i0;
      const cplx ys = k ? cscale(s_ys[i], kb) : s_ys[i];
      const cplx Av = base_a[i * RR];
      const cplx Bl = base_b[i * RR];
      const cplx Bv = b_one ? mk(1.0, 0.0) : Bl;
      dv[k] = cmul(conj_(cmul(Av, Bv)), ys);
      const int t1 = lane - s_ox[i];
      const bool colv = lane < R && t1 >= 0 && t1 < S;
      w1[k] = colv ? s_wx[i * S + (t1 < 0 ? 0 : (t1 >= S ? S - 1 : t1))] : 0.0;
    }
    const int tl = lane < S ? lane : 0;
    wyp = make_double2(s_wy[i0 * S + tl], s_wy[i1 * S + tl]);
  };
  auto store_pair = [&](Scr* sc, const cplx (&dv)[2], double2 wyp) {
    sc->d[0][lane] = dv[0];
    sc->d[1][lane] = dv[1];
    if (lane < S) sc->wy[lane] = wyp;
  };
  // update amplitude of this lane: column tap x interior value (region lanes) or
  // the y-line value (lanes 24..24+E)
  auto lane_u = [&](const Scr* sc, const double (&w1)[2], cplx (&u)[2]) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const cplx ug = cscale(sc->d[k][24], w1[k]);
      u[k] = lane < R ? ug : ((E > 0 && lane - R < E) ? sc->d[k][16 + ly] : mk(0, 0));
    }
  };
  auto band_row = [&](auto KC) {
    constexpr int k = decltype(KC)::value;
    const int oy = warp * BAND + k;
    const int a = rs[oy], b = rs[oy + 1];
    if (a >= b) return;
    cplx dv[2], u[2];
    double2 wyp;
    double w1[2], w1n[2];
    load_pair(a, a + 1 < b ? a + 1 : a, a + 1 < b ? 1.0 : 0.0, dv, wyp, w1);
    __syncwarp();  // previous readers of *cur are done
    store_pair(cur, dv, wyp);
    __syncwarp();
    lane_u(cur, w1, u);
    for (int s = a; s < b; s += 2) {
      const int sb = s + 1 < b ? s + 1 : s;
      const int sn = s + 2;  // next pair (indices clamped; unused past the row end)
      load_pair(sn < b ? sn : b - 1, sn + 1 < b ? sn + 1 : b - 1, sn + 1 < b ? 1.0 : 0.0, dv, wyp, w1n);
      f_upd<k>(acc, u[0], u[1], cur->wy);
      if (E > 0) {
#pragma unroll
        for (int e = 0; e < E; ++e) accx[e] = caxpy(caxpy(accx[e], w1[0], cur->d[0][e]), w1[1], cur->d[1][e]);
        const cplx* rya = s_ry + s * RR;
        const cplx* ryb = s_ry + sb * RR;
#pragma unroll
        for (int uu = 0; uu < NCU; ++uu)  // corners (freq2wave.cpp:349-353)
          if (lane + 32 * uu < NCE)
            cacc[uu] = cadd(cadd(cacc[uu], cmul(cur->d[0][8 + cqa[uu]], conj_(rya[cqb[uu]]))),
                            cmul(cur->d[1][8 + cqa[uu]], conj_(ryb[cqb[uu]])));
      }
      store_pair(nxt, dv, wyp);
      __syncwarp();
      lane_u(nxt, w1n, u);
      w1[0] = w1n[0];
      w1[1] = w1n[1];
      Scr* t = cur;
      cur = nxt;
      nxt = t;
    }
  };
  static_assert(BAND * F_WARPS == T, "the warps' bands tile the sample rows");
  f_static_for<0, BAND>(band_row);
  __syncthreads();  // the fold buffer aliases the staging area
  // dump the warp copies, fold, write this chunk's region / lines / corners once
  cplx* buf = reinterpret_cast<cplx*>(fsm_raw);  // [F_WARPS][PER_WARP]
  cplx* cbuf = buf + F_WARPS * F::PER_WARP;       // [F_WARPS][NCE]
  cplx* mine = buf + warp * F::PER_WARP;
  if (lane < R) {
#pragma unroll
    for (int r = 0; r < AR; ++r) mine[r * R + lane] = acc[r];
#pragma unroll
    for (int e = 0; e < E; ++e) mine[AR * R + E * AR + e * R + lane] = accx[e];
  } else if (lane - R < E) {
#pragma unroll
    for (int r = 0; r < AR; ++r) mine[AR * R + (lane - R) * AR + r] = acc[r];
  }
  if (NCE > 0) {
#pragma unroll
    for (int uu = 0; uu < NCU; ++uu) {
      const int q = lane + 32 * uu;
      if (q < NCE) cbuf[warp * NCE + q] = cacc[uu];
    }
  }
  __syncthreads();
  const int64_t chunk = (int64_t)prob * cap + c;
  cplx* tb = TB + chunk * R * R;
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
    const int r = i / R, cc = i - r * R;
    cplx a = mk(0, 0);
#pragma unroll
    for (int w = 0; w < F_WARPS; ++w) {
      const int rr = r - w * BAND;
      if (rr >= 0 && rr < AR) a = cadd(a, buf[w * F::PER_WARP + rr * R + cc]);
    }
    tb[i] = a;
  }
  if (E > 0) {
    cplx* tl = TL + chunk * 2 * E * R;  // [y-lines e][row] then [x-lines e][column]
    for (int i = threadIdx.x; i < E * R; i += blockDim.x) {
      const int e = i / R, r = i - e * R;
      cplx a = mk(0, 0), bx = mk(0, 0);
#pragma unroll
      for (int w = 0; w < F_WARPS; ++w) {
        const int rr = r - w * BAND;
        if (rr >= 0 && rr < AR) a = cadd(a, buf[w * F::PER_WARP + AR * R + e * AR + rr]);
        bx = cadd(bx, buf[w * F::PER_WARP + AR * R + E * AR + i]);
      }
      tl[i] = a;
      tl[E * R + i] = bx;
    }
    cplx* tc = TC + chunk * NCE;
    for (int q = threadIdx.x; q < NCE; q += blockDim.x) {
      cplx a = cbuf[q];
#pragma unroll
      for (int w = 1; w < F_WARPS; ++w) a = cadd(a, cbuf[w * NCE + q]);
      tc[q] = a;
    }
  }
}

// ------------------------------------------------------------------ spreading on the FP64 tensor cores
// k2f_spread_mma: the same chunk outputs as k2f_spread, computed as small
// real GEMMs over the chunk's samples with mma.sync m8n8k4 f64 (DMMA; B200's
// FP64 tensor rate equals its DFMA rate, but one DMMA does 256 FMAs, so the
// kernel issues ~8x fewer instructions than the lane-per-column form and
// needs no shared-memory broadcasts).  Warp w owns the sample rows
// [3w, 3w+3) of the tile (accumulator rows band0 .. band0+15); K = the warp's
// samples, 4 per step.  With thread (g, t) = (lane/4, lane%4) and s_t the
// step's t-th sample:
//   region  G(r, c)   += sum_s wy_s(r - oy_s) [wx_s(c - ox_s) v2_s]     A1 x B1  (re | im column halves)
//   y-lines LY(e, r)  += sum_s vy_e(s) wy_s(r - oy_s)                   [vy re; im] x A1^T
//   x-lines LX(e, c)  += sum_s vx_e(s) wx_s(c - ox_s)                   [vx re; im] x B3
//   corners P(i', j') += sum_s [ca re; im](i) [b re | im](j)            -> C = ca conj(b)
// with v2 = conj(Dx Dy) y, vx_e = conj(By_e Dx) y, ca_i = conj(Ax_i) y,
// vy_e = conj(Ax_e Dy) y (freq2wave.cpp:332-385).  The fragment values are
// gathered straight from the staged chunk: A1(r, s_t) and the B2 operand of
// the y-lines are the same register, B3 is the bare column tap.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
// m16n8k8: A 16 x 8 (a0 = (g, t), a1 = (g + 8, t), a2 = (g, t + 4), a3 = (g + 8, t + 4)),
// B 8 x 8 (b0 = (t, g), b1 = (t + 4, g)), C rows g (c0, c1) and g + 8 (c2, c3), columns 2t, 2t + 1
__device__ __forceinline__ void dmma1688(double& c0, double& c1, double& c2, double& c3, const double* a,
                                         const double* b) {
  asm("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3)
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}

// CTA of the DMMA spreading kernel: F_MSPLIT warps per band of F_BAND sample
// rows (they take alternate K steps of the band's samples), so 2 CTAs/SM hold
// 4 x F_MSPLIT warps per SMSP pair -- enough to keep the DMMA pipe fed
#ifndef F_MSPLIT
#define F_MSPLIT 1
#endif
#define F_MWARPS (F_WARPS * F_MSPLIT)
#ifndef F_MUNROLL
#define F_MUNROLL 2  // K steps per loop trip: the next step's fragments load under this step's DMMAs
#endif

#ifndef F_SA1V2
#define F_SA1V2 0
#endif
#ifndef F_SREC_GLOBAL
#define F_SREC_GLOBAL 0  // 1: factor records read from global (L2-prefetched), not staged in shared memory
#endif
template <int P>
struct FSpreadM {
  static constexpr int E = P >= 2 ? 2 * P : 0;
  // per-warp fold record: region 16 x 24 (complex), y-lines 8 x 16, x-lines 8 x 24 (complex), corner P 16 x 16 (real)
  // (rows of RP = F_R + 1 complex: the 8 row groups of a DMMA fragment store land in distinct banks)
  static constexpr int RP = F_R + 1;
  static constexpr int REG = 16 * RP, LYN = 8 * 17, LXN = 8 * RP, PN = 16 * 16 / 2;  // in complex units
  static constexpr int PER_WARP = REG + LYN + LXN + PN;
  static constexpr size_t FOLD = sizeof(cplx) * F_WARPS * PER_WARP;  // one record per band
  // staging (structure of arrays, sample order; 16 B of slack each); the factor
  // records only when F_SREC_GLOBAL is 0
  static constexpr int RR = FSpread<P>::RR;
  static constexpr size_t WY = 0;
  static constexpr size_t WX = WY + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t YS = WX + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t OX = YS + sizeof(cplx) * F_CHUNK;
  static constexpr size_t BY = OX + sizeof(int) * F_CHUNK + 16;
  static constexpr size_t RX = BY + sizeof(int) * F_CHUNK + 16;
  static constexpr size_t RY = RX + (F_SREC_GLOBAL ? 0 : sizeof(cplx) * F_CHUNK * RR + 16);
  static constexpr size_t STG_END = RY + (F_SREC_GLOBAL ? 0 : sizeof(cplx) * F_CHUNK * RR + 16);
  static constexpr size_t MAIN = (STG_END > FOLD ? STG_END : FOLD);
  static constexpr size_t bytes() { return (MAIN + 15) / 16 * 16; }
};

#ifndef F_DESC_HOIST
#define F_DESC_HOIST 0  // 1: chunk descriptor loads issued before the live-chunk test resolves (measured slower on C5: off)
#endif
#ifndef F_FOLD_UNROLL
#define F_FOLD_UNROLL 1  // chunk fold with compile-time trip counts (all of a thread's loads in flight)
#endif
#ifndef F_SBLOCKS
#define F_SBLOCKS 3  // resident spreading CTAs per SM the register budget is sized for (smem allows 3 at F_CHUNK 144)
#endif
template <int P, bool BAL>
__global__ void __launch_bounds__(32 * F_MWARPS, F_SBLOCKS)
k2f_spread_mma(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0, const int* __restrict__ ch_s1,
               const int* __restrict__ ch_count, const uint4* __restrict__ ch_rows, int cap, const int* __restrict__ base_x,
               const int* __restrict__ base_y, const double* __restrict__ wx_all, const double* __restrict__ wy_all,
               const cplx* __restrict__ recx_all, const cplx* __restrict__ recy_all, const cplx* __restrict__ yin,
               const int* __restrict__ in_perm, cplx* __restrict__ TB, cplx* __restrict__ TL, cplx* __restrict__ TC) {
  using F = FSpread<P>;
  using FM = FSpreadM<P>;
  constexpr int S = F_S, T = F_T, R = F_R, BAND = F_BAND, E = F::E, RR = F::RR, NCE = F::NCE, MU = F_MUNROLL;
  constexpr int RP = FM::RP;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  cplx* s_ys = reinterpret_cast<cplx*>(fsm_raw + FM::YS);
  const int prob = blockIdx.y, c = blockIdx.x;
  // descriptor loads issued with the live-chunk test, not behind it (one L2 round trip, not two)
#if F_DESC_HOIST == 2
  // dead work-list slots hold an empty sample range: no ch_count round trip before the descriptors
  const int tile = ch_tile[prob * cap + c], s0 = ch_s0[prob * cap + c], s1 = ch_s1[prob * cap + c];
  const uint4 rw = ch_rows[prob * cap + c];
  if (s1 <= s0) return;
#else
#if F_DESC_HOIST
  const int nlive = ch_count[prob];
#else
  if (c >= ch_count[prob]) return;
  constexpr int nlive = 0x7fffffff;
#endif
  const int tile = ch_tile[prob * cap + c], s0 = ch_s0[prob * cap + c], s1 = ch_s1[prob * cap + c];
  const uint4 rw = ch_rows[prob * cap + c];
  if (c >= nlive) return;
#endif
  F_TLS(0);
  const int n = s1 - s0;
  const int ty = tile / Pp.nt, tx = tile - ty * Pp.nt;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t g0 = (int64_t)prob * Pp.M + s0;
  // ---- stage the chunk: weights and factor records by TMA bulk copies (one
  // thread, mbarrier completion), samples and cell offsets by the threads
  __shared__ __align__(8) uint64_t stage_bar;
  const double* wy_src = wy_all + g0 * S;
  const double* wx_src = wx_all + g0 * S;
  const cplx* rx_src = recx_all + g0 * RR;
  const cplx* ry_src = recy_all + g0 * RR;
  const double* s_wy = reinterpret_cast<const double*>(fsm_raw + FM::WY + (reinterpret_cast<uintptr_t>(wy_src) & 15));
  const double* s_wx = reinterpret_cast<const double*>(fsm_raw + FM::WX + (reinterpret_cast<uintptr_t>(wx_src) & 15));
#if F_SREC_GLOBAL
  const cplx* s_rx = rx_src;
  const cplx* s_ry = ry_src;
#else
  const cplx* s_rx = reinterpret_cast<const cplx*>(fsm_raw + FM::RX + (reinterpret_cast<uintptr_t>(rx_src) & 15));
  const cplx* s_ry = reinterpret_cast<const cplx*>(fsm_raw + FM::RY + (reinterpret_cast<uintptr_t>(ry_src) & 15));
#endif
  // window origins and (sorted-order input) samples ride the same TMA transaction
  const cplx* ys_src = yin + g0;
  const int* s_bx = reinterpret_cast<const int*>(fsm_raw + FM::OX + (reinterpret_cast<uintptr_t>(base_x + g0) & 15));
  const int* s_by = reinterpret_cast<const int*>(fsm_raw + FM::BY + (reinterpret_cast<uintptr_t>(base_y + g0) & 15));
  if (threadIdx.x == 0) {
    bar_init(&stage_bar);
    bar_expect(&stage_bar, bulk_bytes(wy_src, sizeof(double) * S * n) + bulk_bytes(wx_src, sizeof(double) * S * n) +
                               (F_SREC_GLOBAL ? 0u : bulk_bytes(rx_src, sizeof(cplx) * RR * n) +
                                                         bulk_bytes(ry_src, sizeof(cplx) * RR * n)) +
                               bulk_bytes(base_x + g0, sizeof(int) * n) + bulk_bytes(base_y + g0, sizeof(int) * n) +
                               (in_perm ? 0u : bulk_bytes(ys_src, sizeof(cplx) * n)));
#if F_SREC_GLOBAL
    l2_prefetch(rx_src, sizeof(cplx) * RR * n);
    l2_prefetch(ry_src, sizeof(cplx) * RR * n);
#else
    bulk_stage(fsm_raw + FM::RX, rx_src, sizeof(cplx) * RR * n, &stage_bar);
    bulk_stage(fsm_raw + FM::RY, ry_src, sizeof(cplx) * RR * n, &stage_bar);
#endif
    bulk_stage(fsm_raw + FM::WY, wy_src, sizeof(double) * S * n, &stage_bar);
    bulk_stage(fsm_raw + FM::WX, wx_src, sizeof(double) * S * n, &stage_bar);
    bulk_stage(fsm_raw + FM::OX, base_x + g0, sizeof(int) * n, &stage_bar);
    bulk_stage(fsm_raw + FM::BY, base_y + g0, sizeof(int) * n, &stage_bar);
    if (!in_perm) bulk_stage(fsm_raw + FM::YS, ys_src, sizeof(cplx) * n, &stage_bar);
  }
  if (threadIdx.x == 32)
    prefetch_chunk_ahead<RR, F_PF_SPREAD>(prob, c, cap, gridDim.y, Pp.M, ch_s0, ch_s1, base_x, base_y, wx_all, wy_all,
                                          recx_all, recy_all, in_perm ? nullptr : yin);
  if (in_perm)  // caller-order input (public apply path): gather
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_ys[i] = ldg2(yin + (int64_t)prob * Pp.M + in_perm[g0 + i]);
  __syncthreads();  // barrier initialised, samples staged
  bar_wait(&stage_bar, 0);
  F_TLS(1);
  const int ty0 = ty * T, tx0 = tx * T;
#if F_MSPLIT == 1
  // balanced schedule: this warp's band and its run of the band's K steps (f_band_schedule)
  constexpr int half = 0;
  int wband[F_WARPS], sa, sb;
  f_band_schedule<F_WARPS, BAND, 4, BAL>(rw, warp, wband, sa, sb);
  const int band = warp;  // fold record of this warp
  int band0 = 0;
#pragma unroll
  for (int w = 0; w < F_WARPS; ++w)
    if (w == warp) band0 = wband[w] * BAND;
#else
  const int band = warp % F_WARPS, half = warp / F_WARPS;  // band of rows, K-step parity
  const int band0 = band * BAND;
  const int sa = row_start(rw, band0), sb = row_start(rw, band0 + BAND);  // precomputed band starts
  int wband[F_WARPS];
#pragma unroll
  for (int w = 0; w < F_WARPS; ++w) wband[w] = w;
#endif
  double rg[2][6][2], ly[2][2][2], lx[2][3][2], co[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 6; ++j) rg[i][j][0] = rg[i][j][1] = 0.0;
#pragma unroll
    for (int j = 0; j < 2; ++j) ly[i][j][0] = ly[i][j][1] = co[i][j][0] = co[i][j][1] = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) lx[i][j][0] = lx[i][j][1] = 0.0;
  }
#pragma unroll MU
  for (int k0 = sa + 4 * half; k0 < sb; k0 += 4 * F_MSPLIT) {
    const int sl = k0 + t;
    const bool valid = sl < sb;
    const int sc = valid ? sl : sa;
    // padded K slots get window offsets no tap reaches (all-zero operands)
    const int oy = valid ? s_by[sc] - ty0 : 64, ox = valid ? s_bx[sc] - tx0 : 64;
    double a1[2], b3[3];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int d = band0 + mt * 8 + g - oy;
      double v = 0.0;
      if ((unsigned)d < (unsigned)S) v = s_wy[sc * S + d];
      a1[mt] = v;
    }
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      const int d = nt * 8 + g - ox;
      double v = 0.0;
      if ((unsigned)d < (unsigned)S) v = s_wx[sc * S + d];
      b3[nt] = v;
    }
    const cplx* rx = s_rx + sc * RR;
    const cplx* ry = s_ry + sc * RR;
    const cplx yv = valid ? s_ys[sc] : mk(0, 0);  // padded K slots contribute nothing
    const cplx t1 = cmul(conj_(rx[0]), yv);  // conj(Dx) y
    const cplx Dy = ry[0];
    const cplx v2 = cmul(conj_(Dy), t1);     // conj(Dx Dy) y
    // column tiles the step's 4 samples do not reach are all-zero: skip them (warp-uniform vote)
    bool hit[3];
#pragma unroll
    for (int nt = 0; nt < 3; ++nt)  // integer window test (KB taps inside the window are >= 1): no FP64 compare
      hit[nt] = __any_sync(0xffffffffu, (unsigned)(nt * 8 + g - ox) < (unsigned)S);
#if F_SA1V2
    // the sample's factor conj(Dx Dy) y scales the row operand (2 x 2 products) instead of each reached column tile
    const double ar[2] = {a1[0] * v2.x, a1[1] * v2.x}, ai[2] = {a1[0] * v2.y, a1[1] * v2.y};
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      if (!hit[nt]) continue;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        dmma884(rg[mt][nt][0], rg[mt][nt][1], ar[mt], b3[nt]);
        dmma884(rg[mt][nt + 3][0], rg[mt][nt + 3][1], ai[mt], b3[nt]);
      }
    }
#else
#pragma unroll
    for (int nt = 0; nt < 3; ++nt) {
      if (!hit[nt]) continue;
      const double bre = b3[nt] * v2.x, bim = b3[nt] * v2.y;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        dmma884(rg[mt][nt][0], rg[mt][nt][1], a1[mt], bre);
        dmma884(rg[mt][nt + 3][0], rg[mt][nt + 3][1], a1[mt], bim);
      }
    }
#endif
    if (E > 0) {
      const bool ge = g < E;
      const cplx Ax = rx[1 + (ge ? g : 0)], By = ry[1 + (ge ? g : 0)];
      const cplx vx = ge ? cmul(conj_(By), t1) : mk(0, 0);  // conj(By_e Dx) y
      const cplx ca = ge ? cmul(conj_(Ax), yv) : mk(0, 0);  // conj(Ax_i) y
      const cplx vy = cmul(conj_(Dy), ca);                  // conj(Ax_e Dy) y
      const cplx bj = ge ? By : mk(0, 0);
      const double vyc[2] = {vy.x, vy.y}, vxc[2] = {vx.x, vx.y}, cac[2] = {ca.x, ca.y}, bjc[2] = {bj.x, bj.y};
#pragma unroll
      for (int mm = 0; mm < 2; ++mm) {
#pragma unroll
        for (int nn = 0; nn < 2; ++nn) {
          dmma884(ly[mm][nn][0], ly[mm][nn][1], vyc[mm], a1[nn]);
          dmma884(co[mm][nn][0], co[mm][nn][1], cac[mm], bjc[nn]);
        }
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
          if (hit[nt]) dmma884(lx[mm][nt][0], lx[mm][nt][1], vxc[mm], b3[nt]);
      }
    }
  }
  F_TLS_SYNC();
  F_TLS(2);
  __syncthreads();  // the fold buffer aliases the staging area
  cplx* buf = reinterpret_cast<cplx*>(fsm_raw);
  cplx* mine = buf + band * FM::PER_WARP;  // one record per band; the K-step halves add in turn
  cplx* mreg = mine;                 // [16][R]  band-relative rows
  cplx* mly = mine + FM::REG;        // [8][16]  y-line e, band-relative row
  cplx* mlx = mly + FM::LYN;         // [8][R]   x-line e, column
  double* mp = reinterpret_cast<double*>(mlx + FM::LXN);  // [16][16] corner products
#pragma unroll 1
  for (int h = 0; h < F_MSPLIT; ++h) {
    if (half == h) {
      const bool add = h > 0;
      auto put = [&](cplx* dst, cplx v) { *dst = add ? cadd(*dst, v) : v; };
      auto putd = [&](double* dst, double v) { *dst = add ? *dst + v : v; };
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j)
            put(&mreg[(mt * 8 + g) * RP + nt * 8 + 2 * t + j], mk(rg[mt][nt][j], rg[mt][nt + 3][j]));
      if (E > 0) {
#pragma unroll
        for (int nn = 0; nn < 2; ++nn)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            put(&mly[g * 17 + nn * 8 + 2 * t + j], mk(ly[0][nn][j], ly[1][nn][j]));
#pragma unroll
            for (int mm = 0; mm < 2; ++mm) putd(&mp[(mm * 8 + g) * 16 + nn * 8 + 2 * t + j], co[mm][nn][j]);
          }
#pragma unroll
        for (int nt = 0; nt < 3; ++nt)
#pragma unroll
          for (int j = 0; j < 2; ++j) put(&mlx[g * RP + nt * 8 + 2 * t + j], mk(lx[0][nt][j], lx[1][nt][j]));
      }
    }
    __syncthreads();
  }
  // chunk fold: every output sums the warp records that cover it, in warp order.  Trip counts
  // are compile-time (NT threads), so the loads of a thread's outputs are all in flight together.
  constexpr int NT = 32 * F_MWARPS;
  constexpr int FU_TB = F_FOLD_UNROLL ? (R * R + NT - 1) / NT : 1, FU_TL = F_FOLD_UNROLL ? (E * R + NT - 1) / NT + 1 : 1;
  const int64_t chunk = (int64_t)prob * cap + c;
  cplx* tb = TB + chunk * R * R;
#pragma unroll FU_TB
  for (int it = 0; it < (R * R + NT - 1) / NT; ++it) {
    const int i = it * NT + (int)threadIdx.x;
    if (i < R * R) {
      const int r = i / R, cc = i - r * R;
      cplx a = mk(0, 0);
#pragma unroll
      for (int w = 0; w < F_WARPS; ++w) {
        const int rr = r - wband[w] * BAND;
        if (rr >= 0 && rr < 16) a = cadd(a, buf[w * FM::PER_WARP + rr * RP + cc]);
      }
      tb[i] = a;
    }
  }
  if (E > 0) {
    cplx* tl = TL + chunk * 2 * E * R;  // [y-lines e][row] then [x-lines e][column]
#pragma unroll FU_TL
    for (int it = 0; it < (E * R + NT - 1) / NT; ++it) {
      const int i = it * NT + (int)threadIdx.x;
      if (i < E * R) {
        const int e = i / R, r = i - e * R;
        cplx a = mk(0, 0), bx = mk(0, 0);
#pragma unroll
        for (int w = 0; w < F_WARPS; ++w) {
          const cplx* wb = buf + w * FM::PER_WARP;
          const int rr = r - wband[w] * BAND;
          if (rr >= 0 && rr < 16) a = cadd(a, wb[FM::REG + e * 17 + rr]);
          bx = cadd(bx, wb[FM::REG + FM::LYN + e * RP + r]);
        }
        tl[i] = a;
        tl[E * R + i] = bx;
      }
    }
    cplx* tc = TC + chunk * NCE;
    for (int q = threadIdx.x; q < NCE; q += NT) {
      const int k = q / (P * P), rem = q - k * P * P, i = rem / P, j = rem - i * P;
      const int ip = (k < 2 ? 0 : P) + i, jp = (k % 2 == 0 ? 0 : P) + j;  // ca index (Lx | Rx), b index (Ly | Ry)
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int w = 0; w < F_WARPS; ++w) {
        const double* wp = reinterpret_cast<const double*>(buf + w * FM::PER_WARP + FM::REG + FM::LYN + FM::LXN);
        re += wp[ip * 16 + jp] + wp[(8 + ip) * 16 + 8 + jp];   // sum ca conj(b): Re = car br + cai bi
        im += wp[(8 + ip) * 16 + jp] - wp[ip * 16 + 8 + jp];   //                 Im = cai br - car bi
      }
      tc[q] = mk(re, im);
    }
  }
  F_TLS_SYNC();
  F_TLS(4);
}

// ------------------------------------------------------------------ interpolation on the FP64 tensor cores
// k2f_interp_mma: the forward 2D apply of a chunk as per-warp DMMA GEMMs.
// Warp w takes the samples of sample rows [3w, 3w+3) eight at a time (one
// sample per B column n = lane/4):
//   H  = [G_re; G_im; LX_re; LX_im](band rows / lines, 24 cols) x Wx   (48 x 8, K = 24 columns)
//   UY = [LY_re; LY_im](e, band rows) x Wy                              (16 x 8, K = 16 rows)
//   CB = [[C_re, -C_im]; [C_im, C_re]] x [b_re; b_im]                   (16 x 8, K = 16)
// with Wx(c, s) = wx_s(c - ox_s), Wy(r, s) = wy_s(r - oy_s), b_j = By_j(s).
// A lane then holds, for two samples, row g of every product and forms
//   Dx Dy sum_r wy(r) H_G(r) + Dx b_g ux_g + a_g (Dy uy_g + (C b)_g)
// (interior freq2wave.cpp:255, sides 272-301, corners 260-270); a three-step
// xor-shuffle over the 8 lanes of the sample finishes every sum.
#define F_GS 28  // row stride (doubles) of the split re / im region: 8 rows x 4 columns hit 32 banks
#ifndef F_IMUNROLL
#define F_IMUNROLL 8  // sample tiles per loop trip: a whole band in one trip (DMMAs of one tile overlap the epilogue of another)
#endif
#ifndef F_IMMA168
#define F_IMMA168 0  // 1: m16n8k8 DMMAs in the interpolation
#endif
#ifndef F_ICONST_RELOAD
#define F_ICONST_RELOAD 0
#endif
// DMMA interpolation CTA shape (measured on C5, 256 problems): 4 warps (bands
// of 3 sample rows), the factor records read from global memory after an L2
// prefetch instead of staged, so a CTA needs ~50 KB of shared memory and 4 CTAs
// (16 warps, 128 registers, a few spills) share an SM: 11.6 ms per apply,
// against 12.4 ms for 2 CTAs of 6 warps with staged records
#ifndef F_IREC_GLOBAL
#define F_IREC_GLOBAL 1  // 1: factor records read from global (L2-prefetched), not staged in shared memory
#endif
#ifndef F_IBLOCKS_M
#define F_IBLOCKS_M 4  // resident DMMA interpolation CTAs per SM the register budget is sized for
#endif
#ifndef F_IWARPS
#define F_IWARPS 4  // warps (bands of F_T / F_IWARPS sample rows) of the DMMA interpolation CTA
#endif
#ifndef F_IMSPLIT
#define F_IMSPLIT 1  // warps per band (alternate sample tiles)
#endif

template <int P>
struct FInterpM {
  static constexpr int RR = 1 + (P >= 2 ? 2 * P : 0);
  // dynamic shared memory: staged weights and factor records (TMA bulk), then the split region / lines
  static constexpr size_t WY = 0;
  static constexpr size_t WX = WY + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t RX = WX + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t RY = RX + (F_IREC_GLOBAL ? 0 : sizeof(cplx) * F_CHUNK * RR + 16);
  static constexpr size_t GRE = RY + (F_IREC_GLOBAL ? 0 : sizeof(cplx) * F_CHUNK * RR + 16);
  static constexpr size_t GIM = GRE + sizeof(double) * F_R * F_GS;
  static constexpr size_t LXRE = GIM + sizeof(double) * F_R * F_GS;
  static constexpr size_t LXIM = LXRE + sizeof(double) * 8 * F_GS;
  static constexpr size_t BX = LXIM + sizeof(double) * 8 * F_GS;  // raw window origins (TMA)
  static constexpr size_t BY = BX + sizeof(int) * F_CHUNK + 16;
  static constexpr size_t END = BY + sizeof(int) * F_CHUNK + 16;
  static constexpr size_t bytes() { return END; }
};

// The forward products of one band of a staged chunk (k2f_interp_mma and the
// persistent k2f_interp_pipe): sample tiles n0 = sa + 8 half, +8 SPLIT, ...
template <int P, int SPLIT>
__device__ __forceinline__ void f_interp_band(int band0, int half, int sa, int sb, int ty0, int tx0,
                                              const double* __restrict__ s_wx, const double* __restrict__ s_wy,
                                              const cplx* __restrict__ s_rx, const cplx* __restrict__ s_ry,
                                              const int* __restrict__ s_bx, const int* __restrict__ s_by,
                                              const double* __restrict__ gre, const double* __restrict__ gim,
                                              const double* __restrict__ lxre, const double* __restrict__ lxim,
                                              const cplx (*__restrict__ lys)[F_R], const cplx* __restrict__ cxs,
                                              int64_t ybase, int64_t g0, int s0, const int* __restrict__ out_perm,
                                              cplx* __restrict__ y) {
  constexpr int S = F_S, R = F_R, RR = 1 + (P >= 2 ? 2 * P : 0), IMU = F_IMUNROLL;
  constexpr int E = P >= 2 ? 2 * P : 0;
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  // constant A operands: y-lines [LY_re; LY_im](g, band0 + 4 ks + t), corner block matrix
  // (F_ICONST_RELOAD: re-read from shared memory at each use instead of held in 32 registers)
  auto ly_op = [&](int ks, double* out2) {
    const int row = band0 + ks * 4 + t;
    const cplx v = (E > 0 && g < E && row < R) ? lys[g < E ? g : 0][row < R ? row : 0] : mk(0, 0);
    out2[0] = v.x;
    out2[1] = v.y;
  };
  auto cr_op = [&](int ks, double* out2) {
    const int part = ks >> 1, j = (ks & 1) * 4 + t;
    cplx cij = mk(0, 0);
    if (E > 0 && g < E && j < E) {
      const int hi = g < P ? 0 : 1, ii = g - hi * P, hj = j < P ? 0 : 1, jj = j - hj * P;
      cij = cxs[(2 * hi + hj) * P * P + ii * P + jj];
    }
    out2[0] = part == 0 ? cij.x : -cij.y;
    out2[1] = part == 0 ? cij.y : cij.x;
  };
  double lyA[2][4], crA[2][4];
#pragma unroll
  for (int ks = 0; ks < (F_ICONST_RELOAD ? 0 : 4); ++ks) {
    const int row = band0 + ks * 4 + t;
    const cplx v = (E > 0 && g < E && row < R) ? lys[g < E ? g : 0][row < R ? row : 0] : mk(0, 0);
    lyA[0][ks] = v.x;
    lyA[1][ks] = v.y;
    const int part = ks >> 1, j = (ks & 1) * 4 + t;  // K index = (re | im part of b, j)
    cplx cij = mk(0, 0);
    if (E > 0 && g < E && j < E) {
      const int hi = g < P ? 0 : 1, ii = g - hi * P, hj = j < P ? 0 : 1, jj = j - hj * P;
      cij = cxs[(2 * hi + hj) * P * P + ii * P + jj];
    }
    crA[0][ks] = part == 0 ? cij.x : -cij.y;  // row block re:  C_re b_re - C_im b_im
    crA[1][ks] = part == 0 ? cij.y : cij.x;   // row block im:  C_im b_re + C_re b_im
  }
#pragma unroll IMU
  for (int n0 = sa + 8 * half; n0 < sb; n0 += 8 * SPLIT) {
    // B operands for sample column g
    const int sg = n0 + g;
    const bool vg = sg < sb;
    const int sgc = vg ? sg : sa;
    // padded sample slots get window offsets no tap reaches (all-zero B columns)
    const int oyg = vg ? s_by[sgc] - ty0 : 64, oxg = vg ? s_bx[sgc] - tx0 : 64;
    const double* wxg = s_wx + sgc * S;
    const double* wyg = s_wy + sgc * S;
    double wb[6], yb[4], cb[4];
#pragma unroll
    for (int ks = 0; ks < 6; ++ks) {
      const int d = ks * 4 + t - oxg;
      double v = 0.0;
      if ((unsigned)d < (unsigned)S) v = wxg[d];
      wb[ks] = v;
    }
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int d = band0 + ks * 4 + t - oyg;
      double v = 0.0;
      if ((unsigned)d < (unsigned)S) v = wyg[d];
      yb[ks] = v;
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int j = kk * 4 + t;
      cplx bj = mk(0, 0);
      if (E > 0 && vg && j < E) bj = s_ry[sgc * RR + 1 + j];
      cb[kk] = bj.x;
      cb[kk + 2] = bj.y;
    }
    // products
    double h[6][2], uy[2][2], cbo[2][2];
#pragma unroll
    for (int mt = 0; mt < 6; ++mt) h[mt][0] = h[mt][1] = 0.0;
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) uy[mt][0] = uy[mt][1] = cbo[mt][0] = cbo[mt][1] = 0.0;
#if F_IMMA168
    // m16n8k8 form: one instruction per 16 rows x 8 columns x 8 samples
    // (A = [re rows 0..15] or [im rows 0..15] or [LX_re; LX_im], K = 8 columns)
    bool hk8[3];
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) hk8[kb] = __any_sync(0xffffffffu, wb[2 * kb] != 0.0 || wb[2 * kb + 1] != 0.0);
#pragma unroll
    for (int kb = 0; kb < 3; ++kb) {
      if (!hk8[kb]) continue;
      const int col = kb * 8 + t;
      const int r0 = band0 + g, r1 = band0 + 8 + g;
      const double bb[2] = {wb[2 * kb], wb[2 * kb + 1]};
      {
        const double a[4] = {r0 < R ? gre[r0 * F_GS + col] : 0.0, r1 < R ? gre[r1 * F_GS + col] : 0.0,
                             r0 < R ? gre[r0 * F_GS + col + 4] : 0.0, r1 < R ? gre[r1 * F_GS + col + 4] : 0.0};
        dmma1688(h[0][0], h[0][1], h[1][0], h[1][1], a, bb);
      }
      {
        const double a[4] = {r0 < R ? gim[r0 * F_GS + col] : 0.0, r1 < R ? gim[r1 * F_GS + col] : 0.0,
                             r0 < R ? gim[r0 * F_GS + col + 4] : 0.0, r1 < R ? gim[r1 * F_GS + col + 4] : 0.0};
        dmma1688(h[2][0], h[2][1], h[3][0], h[3][1], a, bb);
      }
      if (E > 0) {
        const double a[4] = {lxre[g * F_GS + col], lxim[g * F_GS + col], lxre[g * F_GS + col + 4],
                             lxim[g * F_GS + col + 4]};
        dmma1688(h[4][0], h[4][1], h[5][0], h[5][1], a, bb);
      }
    }
    if (E > 0) {
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        const double bu[2] = {yb[2 * kb], yb[2 * kb + 1]}, bc[2] = {cb[2 * kb], cb[2 * kb + 1]};
        const double au[4] = {lyA[0][2 * kb], lyA[1][2 * kb], lyA[0][2 * kb + 1], lyA[1][2 * kb + 1]};
        const double ac[4] = {crA[0][2 * kb], crA[1][2 * kb], crA[0][2 * kb + 1], crA[1][2 * kb + 1]};
        dmma1688(uy[0][0], uy[0][1], uy[1][0], uy[1][1], au, bu);
        dmma1688(cbo[0][0], cbo[0][1], cbo[1][0], cbo[1][1], ac, bc);
      }
    }
#else
    // column blocks no sample of the tile reaches are all-zero: skip them (warp-uniform vote)
    bool hk[6];
#pragma unroll
    for (int ks = 0; ks < 6; ++ks)  // integer window test (KB taps inside the window are >= 1): no FP64 compare
      hk[ks] = __any_sync(0xffffffffu, (unsigned)(ks * 4 + t - oxg) < (unsigned)S);
#pragma unroll
    for (int ks = 0; ks < 6; ++ks) {
      if (!hk[ks]) continue;
      const int col = ks * 4 + t;
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double* src = mt < 2 ? gre : gim;
        const int row = band0 + (mt & 1) * 8 + g;
        const double a = row < R ? src[row * F_GS + col] : 0.0;
        dmma884(h[mt][0], h[mt][1], a, wb[ks]);
      }
      if (E > 0) {
        dmma884(h[4][0], h[4][1], lxre[g * F_GS + col], wb[ks]);
        dmma884(h[5][0], h[5][1], lxim[g * F_GS + col], wb[ks]);
      }
    }
    if (E > 0) {
#pragma unroll
      for (int ks = 0; ks < 4; ++ks)
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          if (F_ICONST_RELOAD) {
            double la[2], ca[2];
            ly_op(ks, la);
            cr_op(ks, ca);
            dmma884(uy[mt][0], uy[mt][1], la[mt], yb[ks]);
            dmma884(cbo[mt][0], cbo[mt][1], ca[mt], cb[ks]);
          } else {
            dmma884(uy[mt][0], uy[mt][1], lyA[mt][ks], yb[ks]);
            dmma884(cbo[mt][0], cbo[mt][1], crA[mt][ks], cb[ks]);
          }
        }
    }
#endif
    // epilogue: lane (g, t) holds row g of every product for samples n0 + 2t + j
    // part = Dx (Dy rp + b_g hx_g) + a_g (Dy uy_g + (C b)_g), then the sum over g
    cplx pj[2];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int sn = n0 + 2 * t + j;
      const int snc = sn < sb ? sn : sa;
      const int oyn = s_by[snc] - ty0;
      const cplx* rx = s_rx + snc * RR;
      const cplx* ry = s_ry + snc * RR;
      const cplx Dx = rx[0], Dy = ry[0];
      cplx rp = mk(0, 0);
#pragma unroll
      for (int mh = 0; mh < 2; ++mh) {
        const int d = band0 + mh * 8 + g - oyn;
        double w = 0.0;
        if ((unsigned)d < (unsigned)S) w = s_wy[snc * S + d];
        rp = caxpy(rp, w, mk(h[mh][j], h[2 + mh][j]));
      }
      cplx part;
      if (E > 0 && g < E) {
        const cplx ag = rx[1 + g], bg = ry[1 + g];
        part = cmul(Dx, cadd(cmul(Dy, rp), cmul(bg, mk(h[4][j], h[5][j]))));
        part = cadd(part, cmul(ag, cadd(cmul(Dy, mk(uy[0][j], uy[1][j])), mk(cbo[0][j], cbo[1][j]))));
      } else {
        part = cmul(Dx, cmul(Dy, rp));
      }
      pj[j] = part;
    }
    // transposing reduction over the 8 lanes of a sample column: the first
    // exchange leaves lane g with sample 2t + (g & 1) only, so the two later
    // steps move and add one complex per lane instead of two
    const int jj = g & 1;
    const cplx send = jj ? pj[0] : pj[1];
    cplx acc = jj ? pj[1] : pj[0];
    acc.x += __shfl_xor_sync(0xffffffffu, send.x, 4);
    acc.y += __shfl_xor_sync(0xffffffffu, send.y, 4);
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    const int sn = n0 + 2 * t + jj;
    if (g < 2 && sn < sb) {
      const int64_t gs = g0 + sn;
      y[ybase + (out_perm ? (int64_t)out_perm[gs] : (int64_t)(s0 + sn))] = acc;
    }
  }
}

template <int P, bool BAL>
__global__ void __launch_bounds__(32 * F_IWARPS * F_IMSPLIT, F_IBLOCKS_M)
k2f_interp_mma(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0, const int* __restrict__ ch_s1,
               const int* __restrict__ ch_count, const uint4* __restrict__ ch_rows, int cap,
               const int* __restrict__ base_x,
               const int* __restrict__ base_y, const double* __restrict__ wx_all, const double* __restrict__ wy_all,
               const cplx* __restrict__ recx_all, const cplx* __restrict__ recy_all, const cplx* __restrict__ G,
               const cplx* __restrict__ lines, const cplx* __restrict__ x, const int* __restrict__ out_perm,
               cplx* __restrict__ y) {
  using FI = FInterpM<P>;
  constexpr int S = F_S, T = F_T, R = F_R, BAND = F_T / F_IWARPS, RR = FI::RR, IMU = F_IMUNROLL;
  constexpr int E = P >= 2 ? 2 * P : 0, EE = E > 0 ? E : 1;
  extern __shared__ __align__(16) unsigned char fim_raw[];
  double* gre = reinterpret_cast<double*>(fim_raw + FI::GRE);
  double* gim = reinterpret_cast<double*>(fim_raw + FI::GIM);
  double* lxre = reinterpret_cast<double*>(fim_raw + FI::LXRE);
  double* lxim = reinterpret_cast<double*>(fim_raw + FI::LXIM);
  __shared__ __align__(16) cplx lys[EE][R];
  __shared__ __align__(16) cplx cxs[P >= 2 ? 4 * P * P : 1];
  __shared__ __align__(8) uint64_t stage_bar;
  const int prob = blockIdx.y, c = blockIdx.x;
  const int64_t chunk = (int64_t)prob * cap + c;
  // descriptor loads issued with the live-chunk test, not behind it (one L2 round trip, not two)
#if F_DESC_HOIST == 2
  const int tile = ch_tile[chunk], s0 = ch_s0[chunk], s1 = ch_s1[chunk];
  const uint4 rw = ch_rows[chunk];
  if (s1 <= s0) return;
#else
#if F_DESC_HOIST
  const int nlive = ch_count[prob];
#else
  if (c >= ch_count[prob]) return;
  constexpr int nlive = 0x7fffffff;
#endif
  const int tile = ch_tile[chunk], s0 = ch_s0[chunk], s1 = ch_s1[chunk];
  const uint4 rw = ch_rows[chunk];
  if (c >= nlive) return;
#endif
  F_TL(0);
  const int n = s1 - s0;
  const int ty = tile / Pp.nt, tx = tile - ty * Pp.nt;
  const int ty0 = ty * T, tx0 = tx * T;
  const int n_ov = Pp.n_ov, mask = n_ov - 1, nn = Pp.n;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int64_t g0 = (int64_t)prob * Pp.M + s0;
  // ---- staging, all of it asynchronous so that no thread waits on one load
  // before issuing the next: weights / records / window origins by TMA bulk
  // copies (mbarrier), the grid region and lines by cp.async 8-B copies split
  // into re / im planes (cp.async group)
  const double* wy_src = wy_all + g0 * S;
  const double* wx_src = wx_all + g0 * S;
  const cplx* rx_src = recx_all + g0 * RR;
  const cplx* ry_src = recy_all + g0 * RR;
  const double* s_wy = reinterpret_cast<const double*>(fim_raw + FI::WY + (reinterpret_cast<uintptr_t>(wy_src) & 15));
  const double* s_wx = reinterpret_cast<const double*>(fim_raw + FI::WX + (reinterpret_cast<uintptr_t>(wx_src) & 15));
#if F_IREC_GLOBAL
  const cplx* s_rx = rx_src;
  const cplx* s_ry = ry_src;
#else
  const cplx* s_rx = reinterpret_cast<const cplx*>(fim_raw + FI::RX + (reinterpret_cast<uintptr_t>(rx_src) & 15));
  const cplx* s_ry = reinterpret_cast<const cplx*>(fim_raw + FI::RY + (reinterpret_cast<uintptr_t>(ry_src) & 15));
#endif
  const int* s_bx = reinterpret_cast<const int*>(fim_raw + FI::BX + (reinterpret_cast<uintptr_t>(base_x + g0) & 15));
  const int* s_by = reinterpret_cast<const int*>(fim_raw + FI::BY + (reinterpret_cast<uintptr_t>(base_y + g0) & 15));
  if (threadIdx.x == 0) {
    bar_init(&stage_bar);
    bar_expect(&stage_bar, bulk_bytes(wy_src, sizeof(double) * S * n) + bulk_bytes(wx_src, sizeof(double) * S * n) +
                               (F_IREC_GLOBAL ? 0u : bulk_bytes(rx_src, sizeof(cplx) * RR * n) +
                                                         bulk_bytes(ry_src, sizeof(cplx) * RR * n)) +
                               bulk_bytes(base_x + g0, sizeof(int) * n) + bulk_bytes(base_y + g0, sizeof(int) * n));
#if F_IREC_GLOBAL
    l2_prefetch(rx_src, sizeof(cplx) * RR * n);
    l2_prefetch(ry_src, sizeof(cplx) * RR * n);
#endif
    bulk_stage(fim_raw + FI::WY, wy_src, sizeof(double) * S * n, &stage_bar);
    bulk_stage(fim_raw + FI::WX, wx_src, sizeof(double) * S * n, &stage_bar);
#if !F_IREC_GLOBAL
    bulk_stage(fim_raw + FI::RX, rx_src, sizeof(cplx) * RR * n, &stage_bar);
    bulk_stage(fim_raw + FI::RY, ry_src, sizeof(cplx) * RR * n, &stage_bar);
#endif
    bulk_stage(fim_raw + FI::BX, base_x + g0, sizeof(int) * n, &stage_bar);
    bulk_stage(fim_raw + FI::BY, base_y + g0, sizeof(int) * n, &stage_bar);
  }
  if (threadIdx.x == 32)
    prefetch_chunk_ahead<RR, F_PF_INTERP>(prob, c, cap, gridDim.y, Pp.M, ch_s0, ch_s1, base_x, base_y, wx_all, wy_all,
                                          recx_all, recy_all, nullptr);
  const cplx* gp = G + (int64_t)prob * n_ov * n_ov;
#pragma unroll 4
  for (int i = threadIdx.x; i < R * R; i += blockDim.x) {
    const int r = i / R, cc = i - r * R;
    const double* src = reinterpret_cast<const double*>(gp + (int64_t)((ty0 + r) & mask) * n_ov + ((tx0 + cc) & mask));
    cp_async8(gre + r * F_GS + cc, src);
    cp_async8(gim + r * F_GS + cc, src + 1);
  }
  if (E > 0) {
    const cplx* LY = lines + (int64_t)prob * 2 * E * n_ov;
    const cplx* LX = LY + (int64_t)E * n_ov;
    for (int i = threadIdx.x; i < E * R; i += blockDim.x) {
      const int e = i / R, r = i - e * R;
      const double* vx = reinterpret_cast<const double*>(LX + (int64_t)e * n_ov + ((tx0 + r) & mask));
      cp_async8(lxre + e * F_GS + r, vx);
      cp_async8(lxim + e * F_GS + r, vx + 1);
      cp_async16(&lys[e][r], LY + (int64_t)e * n_ov + ((ty0 + r) & mask));
    }
    for (int i = E * R + threadIdx.x; i < 8 * R; i += blockDim.x) {  // rows E..7 of the x-line operand are zero
      const int e = i / R, r = i - e * R;
      lxre[e * F_GS + r] = 0.0;
      lxim[e * F_GS + r] = 0.0;
    }
    const cplx* X = x + (int64_t)prob * nn * nn;
    for (int q = threadIdx.x; q < 4 * P * P; q += blockDim.x) {
      const int k = q / (P * P), rem = q - k * P * P, i = rem / P, j = rem - i * P;
      const int row0 = (k < 2) ? 0 : nn - P, col0 = (k % 2 == 0) ? 0 : nn - P;
      cp_async16(&cxs[q], X + (int64_t)(col0 + j) * nn + row0 + i);
    }
  }
  cp_async_wait_all();
  __syncthreads();  // barrier initialised, region / lines / corners landed
  bar_wait(&stage_bar, 0);
  F_TL(1);
#if F_IMSPLIT == 1
  // balanced schedule: this warp's band and its run of the band's 8-sample tiles (f_band_schedule)
  constexpr int half = 0;
  int wband[F_IWARPS], sa, sb, band0 = 0;
  f_band_schedule<F_IWARPS, BAND, 8, BAL>(rw, warp, wband, sa, sb);
#pragma unroll
  for (int w = 0; w < F_IWARPS; ++w)
    if (w == warp) band0 = wband[w] * BAND;
#else
  const int band0 = (warp % F_IWARPS) * BAND, half = warp / F_IWARPS;
  const int sa = row_start(rw, band0), sb = row_start(rw, band0 + BAND);  // precomputed band starts
#endif
  f_interp_band<P, F_IMSPLIT>(band0, half, sa, sb, ty0, tx0, s_wx, s_wy, s_rx, s_ry, s_bx, s_by, gre, gim, lxre, lxim,
                              lys, cxs, (int64_t)prob * Pp.M, g0, s0, out_perm, y);
  F_TL_SYNC();
  F_TL(2);
}

