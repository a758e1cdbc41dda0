// kernels_nfft2d_fast.cuh -- sm_100a fast path of the 2D route for the default
// Kaiser-Bessel window (w = 6, S = 13 taps) and p <= 4 (haar .. db4):
//
//  * samples are bin-sorted by 12x12 grid tile and, inside a tile, by cell
//    (row-major); the work list is (tile, chunk of <= 512 samples) so dense
//    tiles (the spiral's centre) split across CTAs;
//  * k2f_interp  -- one CTA per chunk stages the tile's (T+12)^2 grid region,
//    its 2 x 2p side-line segments and the 4 p x p corner blocks in shared
//    memory once, then one thread per sample interpolates from shared memory
//    (nufft.cpp:287-303 + freq2wave.cpp:255-301);
//  * k2f_spread  -- output-stationary in registers: lane c < 24 owns grid
//    column c of the 24-row region (24 complex accumulators) and the 2p
//    x-line entries at column c, lanes 24..31 own the 2p y-lines.  A warp
//    takes whole sample rows of the chunk, so the row offset of every rank-1
//    update is a compile-time constant (12 instantiations) and all register
//    indices are static.  The 4 warps' copies are folded once per chunk and
//    written with no atomics (transpose of the interpolation,
//    nufft.cpp:324-338 + freq2wave.cpp:332-385).
#pragma once
#include "kernels_nfft.cuh"

#define F_S 13
#define F_T 12
#define F_R 24
#define F_CHUNK 160  // samples per work item (chunks of a tile are staged in shared memory)

// ------------------------------------------------------------------ interpolation
template <int P>
__global__ void __launch_bounds__(128, 3) k2f_interp(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0,
                                                     const int* __restrict__ ch_s1, const int* __restrict__ ch_count,
                                                     int cap, const int* __restrict__ base_x, const int* __restrict__ base_y,
                                                     const double* __restrict__ wx_all, const double* __restrict__ wy_all,
                                                     const cplx* __restrict__ recx_all, const cplx* __restrict__ recy_all,
                                                     const cplx* __restrict__ G, const cplx* __restrict__ lines,
                                                     const cplx* __restrict__ x, const int* __restrict__ out_perm,
                                                     cplx* __restrict__ y) {
  constexpr int S = F_S, T = F_T, R = F_R;
  constexpr int E = P >= 2 ? 2 * P : 0;
  constexpr int EE = E > 0 ? E : 1;
  constexpr int RR = 1 + E;
  constexpr int NC = P >= 2 ? 4 * P * P : 1;
  constexpr int RS = R + 1;  // padded row stride: rows 384 B apart would alias the same banks
  __shared__ cplx reg[R * RS];
  __shared__ cplx ly[EE][R];
  __shared__ cplx lx[EE][R];
  __shared__ cplx cx[NC];
  const int prob = blockIdx.y, c = blockIdx.x;
  if (c >= ch_count[prob]) return;
  const int tile = ch_tile[prob * cap + c], s0 = ch_s0[prob * cap + c], s1 = ch_s1[prob * cap + c];
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
    cp16(reg + r * RS + cc, g + (int64_t)((ty * T + r) & mask) * n_ov + ((tx * T + cc) & mask));
  }
  if (E > 0) {
    const cplx* LY = lines + (int64_t)prob * 2 * E * n_ov;
    const cplx* LX = LY + (int64_t)E * n_ov;
    for (int i = threadIdx.x; i < E * R; i += blockDim.x) {
      const int e = i / R, r = i - e * R;
      cp16(&ly[e][r], LY + (int64_t)e * n_ov + ((ty * T + r) & mask));
      cp16(&lx[e][r], LX + (int64_t)e * n_ov + ((tx * T + r) & mask));
    }
    const cplx* X = x + (int64_t)prob * n * n;
    for (int q = threadIdx.x; q < 4 * P * P; q += blockDim.x) {
      const int k = q / (P * P), rem = q - k * P * P, i = rem / P, j = rem - i * P;
      const int row0 = (k < 2) ? 0 : n - P, col0 = (k % 2 == 0) ? 0 : n - P;
      cp16(cx + q, X + (int64_t)(col0 + j) * n + row0 + i);
    }
  }
  // the chunk's window weights (contiguous ranges, staged 16-B aligned-down)
  const int64_t g0 = (int64_t)prob * Pp.M + s0;
  const int nn = s1 - s0;
  auto stage = [&](double* dst, const double* src, int count) -> const double* {
    const uintptr_t a = reinterpret_cast<uintptr_t>(src), al = a & ~uintptr_t(15);
    const int off = (int)(a - al), nv = (off + count * 8 + 15) / 16;
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    for (int i = threadIdx.x; i < nv; i += blockDim.x)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d + 16u * i),
                   "l"(reinterpret_cast<const char*>(al) + 16 * i)
                   : "memory");
    return reinterpret_cast<const double*>(reinterpret_cast<const char*>(dst) + off);
  };
  extern __shared__ __align__(16) double fi_dyn[];  // [2][F_CHUNK * S + 2]
  double* swy = fi_dyn;
  double* swx = fi_dyn + F_CHUNK * S + 2;
  const double* wys = stage(swy, wy_all + g0 * S, nn * S);
  const double* wxs = stage(swx, wx_all + g0 * S, nn * S);
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const int64_t gs = (int64_t)prob * Pp.M + s;
    const int oy = base_y[gs] - ty * T, ox = base_x[gs] - tx * T;
    const double* wyp = wys + (s - s0) * S;
    const double* wxp = wxs + (s - s0) * S;
    const cplx* rx = recx_all + gs * RR;
    const cplx* ry = recy_all + gs * RR;
    const cplx Dx = ldg2(rx), Dy = ldg2(ry);
    // out = Dx Dy acc + Dx (b . ux) + a^T (C b + Dy uy): interior (freq2wave.cpp:255),
    // the 4 corner blocks C (260-270) and both side families (272-301), with
    // a = [Lx|Rx](m,:), b = [Ly|Ry](m,:)
    cplx bv[EE];
#pragma unroll
    for (int e = 0; e < E; ++e) bv[e] = ldg2(ry + 1 + e);
    cplx out;
    {
      double wx[S];
#pragma unroll
      for (int t = 0; t < S; ++t) wx[t] = wxp[t];
      cplx acc = mk(0, 0);
#pragma unroll
      for (int t0 = 0; t0 < S; ++t0) {
        const cplx* row = reg + (oy + t0) * RS + ox;
        cplx ra = mk(0, 0);
#pragma unroll
        for (int t1 = 0; t1 < S; ++t1) ra = caxpy(ra, wx[t1], row[t1]);
        acc = caxpy(acc, wyp[t0], ra);
      }
      out = cmul(cmul(Dx, Dy), acc);
      if (E > 0) {
        cplx sx = mk(0, 0);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          cplx u = mk(0, 0);
#pragma unroll
          for (int t = 0; t < S; ++t) u = caxpy(u, wx[t], lx[e][ox + t]);
          sx = cadd(sx, cmul(bv[e], u));
        }
        out = cadd(out, cmul(Dx, sx));
      }
    }
    if (E > 0) {
      double wy[S];
#pragma unroll
      for (int t = 0; t < S; ++t) wy[t] = wyp[t];
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int hi = i < P ? 0 : 1, ii = i - hi * P;
        cplx u = mk(0, 0);
#pragma unroll
        for (int t = 0; t < S; ++t) u = caxpy(u, wy[t], ly[i][oy + t]);
        cplx v = cmul(Dy, u);
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int hj = j < P ? 0 : 1, jj = j - hj * P;
          v = cadd(v, cmul(cx[(2 * hi + hj) * P * P + ii * P + jj], bv[j]));
        }
        out = cadd(out, cmul(ldg2(rx + 1 + i), v));
      }
    }
    const int64_t o = out_perm ? (int64_t)out_perm[gs] : s;
    y[(int64_t)prob * Pp.M + o] = out;
  }
}

// ------------------------------------------------------------------ spreading
#define F_WARPS 4

template <int P>
struct FSpread {
  static constexpr int E = P >= 2 ? 2 * P : 0;
  static constexpr int EE = E > 0 ? E : 1;
  static constexpr int RR = 1 + E;
  static constexpr int NCE = P >= 2 ? 4 * P * P : 0;
  static constexpr int NCU = NCE > 0 ? (NCE + 31) / 32 : 1;
  static constexpr int PER_WARP = F_R * F_R + 2 * E * F_R;  // region + y-lines + x-lines
  // staged chunk (structure of arrays, in sample order)
  // each staged array gets 16 B of slack: copies start at the 16-B-aligned address below
  static constexpr size_t STG_WY = 0;
  static constexpr size_t STG_WX = STG_WY + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t STG_RX = STG_WX + sizeof(double) * F_CHUNK * F_S + 32;
  static constexpr size_t STG_RY = STG_RX + sizeof(cplx) * F_CHUNK * RR + 16;
  static constexpr size_t STG_YS = STG_RY + sizeof(cplx) * F_CHUNK * RR + 16;
  static constexpr size_t STG_OX = STG_YS + sizeof(cplx) * F_CHUNK;
  static constexpr size_t STG_END = STG_OX + sizeof(int) * F_CHUNK;
  static constexpr size_t FOLD = sizeof(cplx) * (F_WARPS * PER_WARP + F_WARPS * (NCE > 0 ? NCE : 1));
  static constexpr size_t MAIN = (STG_END > FOLD ? STG_END : FOLD);  // fold buffer aliases the staging
  struct Scratch {  // derived per-sample values shared inside a warp (two samples in flight)
    cplx d[2][32];
    double2 wy[16];  // row taps of the two samples, packed (wy_a[t], wy_b[t])
  };
  static constexpr size_t bytes() { return (MAIN + 15) / 16 * 16 + sizeof(Scratch) * F_WARPS; }
};

// acc[OY + t] += w[t].x u0 + w[t].y u1, t < 13 (w = the two samples' row taps,
// packed pairwise), with OY a compile-time row offset
template <int OY>
__device__ __forceinline__ void f_upd(cplx (&acc)[F_R], cplx u0, cplx u1, const double2* w) {
#pragma unroll
  for (int t = 0; t < F_S; ++t) {
    const double2 ww = w[t];
    acc[OY + t].x = fma(ww.y, u1.x, fma(ww.x, u0.x, acc[OY + t].x));
    acc[OY + t].y = fma(ww.y, u1.y, fma(ww.x, u0.y, acc[OY + t].y));
  }
}
__device__ __forceinline__ void f_upd_dispatch(int oy, cplx (&acc)[F_R], cplx u0, cplx u1, const double2* w) {
  switch (oy) {
    case 0: f_upd<0>(acc, u0, u1, w); break;
    case 1: f_upd<1>(acc, u0, u1, w); break;
    case 2: f_upd<2>(acc, u0, u1, w); break;
    case 3: f_upd<3>(acc, u0, u1, w); break;
    case 4: f_upd<4>(acc, u0, u1, w); break;
    case 5: f_upd<5>(acc, u0, u1, w); break;
    case 6: f_upd<6>(acc, u0, u1, w); break;
    case 7: f_upd<7>(acc, u0, u1, w); break;
    case 8: f_upd<8>(acc, u0, u1, w); break;
    case 9: f_upd<9>(acc, u0, u1, w); break;
    case 10: f_upd<10>(acc, u0, u1, w); break;
    case 11: f_upd<11>(acc, u0, u1, w); break;
    default: __builtin_unreachable();
  }
}

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

template <int P>
__global__ void __launch_bounds__(32 * F_WARPS, 2)
k2f_spread(NfP Pp, const int* __restrict__ ch_tile, const int* __restrict__ ch_s0, const int* __restrict__ ch_s1,
           const int* __restrict__ ch_count, int cap, const int* __restrict__ base_x, const int* __restrict__ base_y,
           const double* __restrict__ wx_all, const double* __restrict__ wy_all, const cplx* __restrict__ recx_all,
           const cplx* __restrict__ recy_all, const cplx* __restrict__ yin, const int* __restrict__ in_perm,
           cplx* __restrict__ TB, cplx* __restrict__ TL, cplx* __restrict__ TC) {
  using F = FSpread<P>;
  constexpr int S = F_S, T = F_T, R = F_R, E = F::E, EE = F::EE, RR = F::RR, NCE = F::NCE, NCU = F::NCU;
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  cplx* s_ys = reinterpret_cast<cplx*>(fsm_raw + F::STG_YS);
  int* s_ox = reinterpret_cast<int*>(fsm_raw + F::STG_OX);
  typename F::Scratch* scr_all = reinterpret_cast<typename F::Scratch*>(fsm_raw + (F::MAIN + 15) / 16 * 16);
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
  typename F::Scratch& scr = scr_all[warp];
  cplx acc[R];
  cplx accx[EE];
  cplx cacc[NCU];
  int cqa[NCU], cqb[NCU];
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = mk(0, 0);
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
  // lane roles of the derived values (see the loop): A from ry (lanes 0..7) or rx,
  // record index 1 + e (clamped to the family) or 0 (lane >= 24); B = Dx | 1 | Dy
  const int role_e = E > 0 ? ((lane & 7) < E ? (lane & 7) : E - 1) : 0;
  const bool role_a_y = lane < 8;
  const int role_idx = (lane < 24 && E > 0) ? 1 + role_e : 0;
  const int role_b = lane < 8 ? 0 : (lane < 16 ? 1 : 2);
  for (int oy = warp; oy < T; oy += F_WARPS) {
    const int a = rs[oy], b = rs[oy + 1];
    for (int s = a; s < b; s += 2) {
      const int sb = s + 1 < b ? s + 1 : s;     // odd tail: second slot repeats the first ...
      const double kb = s + 1 < b ? 1.0 : 0.0;  // ... with zero amplitude
      // derived per-sample values, one per lane, z = conj(A B) ys:
      //   lanes 0..7  vx_e = conj(By(m,e) Dx) y   (side_y_edge, freq2wave.cpp:376)
      //   lanes 8..15 ca_i = conj(Ax(m,i)) y      (corner rows, freq2wave.cpp:351)
      //   lanes 16..23 vy_e = conj(Ax(m,e) Dy) y  (side_x_edge, freq2wave.cpp:363)
      //   lane 24      v2  = conj(Dx Dy) y        (interior,    freq2wave.cpp:335)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = k ? sb : s;
        const cplx* rx = s_rx + i * RR;
        const cplx* ry = s_ry + i * RR;
        const cplx ys = k ? cscale(s_ys[i], kb) : s_ys[i];
        const cplx Av = role_a_y ? ry[role_idx] : rx[role_idx];
        const cplx Bv = role_b == 0 ? rx[0] : (role_b == 1 ? mk(1.0, 0.0) : ry[0]);
        scr.d[k][lane] = cmul(conj_(cmul(Av, Bv)), ys);
      }
      if (lane < S) scr.wy[lane] = make_double2(s_wy[s * S + lane], s_wy[sb * S + lane]);
      __syncwarp();
      cplx u[2];
      double w1[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int i = k ? sb : s;
        const int t1 = lane - s_ox[i];
        const bool colv = lane < R && t1 >= 0 && t1 < S;
        w1[k] = colv ? s_wx[i * S + (t1 < 0 ? 0 : (t1 >= S ? S - 1 : t1))] : 0.0;
        const cplx ug = cscale(scr.d[k][24], w1[k]);
        u[k] = lane < R ? ug : ((E > 0 && lane - R < E) ? scr.d[k][16 + ly] : mk(0, 0));
      }
      f_upd_dispatch(oy, acc, u[0], u[1], scr.wy);
      if (E > 0) {
#pragma unroll
        for (int e = 0; e < E; ++e) accx[e] = caxpy(caxpy(accx[e], w1[0], scr.d[0][e]), w1[1], scr.d[1][e]);
        const cplx* rya = s_ry + s * RR;
        const cplx* ryb = s_ry + sb * RR;
#pragma unroll
        for (int uu = 0; uu < NCU; ++uu)  // corners (freq2wave.cpp:349-353)
          if (lane + 32 * uu < NCE)
            cacc[uu] = cadd(cadd(cacc[uu], cmul(scr.d[0][8 + cqa[uu]], conj_(rya[cqb[uu]]))),
                            cmul(scr.d[1][8 + cqa[uu]], conj_(ryb[cqb[uu]])));
      }
      __syncwarp();
    }
  }
  __syncthreads();  // the fold buffer aliases the staging area
  // dump the warp copies, fold, write this chunk's region / lines / corners once
  cplx* buf = reinterpret_cast<cplx*>(fsm_raw);  // [F_WARPS][PER_WARP]
  cplx* cbuf = buf + F_WARPS * F::PER_WARP;       // [F_WARPS][NCE]
  cplx* mine = buf + warp * F::PER_WARP;
  if (lane < R) {
#pragma unroll
    for (int r = 0; r < R; ++r) mine[r * R + lane] = acc[r];
#pragma unroll
    for (int e = 0; e < E; ++e) mine[R * R + E * R + e * R + lane] = accx[e];
  } else if (lane - R < E) {
#pragma unroll
    for (int r = 0; r < R; ++r) mine[R * R + (lane - R) * R + r] = acc[r];
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
    cplx a = buf[i];
#pragma unroll
    for (int w = 1; w < F_WARPS; ++w) a = cadd(a, buf[w * F::PER_WARP + i]);
    tb[i] = a;
  }
  if (E > 0) {
    cplx* tl = TL + chunk * 2 * E * R;
    for (int i = threadIdx.x; i < 2 * E * R; i += blockDim.x) {
      cplx a = buf[R * R + i];
#pragma unroll
      for (int w = 1; w < F_WARPS; ++w) a = cadd(a, buf[w * F::PER_WARP + R * R + i]);
      tl[i] = a;
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
