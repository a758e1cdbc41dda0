// voronoi_common.h -- one 2D Voronoi cell clipped to [-K, K]^2 (weights.cpp:
// 20-70 semantics: the same half-plane clip and shoelace area), evaluated
// against the point's neighbours only, ring by ring over a bucket grid in
// increasing (distance^2, index) order, until no farther point can cut it.
// Shared verbatim by the host harness (host_inputs.cpp) and the GPU kernel
// (gs_voronoi.cu, compiled without FMA contraction) so both produce the same
// doubles.  CAP_V / CAP_C bound the polygon and per-ring candidate buffers;
// exceeding them returns VOR_OVERFLOW (the GPU then recomputes that point on
// the host with unbounded buffers).
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define GS_HD __host__ __device__
#else
#define GS_HD
#endif

#define VOR_OK 0
#define VOR_OVERFLOW 1
#ifndef VOR_STREAM_MAXPOP
#define VOR_STREAM_MAXPOP 160  // ring population beyond which vor_cell_stream hands the cell back
#endif

#include <vector>
// host_inputs.cpp: bucket grid + range / duplicate checks; 0 or an error code (message: gs_inputs_last_error)
extern "C++" int vor_grid_build(int64_t M, const double* coords, double K, std::vector<int64_t>& start,
                                std::vector<int64_t>& idx, int& G, double& h);

struct VorGrid {
  const double* c;       // [M][2]
  const int64_t* start;  // [G*G + 1] bucket starts
  const int64_t* idx;    // [M] point indices grouped by bucket
  int64_t M;
  int G;
  double K, h;
};

GS_HD inline int vor_bucket(const VorGrid& g, double v) {
  int b = (int)floor((v + g.K) / g.h);
  return b < 0 ? 0 : (b > g.G - 1 ? g.G - 1 : b);
}

// clip (px, py)[n] against a.(q - mid) <= 0 into (ox, oy); returns the new
// count or -1 when it would exceed cap (weights.cpp:20-38)
GS_HD inline int vor_clip(const double* px, const double* py, int n, double midx, double midy, double ax, double ay,
                          double* ox, double* oy, int cap) {
  int k = 0;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    const double dc = ax * (px[i] - midx) + ay * (py[i] - midy);
    const double dn = ax * (px[j] - midx) + ay * (py[j] - midy);
    if (dc <= 0) {
      if (k >= cap) return -1;
      ox[k] = px[i];
      oy[k] = py[i];
      ++k;
    }
    if ((dc < 0 && dn > 0) || (dc > 0 && dn < 0)) {
      if (k >= cap) return -1;
      const double t = dc / (dc - dn);
      ox[k] = px[i] + t * (px[j] - px[i]);
      oy[k] = py[i] + t * (py[j] - py[i]);
      ++k;
    }
  }
  return k;
}

// mu = cell area (weights.cpp:40-49), rad = farthest vertex (density candidates)
// buffers: px, py, qx, qy [CAP_V]; cd [CAP_C] distances, cj [CAP_C] indices
GS_HD inline int vor_cell(const VorGrid& g, int64_t m, double* px, double* py, double* qx, double* qy, int capv,
                          double* cd, int64_t* cj, int capc, double* mu, double* rad) {
  const double ownx = g.c[2 * m], owny = g.c[2 * m + 1], K = g.K;
  const int cx = vor_bucket(g, ownx), cy = vor_bucket(g, owny);
  int n = 4;
  px[0] = -K; py[0] = -K;
  px[1] = K;  py[1] = -K;
  px[2] = K;  py[2] = K;
  px[3] = -K; py[3] = K;
  for (int ring = 0;; ++ring) {
    int nc = 0;
    for (int gy = cy - ring; gy <= cy + ring; ++gy) {
      if (gy < 0 || gy >= g.G) continue;
      for (int gx = cx - ring; gx <= cx + ring; ++gx) {
        if (gx < 0 || gx >= g.G) continue;
        const int dxr = gx - cx < 0 ? cx - gx : gx - cx, dyr = gy - cy < 0 ? cy - gy : gy - cy;
        if ((dxr > dyr ? dxr : dyr) != ring) continue;
        const int64_t b = (int64_t)gy * g.G + gx;
        for (int64_t i = g.start[b]; i < g.start[b + 1]; ++i) {
          const int64_t j = g.idx[i];
          if (j == m) continue;
          const double dx = g.c[2 * j] - ownx, dy = g.c[2 * j + 1] - owny;
          const double d2 = dx * dx + dy * dy;
          if (nc >= capc) return VOR_OVERFLOW;
          // insertion by (d2, j): the order std::sort gives the host's pairs
          int k = nc++;
          while (k > 0 && (cd[k - 1] > d2 || (cd[k - 1] == d2 && cj[k - 1] > j))) {
            cd[k] = cd[k - 1];
            cj[k] = cj[k - 1];
            --k;
          }
          cd[k] = d2;
          cj[k] = j;
        }
      }
    }
    for (int t = 0; t < nc && n > 0; ++t) {
      const double qxj = g.c[2 * cj[t]], qyj = g.c[2 * cj[t] + 1];
      const int nn = vor_clip(px, py, n, (ownx + qxj) / 2, (owny + qyj) / 2, qxj - ownx, qyj - owny, qx, qy, capv);
      if (nn < 0) return VOR_OVERFLOW;
      for (int i = 0; i < nn; ++i) {
        px[i] = qx[i];
        py[i] = qy[i];
      }
      n = nn;
    }
    if (n == 0) break;
    // every point outside rings <= ring is at least `reach` from the owner
    const double h = g.h;
    const double ax0 = ownx - (-K + (cx - ring) * h), ax1 = (-K + (cx + ring + 1) * h) - ownx;
    const double ay0 = owny - (-K + (cy - ring) * h), ay1 = (-K + (cy + ring + 1) * h) - owny;
    const double dxm = ax0 < ax1 ? ax0 : ax1, dym = ay0 < ay1 ? ay0 : ay1;
    const double reach = dxm < dym ? dxm : dym;
    const bool covers_all = cx - ring <= 0 && cy - ring <= 0 && cx + ring >= g.G - 1 && cy + ring >= g.G - 1;
    double rmax2 = 0.0;
    for (int i = 0; i < n; ++i) {
      const double r2 = (px[i] - ownx) * (px[i] - ownx) + (py[i] - owny) * (py[i] - owny);
      rmax2 = r2 > rmax2 ? r2 : rmax2;
    }
    if (covers_all || 4.0 * rmax2 <= reach * reach) break;
  }
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    acc += px[i] * py[j] - px[j] * py[i];
  }
  if (mu) *mu = 0.5 * fabs(acc);
  if (rad) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d = hypot(px[i] - ownx, py[i] - owny);
      r = d > r ? d : r;
    }
    *rad = r;
  }
  return VOR_OK;
}

// The same cell, for the GPU thread with no candidate buffer: within a ring
// the candidates are visited in the host's (d2, j) order by repeated min-scans
// of the ring's buckets, and the scan stops at the first candidate with
// d2 > 4.5 rmax^2 of the current polygon.  Such a candidate's bisector clears
// every vertex by >= 0.06 d rmax (|v - own| <= rmax < d / 2.12), so its clip
// -- and every later one in the ring, rmax only shrinks -- leaves the polygon
// unchanged exactly: the host's clip sequence minus its no-ops, hence the
// same doubles.  Dense buckets (the spiral's arms) cost scans, not memory.
GS_HD inline int vor_cell_stream(const VorGrid& g, int64_t m, double* px, double* py, double* qx, double* qy, int capv,
                                 double* mu) {
  const double ownx = g.c[2 * m], owny = g.c[2 * m + 1], K = g.K;
  const int cx = vor_bucket(g, ownx), cy = vor_bucket(g, owny);
  int n = 4;
  px[0] = -K; py[0] = -K;
  px[1] = K;  py[1] = -K;
  px[2] = K;  py[2] = K;
  px[3] = -K; py[3] = K;
  double rmax2 = 2.0 * K * K * 4.0;  // box diagonal bound: nothing pruned before the first clip
  for (int ring = 0;; ++ring) {
    double last_d2 = -1.0;
    int64_t last_j = -1;
    {  // the min-scans are quadratic in the ring's population: dense rings go to the host
      int64_t pop = 0;
      for (int gy = cy - ring; gy <= cy + ring; ++gy) {
        if (gy < 0 || gy >= g.G) continue;
        for (int gx = cx - ring; gx <= cx + ring; ++gx) {
          if (gx < 0 || gx >= g.G) continue;
          const int dxr = gx - cx < 0 ? cx - gx : gx - cx, dyr = gy - cy < 0 ? cy - gy : gy - cy;
          if ((dxr > dyr ? dxr : dyr) != ring) continue;
          const int64_t b = (int64_t)gy * g.G + gx;
          pop += g.start[b + 1] - g.start[b];
        }
      }
      if (pop > VOR_STREAM_MAXPOP) return VOR_OVERFLOW;
    }
    while (n > 0) {
      double best_d2 = 0.0;
      int64_t best_j = -1;
      for (int gy = cy - ring; gy <= cy + ring; ++gy) {
        if (gy < 0 || gy >= g.G) continue;
        for (int gx = cx - ring; gx <= cx + ring; ++gx) {
          if (gx < 0 || gx >= g.G) continue;
          const int dxr = gx - cx < 0 ? cx - gx : gx - cx, dyr = gy - cy < 0 ? cy - gy : gy - cy;
          if ((dxr > dyr ? dxr : dyr) != ring) continue;
          const int64_t b = (int64_t)gy * g.G + gx;
          for (int64_t i = g.start[b]; i < g.start[b + 1]; ++i) {
            const int64_t j = g.idx[i];
            if (j == m) continue;
            const double dx = g.c[2 * j] - ownx, dy = g.c[2 * j + 1] - owny;
            const double d2 = dx * dx + dy * dy;
            const bool after = d2 > last_d2 || (d2 == last_d2 && j > last_j);
            const bool before = best_j < 0 || d2 < best_d2 || (d2 == best_d2 && j < best_j);
            if (after && before) {
              best_d2 = d2;
              best_j = j;
            }
          }
        }
      }
      if (best_j < 0 || best_d2 > 4.5 * rmax2) break;  // ring exhausted, or every remaining clip is a no-op
      last_d2 = best_d2;
      last_j = best_j;
      const double qxj = g.c[2 * best_j], qyj = g.c[2 * best_j + 1];
      const int nn = vor_clip(px, py, n, (ownx + qxj) / 2, (owny + qyj) / 2, qxj - ownx, qyj - owny, qx, qy, capv);
      if (nn < 0) return VOR_OVERFLOW;
      for (int i = 0; i < nn; ++i) {
        px[i] = qx[i];
        py[i] = qy[i];
      }
      n = nn;
      rmax2 = 0.0;
      for (int i = 0; i < n; ++i) {
        const double r2 = (px[i] - ownx) * (px[i] - ownx) + (py[i] - owny) * (py[i] - owny);
        rmax2 = r2 > rmax2 ? r2 : rmax2;
      }
    }
    if (n == 0) break;
    const double h = g.h;
    const double ax0 = ownx - (-K + (cx - ring) * h), ax1 = (-K + (cx + ring + 1) * h) - ownx;
    const double ay0 = owny - (-K + (cy - ring) * h), ay1 = (-K + (cy + ring + 1) * h) - owny;
    const double dxm = ax0 < ax1 ? ax0 : ax1, dym = ay0 < ay1 ? ay0 : ay1;
    const double reach = dxm < dym ? dxm : dym;
    const bool covers_all = cx - ring <= 0 && cy - ring <= 0 && cx + ring >= g.G - 1 && cy + ring >= g.G - 1;
    if (covers_all || 4.0 * rmax2 <= reach * reach) break;
  }
  double acc = 0.0;
  for (int i = 0; i < n; ++i) {
    const int j = (i + 1) % n;
    acc += px[i] * py[j] - px[j] * py[i];
  }
  *mu = 0.5 * fabs(acc);
  return VOR_OK;
}
