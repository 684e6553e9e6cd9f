/*
 * opc_oracle.c -- scalar float64 C restatement of the reference's OPC front-end.
 * TEST INFRASTRUCTURE ONLY (checker for tests/, smoke(), bench.py cpu_baseline).
 * The product library (libopcfe.so) never links or calls this code.
 *
 * Compiled with -O2 -ffp-contract=off (as the reference's setup.py:24-26) so the
 * float64 arithmetic follows the reference's operation order without FMA
 * contraction.  Rows are independent within one iteration, so OpenMP over rows
 * leaves every result bit-identical to the single-threaded run.
 *
 * Reference (paths relative to /root/reference/pkg/src/flatpoly):
 *   oracle_laplacian   <- _kernels/_native.pyx:225-284 (semantics _fallback.py:82-117)
 *   oracle_bilateral   <- _kernels/_native.pyx:287-364 (semantics _fallback.py:120-166)
 *   oracle_fc_data     <- smoothing.py:61-88
 *   oracle_triangulate <- mesh.py:58-96 (trimap/triangles) + mesh.py:99-135 (twins)
 *   oracle_tri_normals <- geometry.py:134-147
 *   oracle_max_edge    <- segmentation.py:59-67,73
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static int finite3(const double *p) {
  return isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2]);
}

/* in/out: (M, N, 3) contiguous; tmp: scratch of the same size. Result in out. */
void oracle_laplacian(const double *in, double *out, double *tmp, int M, int N,
                      double lam, int ksize, int iters) {
  const int h = ksize / 2;
  const size_t n = (size_t)M * N * 3;
  double *bufs[2] = {out, tmp};
  /* pick the first destination so that the last iteration lands in `out` */
  int dst = (iters % 2 == 1) ? 0 : 1;
  const double *src = in;
  for (int it = 0; it < iters; ++it) {
    double *d = bufs[dst];
#pragma omp parallel for schedule(static)
    for (int u = 0; u < M; ++u) {
      for (int v = 0; v < N; ++v) {
        const double *p = src + ((size_t)u * N + v) * 3;
        double *q = d + ((size_t)u * N + v) * 3;
        q[0] = p[0]; q[1] = p[1]; q[2] = p[2];
        if (u == 0 || v == 0 || u == M - 1 || v == N - 1) continue;
        if (!finite3(p)) continue;
        double ws = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
        for (int du = -h; du <= h; ++du) {
          int uu = u + du;
          if (uu < 0 || uu >= M) continue;
          for (int dv = -h; dv <= h; ++dv) {
            int vv = v + dv;
            if ((du == 0 && dv == 0) || vv < 0 || vv >= N) continue;
            const double *r = src + ((size_t)uu * N + vv) * 3;
            double dx = r[0] - p[0], dy = r[1] - p[1], dz = r[2] - p[2];
            double dist = sqrt(dx * dx + dy * dy + dz * dz);
            if (!(dist > 0.0) || isnan(dist)) continue;
            double w = 1.0 / dist;
            ax += dx * w; ay += dy * w; az += dz * w;
            ws += w;
          }
        }
        if (ws > 0.0) {
          double s = lam / ws;
          q[0] = p[0] + s * ax; q[1] = p[1] + s * ay; q[2] = p[2] + s * az;
        }
      }
    }
    src = d;
    dst ^= 1;
  }
  if (iters == 0) memcpy(out, in, n * sizeof(double));
}

static void cross_unit(const double *a, const double *b, const double *c, double *n) {
  double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
  double e2x = c[0] - a[0], e2y = c[1] - a[1], e2z = c[2] - a[2];
  double x = e1y * e2z - e1z * e2y;
  double y = e1z * e2x - e1x * e2z;
  double z = e1x * e2y - e1y * e2x;
  double nrm = sqrt((x * x + y * y) + z * z);
  if (nrm > 0.0) {
    n[0] = x / nrm; n[1] = y / nrm; n[2] = z / nrm;
  } else {
    n[0] = n[1] = n[2] = NAN;
  }
}

/* opc (M,N,3) -> centroids, normals (M-1, N-1, 2, 3) */
void oracle_fc_data(const double *opc, int M, int N, double *cen, double *nrm) {
  const int Nq = N - 1;
#pragma omp parallel for schedule(static)
  for (int u = 0; u < M - 1; ++u) {
    for (int v = 0; v < Nq; ++v) {
      const double *p1 = opc + ((size_t)u * N + v) * 3;
      const double *p2 = p1 + 3;
      const double *p4 = p1 + (size_t)N * 3;
      const double *p3 = p4 + 3;
      const double *tri[2][3] = {{p3, p2, p1}, {p1, p4, p3}};
      for (int k = 0; k < 2; ++k) {
        size_t o = (((size_t)u * Nq + v) * 2 + k) * 3;
        const double *a = tri[k][0], *b = tri[k][1], *c = tri[k][2];
        for (int j = 0; j < 3; ++j) cen[o + j] = ((a[j] + b[j]) + c[j]) / 3.0;
        cross_unit(a, b, c, nrm + o);
      }
    }
  }
}

/* centroids/normals (Mq,Nq,2,3); result in out (same shape); tmp scratch. */
void oracle_bilateral(const double *cen, const double *nrm_in, double *out, double *tmp,
                      int Mq, int Nq, double sl, double sa, int ksize, int iters) {
  const int h = ksize / 2;
  const double ic = 1.0 / (2.0 * sl * sl), is = 1.0 / (2.0 * sa * sa);
  double *bufs[2] = {out, tmp};
  int dst = (iters % 2 == 1) ? 0 : 1;
  const double *cur = nrm_in;
  for (int it = 0; it < iters; ++it) {
    double *nx = bufs[dst];
#pragma omp parallel for schedule(static)
    for (int u = 0; u < Mq; ++u) {
      for (int v = 0; v < Nq; ++v) {
        for (int k = 0; k < 2; ++k) {
          size_t o = (((size_t)u * Nq + v) * 2 + k) * 3;
          const double *n0 = cur + o, *c0 = cen + o;
          nx[o] = n0[0]; nx[o + 1] = n0[1]; nx[o + 2] = n0[2];
          if (isnan(n0[0]) || isnan(n0[1]) || isnan(n0[2])) continue;
          double ws = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
          for (int du = -h; du <= h; ++du) {
            int uu = u + du;
            if (uu < 0 || uu >= Mq) continue;
            for (int dv = -h; dv <= h; ++dv) {
              int vv = v + dv;
              if (vv < 0 || vv >= Nq) continue;
              for (int kk = 0; kk < 2; ++kk) {
                if (du == 0 && dv == 0 && kk == k) continue;
                size_t q = (((size_t)uu * Nq + vv) * 2 + kk) * 3;
                const double *m = cur + q, *c1 = cen + q;
                if (isnan(m[0]) || isnan(m[1]) || isnan(m[2])) continue;
                double dx = c1[0] - c0[0], dy = c1[1] - c0[1], dz = c1[2] - c0[2];
                double dc2 = dx * dx + dy * dy + dz * dz;
                dx = m[0] - n0[0]; dy = m[1] - n0[1]; dz = m[2] - n0[2];
                double dn2 = dx * dx + dy * dy + dz * dz;
                double w = exp(-dc2 * ic - dn2 * is);
                ax += m[0] * w; ay += m[1] * w; az += m[2] * w;
                ws += w;
              }
            }
          }
          double len = sqrt(ax * ax + ay * ay + az * az);
          if (ws > 0.0 && len > 1e-30) {
            nx[o] = ax / len; nx[o + 1] = ay / len; nx[o + 2] = az / len;
          }
        }
      }
    }
    cur = nx;
    dst ^= 1;
  }
  if (iters == 0) memcpy(out, nrm_in, (size_t)Mq * Nq * 6 * sizeof(double));
}

/* Validity from the NaN mask; trimap (G), triangles (cap 3G), twins (cap 3G).
 * Returns the number of valid triangles. */
int64_t oracle_triangulate(const double *opc, int M, int N, int64_t *trimap,
                           int64_t *tris, int64_t *he) {
  const int Mq = M - 1, Nq = N - 1;
  const int64_t G = 2LL * Mq * Nq;
  int64_t t = 0;
  for (int u = 0; u < Mq; ++u) {
    for (int v = 0; v < Nq; ++v) {
      const double *p1 = opc + ((size_t)u * N + v) * 3;
      int ok1 = finite3(p1), ok2 = finite3(p1 + 3);
      int ok4 = finite3(p1 + (size_t)N * 3), ok3 = finite3(p1 + (size_t)N * 3 + 3);
      int64_t g = 2LL * ((int64_t)u * Nq + v);
      int64_t i1 = (int64_t)u * N + v, i2 = i1 + 1, i4 = i1 + N, i3 = i4 + 1;
      if (ok1 && ok2 && ok3) {
        trimap[g] = t;
        tris[3 * t] = i3; tris[3 * t + 1] = i2; tris[3 * t + 2] = i1;
        ++t;
      } else {
        trimap[g] = -1;
      }
      if (ok1 && ok3 && ok4) {
        trimap[g + 1] = t;
        tris[3 * t] = i1; tris[3 * t + 1] = i4; tris[3 * t + 2] = i3;
        ++t;
      } else {
        trimap[g + 1] = -1;
      }
    }
  }
  (void)G;
  for (int u = 0; u < Mq; ++u) {
    for (int v = 0; v < Nq; ++v) {
      int64_t g = 2LL * ((int64_t)u * Nq + v);
      /* neighbour GIDs per (k, edge): mesh.py:129-134 */
      int64_t nb[2][3];
      nb[0][0] = (v + 1 < Nq) ? g + 3 : -1;                     /* (u, v+1, 1) */
      nb[0][1] = (u > 0) ? g - 2LL * Nq + 1 : -1;               /* (u-1, v, 1) */
      nb[0][2] = g + 1;                                         /* (u, v, 1)   */
      nb[1][0] = (v > 0) ? g - 2 : -1;                          /* (u, v-1, 0) */
      nb[1][1] = (u + 1 < Mq) ? g + 2LL * Nq : -1;              /* (u+1, v, 0) */
      nb[1][2] = g;                                             /* (u, v, 0)   */
      for (int k = 0; k < 2; ++k) {
        int64_t tt = trimap[g + k];
        if (tt < 0) continue;
        for (int e = 0; e < 3; ++e) {
          int64_t n = nb[k][e];
          int64_t tn = (n >= 0) ? trimap[n] : -1;
          he[3 * tt + e] = (tn >= 0) ? 3 * tn + e : -1;
        }
      }
    }
  }
  return t;
}

void oracle_tri_normals(const double *pts, const int64_t *tris, int64_t T, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    cross_unit(pts + 3 * tris[3 * t], pts + 3 * tris[3 * t + 1], pts + 3 * tris[3 * t + 2],
               out + 3 * t);
  }
}

static double edge_len(const double *p, const double *q) {
  double dx = q[0] - p[0], dy = q[1] - p[1], dz = q[2] - p[2];
  return sqrt((dx * dx + dy * dy) + dz * dz);
}

/* ---- FastGA cell search: sfc.py:46-104 (s2_id) + _kernels/_fallback.py:14-44 (find_cells) */
#ifndef M_PI
#define M_PI 3.14159265358979323846 /* == numpy.pi as a double */
#endif
#define HB_ORDER 30
static const int64_t HB_GRID = (int64_t)1 << HB_ORDER;
/* face chain -y, +x, +z, -x, -z, +y: (u axis, v axis, swap, neg_u, neg_v) (sfc.py:24-31) */
static const int FACE_U[6] = {0, 1, 0, 1, 0, 0}, FACE_V[6] = {2, 2, 1, 2, 1, 2};
static const int FACE_SWAP[6] = {0, 1, 0, 1, 1, 0}, FACE_NEGU[6] = {0, 0, 1, 1, 0, 0};
/* axis*2 + (sign<0) -> face (sfc.py:34-36) */
static const int FACE_OF[6] = {1, 3, 5, 0, 2, 4};

static int64_t hb_quantize(double t) {
  double a = atan(t) * (4.0 / M_PI);
  double f = floor((a + 1.0) * 0.5 * (double)HB_GRID);
  int64_t i = (int64_t)f;
  return i < 0 ? 0 : (i > HB_GRID - 1 ? HB_GRID - 1 : i);
}

static int64_t hb_d(int64_t x, int64_t y) { /* sfc.py:46-61 */
  int64_t d = 0;
  for (int64_t s = HB_GRID >> 1; s > 0; s >>= 1) {
    int64_t rx = (x & s) > 0, ry = (y & s) > 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) { x = s - 1 - x; y = s - 1 - y; }
      int64_t t = x; x = y; y = t;
    }
  }
  return d;
}

uint64_t oracle_s2id(const double *q) {
  double nrm = sqrt((q[0] * q[0] + q[1] * q[1]) + q[2] * q[2]);
  double n[3] = {q[0] / nrm, q[1] / nrm, q[2] / nrm};
  int ax = 0; /* argmax |n| (first max) */
  if (fabs(n[1]) > fabs(n[ax])) ax = 1;
  if (fabs(n[2]) > fabs(n[ax])) ax = 2;
  double dom = n[ax];
  int face = FACE_OF[ax * 2 + (dom < 0)];
  double u = n[FACE_U[face]] / fabs(dom), v = n[FACE_V[face]] / fabs(dom);
  int64_t iu = hb_quantize(u), iv = hb_quantize(v);
  if (FACE_SWAP[face]) { int64_t t = iu; iu = iv; iv = t; }
  if (FACE_NEGU[face]) iu = HB_GRID - 1 - iu;
  return ((uint64_t)face << (2 * HB_ORDER)) | (uint64_t)hb_d(iu, iv);
}

void oracle_find_cells(const double *q, int64_t n, const uint64_t *ids, const double *cn,
                       const int64_t *nbrs, int64_t ncell, double slope, double icpt, int64_t wlo,
                       int64_t whi, int64_t *out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    const double *qi = q + 3 * i;
    uint64_t id = oracle_s2id(qi);
    int64_t kp = (int64_t)rint(slope * (double)id + icpt);
    int64_t lo = kp + wlo, hi = kp + whi;
    lo = lo < 0 ? 0 : (lo > ncell - 1 ? ncell - 1 : lo);
    hi = hi < 0 ? 0 : (hi > ncell - 1 ? ncell - 1 : hi);
    int64_t a = 0, b = ncell; /* searchsorted left */
    while (a < b) { int64_t m = (a + b) / 2; if (ids[m] < id) a = m + 1; else b = m; }
    int64_t ch = a < lo ? lo : (a > hi ? hi : a);
    int64_t cl = a - 1 < lo ? lo : (a - 1 > hi ? hi : a - 1);
    uint64_t dh = ids[ch] > id ? ids[ch] - id : id - ids[ch];
    uint64_t dl = ids[cl] > id ? ids[cl] - id : id - ids[cl];
    int64_t j = dl <= dh ? cl : ch;
    int64_t best = j;
    double bd = INFINITY;
    for (int k = -1; k < 12; ++k) {
      int64_t c = k < 0 ? j : nbrs[12 * j + k];
      if (c < 0) continue;
      double dx = cn[3 * c] - qi[0], dy = cn[3 * c + 1] - qi[1], dz = cn[3 * c + 2] - qi[2];
      double d2 = (dx * dx + dy * dy) + dz * dz;
      if (d2 < bd) { bd = d2; best = c; }
    }
    out[i] = best;
  }
}

/* group labels: segmentation.py:52-74.  Scores in the FMA order of numpy's BLAS matmul
 * (normals @ dn.T -> dgemm k-loop: fma(n2,d2, fma(n1,d1, n0*d0))); first maximum wins,
 * NaN maximal; 255 unless best >= ang_min; flag (nullable) forces 255. */
void oracle_group_assign(const double *nrm, int64_t T, const double *dn, int G, double ang_min,
                         const uint8_t *flag, uint8_t *labels) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const double *n = nrm + 3 * t;
    double best = fma(n[2], dn[2], fma(n[1], dn[1], n[0] * dn[0]));
    int arg = 0;
    for (int g = 1; g < G && !isnan(best); ++g) {
      double s = fma(n[2], dn[3 * g + 2], fma(n[1], dn[3 * g + 1], n[0] * dn[3 * g]));
      if (isnan(s) || s > best) { best = s; arg = g; }
    }
    uint8_t lab = (uint8_t)arg;
    if (!(best >= ang_min)) lab = 255;
    if (flag && flag[t]) lab = 255;
    labels[t] = lab;
  }
}

void oracle_max_edge(const double *pts, const int64_t *tris, int64_t T, double l_max,
                     uint8_t *flag) {
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < T; ++t) {
    const double *a = pts + 3 * tris[3 * t], *b = pts + 3 * tris[3 * t + 1],
                 *c = pts + 3 * tris[3 * t + 2];
    double lab = edge_len(a, b), lbc = edge_len(b, c), lca = edge_len(c, a);
    double m = fmax(lbc, lca);
    if (isnan(lbc) || isnan(lca)) m = NAN;
    double e = (isnan(lab) || isnan(m)) ? NAN : fmax(lab, m);
    flag[t] = (uint8_t)(e > l_max);
  }
}

/* Gather FC normals (G x 3) through trimap into mesh order: smoothing.py:108-114 */
void oracle_gather(const double *fc, const int64_t *trimap, int64_t G, double *out) {
  for (int64_t g = 0; g < G; ++g) {
    int64_t t = trimap[g];
    if (t < 0) continue;
    out[3 * t] = fc[3 * g]; out[3 * t + 1] = fc[3 * g + 1]; out[3 * t + 2] = fc[3 * g + 2];
  }
}
