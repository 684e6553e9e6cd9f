// Bilateral filtering of triangle normals on the fully-connected (FC) triangle grid,
// with the FC normal/centroid computation fused into the first iteration and the
// GID -> mesh-order scatter fused into the last one.
//
// Reference semantics:
//   * FC data (smoothing.py:61-88): triangle k of quad (u,v) = (p3,p2,p1) for k=0,
//     (p1,p4,p3) for k=1; centroid ((a+b)+c)/3; normal cross(b-a,c-a)/|.|, NaN
//     unless |.| > 0;
//   * one iteration (_fallback.py:120-166 == _native.pyx:287-364): for every
//     triangle with a finite normal, neighbours (u+du, v+dv, kk) in the (2h+1)^2
//     quad window (du, dv, kk order), self excluded, off-grid / NaN neighbours
//     skipped; w = exp(-|dc|^2/(2 sl^2) - |dn|^2/(2 sa^2)); n' = acc/|acc| if
//     wsum > 0 and |acc| > 1e-30 else n;
//   * gather to mesh order through trimap (smoothing.py:108-114).
//
// B200 mapping (issue-bound kernel: 15 FP32 ops + 1 MUFU per directed pair, 34 pairs
// per quad at k=3, against 60 B of HBM traffic per quad):
//   * one CTA = 32 x 16 quads, 256 threads, each thread 2 vertically adjacent quads
//     (both triangles of each), so a neighbour record loaded from shared memory feeds
//     up to 8 (own, neighbour) triangle pairs;
//   * PACKED FP32x2 math (sm_100 FADD2 / FMUL2 / FFMA2): the two triangles of a
//     neighbour quad are the two lanes of every packed register and the own triangle's
//     values enter as a broadcast scalar operand, so one issue slot does the work of two
//     pairs.  The FMA pipe still retires 128 FP32 ops / clk / SM (measured: FFMA and
//     FFMA2 streams both reach 125 / clk / SM), but the kernel was issue-bound (MUFU,
//     LDS and FP32 instructions share one issue slot per clk per SM sub-partition):
//     8.5 instead of 16 issue slots per pair;
//   * tile + halo arrive by TMA 3-D box loads with NaN out-of-bounds fill (== the
//     reference's "off-grid neighbours are skipped"): the point tile (centroids are
//     recomputed from points every iteration: 12 B/point instead of 24 B/quad of
//     stored centroids) and, after iteration 1, the previous normal tile;
//   * a pack step turns each halo quad into 3 float4 planes of (triangle 0, triangle 1)
//     lane pairs (conflict-free LDS.128): per triangle n' = n*sqrt(B), c' = c*sqrt(A)
//     with B, A the exponent scales pre-multiplied by log2(e), so
//     w = ex2(-(|c'_i - c'_j|^2 + |n'_i - n'_j|^2)).  Missing / NaN-normal triangles
//     carry n' = 0, c' = 1e18, so their weight to any valid triangle underflows to
//     exactly 0: no per-pair NaN test;
//   * iteration 1 computes FC normals with fp64 edges + cross product (no cancellation
//     on slivers) and an fp32 normalisation;
//   * the |acc| > 1e-30 test is evaluated underflow-safely.  Each own
//     triangle accumulates its kk = 0 and kk = 1 neighbours in the two packed lanes
//     (each in the reference's (du, dv) order) and adds the lanes at the end.
// Rejected variants (code in history, commit 22bf460): a pair-symmetric
// persistent kernel (half the weights; 127 registers -> 2 CTAs/SM, slower), a warp-
// specialised producer/consumer persistent kernel, a persistent kernel prefetching the
// next tile during compute (2.60 vs 2.26 ms), one quad per thread (2.77 ms) and the
// dot-product form of the normal term (exponent error ~B * 2^-24: 1.2e-5 at sa = 0.05).
#include "common.cuh"
#include "opcfe_internal.h"

#include <cmath>
#include <algorithm>
#include <cstdlib>

namespace opcfe {

namespace {

constexpr int kBilTQW = 32;  // interior quads per tile row (= one warp)
#ifndef OPCFE_BIL_TQH
#define OPCFE_BIL_TQH 8
#endif
constexpr int kBilTQH = OPCFE_BIL_TQH;  // interior quad rows per tile (A/B: -DOPCFE_BIL_TQH)
constexpr int kQPT = 2;                         // interior quads per thread (vertical)
constexpr int kBilNT = kBilTQW * kBilTQH / kQPT;  // threads per CTA
// resident CTAs the register budget targets: k = 3 -> 7 (72 registers; its packed kernel
// needs 17.7 KB of shared memory); larger windows have larger tiles (fewer CTAs by shared
// memory anyway) and more registers live
#ifndef OPCFE_BIL_BLOCKS3
#define OPCFE_BIL_BLOCKS3 7
#endif
constexpr int bil_min_blocks(int h) { return h == 1 ? OPCFE_BIL_BLOCKS3 : (h == 2 ? 5 : 4); }

enum BilMode : int {
  kFromPoints = 0,     // iteration 1: normals + centroids from the point grid
  kNormalsBuf = 1,     // normals from the previous iteration, centroids from points
  kNormalsCentBuf = 2,  // normals and centroids from FC arrays (drop-in bilateral_iterate)
  kFromPoints64 = 3     // fused iteration 1 of the mixed front end: FC data from the f64 grid
};

template <int H>
struct BilTile {
  // TMA rule (measured on B200): a box start along the innermost dimension must be
  // 16-B aligned.  FC rows are 24 B per quad -> the box starts LQ = round_up(H, 2)
  // quads left of the tile; point rows are 12 B per point -> LP = round_up(H, 4).
  static constexpr int LQ = (H + 1) / 2 * 2;
  static constexpr int LP = (H + 3) / 4 * 4;
  static constexpr int QW = ((LQ + kBilTQW + H + 1) / 2) * 2;      // FC box width (quads)
  static constexpr int QH = kBilTQH + 2 * H;
  static constexpr int PW = ((LP + kBilTQW + H + 1 + 3) / 4) * 4;  // point box width
  static constexpr int PH = QH + 1;
  static constexpr int PSHIFT = LP - LQ;  // point column of pack column 0
  static constexpr int NQ = QW * QH;      // quads in the pack
  // pack columns any weighing reads: [CB, CB + CW); the rest (16-B alignment padding of
  // the FC / packed boxes) are never packed
  static constexpr int CB = LQ - H;
  static constexpr int CW = kBilTQW + 2 * H;
  static_assert(CB >= 0 && CB + CW <= QW, "weighing window inside the pack");
  static constexpr int PTS_F = ((PW * 3 * PH) + 31) / 32 * 32;
  static constexpr int FC_F = ((QW * 6 * QH) + 31) / 32 * 32;
  // 4 pack planes (pack_quad), each 128-B aligned so TMA can fill them directly:
  //   C0 float4 (c'x0, c'x1, c'y0, c'y1)  C1 float2 (c'z0, c'z1)
  //   N0 float4 (n'x0, n'x1, n'y0, n'y1)  N1 float2 (n'z0, n'z1)
  static constexpr int P_C1 = (4 * NQ + 31) / 32 * 32;
  static constexpr int P_N0 = P_C1 + (2 * NQ + 31) / 32 * 32;
  static constexpr int P_N1 = P_N0 + (4 * NQ + 31) / 32 * 32;
  static constexpr int PACK_F = P_N1 + (2 * NQ + 31) / 32 * 32;
  static constexpr int OUT_F = kBilTQW * 6 * kBilTQH;
  static_assert(QW * 6 <= 256 && PW * 3 <= 256 && PH <= 256, "TMA box extent must be <= 256");
  static_assert((QW * 6) % 4 == 0, "FC box rows must be 16-B multiples");
  static_assert(FC_F >= OUT_F, "out tile aliases the FC normal tile");
};

// out tile: its own region in mode 0; aliases the (dead after packing) FC tile otherwise
template <int H, int MODE>
constexpr int bil_smem_bytes() {
  using T = BilTile<H>;
  if constexpr (MODE == kFromPoints64) return (2 * T::PTS_F + T::PACK_F) * 4 + kSmemSlack;
  return (((MODE != kNormalsCentBuf) ? T::PTS_F : 0) + ((MODE != kFromPoints) ? T::FC_F : 0) +
          ((MODE == kNormalsCentBuf) ? 2 * T::FC_F : 0) + T::PACK_F +  // f64 centroid tile
          ((MODE == kFromPoints) ? T::OUT_F : 0)) *
             4 +
         kSmemSlack;
}

struct BilArgs {
  int M, N;          // point grid (Mq = M-1, Nq = N-1 quads)
  int F;             // frames
  float sA, sB;      // sqrt(log2(e)/(2 sl^2)), sqrt(log2(e)/(2 sa^2))
  const int64_t* trimap;  // scatter mode: per frame [G]
  long long tm_fs;
  float* out_mesh;   // scatter destination: per frame [cap][3]
  double* out_mesh64;  // ... or float64 (the mixed-precision front end), when non-null
  long long out_fs;  // floats per frame
  long long n_out;   // rows per frame available in out_mesh (bounds check)
  const float* pts;  // point grid (packed scatter: exact rebuild of unchanged normals)
  int pitch;
  long long pts_fs;
  char* cwin;        // fused pipeline: per-tile centroid windows [F][gy][gx] (see below)
  long long wstride; // bytes per window
  int gx, gy;        // tile grid (kBilTQW x kBilTQH quads per tile)
};

// Centroids are handled relative to a per-tile origin o (the box's centre value, else the
// first finite one): an fp32 centroid far from the coordinate origin carries an absolute
// rounding of |c| * 2^-24, which the weight exponent would see as a relative error
// |c| h / sl^2 * 1.2e-7 (h the spacing) -- at 8.6 m with sl = 2 cm that broke the 1e-5
// contract.  Relative to o, the rounding scales with the tile extent instead.  Halo quads
// need the SAME origin, so the fused pipeline's iteration 1 stores each tile's whole packed
// centroid window (tile + halo, ~1.4x the quads) and later iterations bulk-load their own
// window: no re-basing, and the values equal what a pack from the points computes.
template <int NT, typename S>
__device__ __forceinline__ auto tile_origin(const S* v, int count, int stride, int* s_first) {
  if (threadIdx.x == 0) *s_first = 0x7fffffff;
  __syncthreads();
  for (int i = threadIdx.x; i < count; i += NT) {
    const S* q = v + i * stride;
    if (isfinite(q[0]) && isfinite(q[1]) && isfinite(q[2])) {
      atomicMin(s_first, i);
      break;
    }
  }
  __syncthreads();
  const int i = *s_first;
  if constexpr (sizeof(S) == 8)
    return i == 0x7fffffff ? make_double3(0.0, 0.0, 0.0)
                           : make_double3(v[i * stride], v[i * stride + 1], v[i * stride + 2]);
  else
    return i == 0x7fffffff ? make_float3(0.f, 0.f, 0.f)
                           : make_float3(v[i * stride], v[i * stride + 1], v[i * stride + 2]);
}

// centroid of triangle k of pack quad (r, c) from the f64 point box (mode 3): the mixed FC
// data's ((a + b) + c) * (1/3), triangles (p3, p2, p1) and (p1, p4, p3)
template <int H>
__device__ __forceinline__ void fc64_centroid_t(const double* pts, int r, int c, int k, double* out) {
  using T = BilTile<H>;
  const double* P1 = pts + (r * T::PW + c + T::PSHIFT) * 3;
  const double* P2 = P1 + 3;
  const double* P4 = P1 + T::PW * 3;
  const double* P3 = P4 + 3;
  const double* A = k == 0 ? P3 : P1;
  const double* B = k == 0 ? P2 : P4;
  const double* C = k == 0 ? P1 : P3;
#pragma unroll
  for (int j = 0; j < 3; ++j) out[j] = mixed_centroid(A[j], B[j], C[j]);
}

// FC normals of a quad's two triangles (p3, p2, p1) and (p1, p4, p3) for the bilateral
// input: edges and cross products in fp64 (exact edge differences of fp32 vertices; no
// cancellation on slivers), normalisation in fp32.  Each vertex is converted to fp64 once
// and the shared diagonal p1 - p3 is formed once (12 conversions + 9 subtractions per quad
// instead of 18 + 12); the fp32 normalisation uses MUFU rcp / rsqrt + one Newton step
// instead of IEEE divide / sqrt (whose slow-path checks dominated the pack phase).
// |n - float32(reference)| ~ 1e-7, far inside the 1e-5 contract, at a fraction of the
// cost of the correctly rounded fp64 divide/sqrt used where bit-exact normals are
// returned (gridops.cu).  Tiny triangles (|cross| below the fp32 normal range, i.e.
// vertices closer than ~1e-19 m) are out of contract.
__device__ __forceinline__ void fc_normals_quad(const float* P1, const float* P2, const float* P3,
                                                const float* P4, float* n) {
  double d13[3], e1f[3], e1s[3];  // p1 - p3; first e1 = p2 - p3; second e1 = p4 - p1
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double p1 = P1[j], p3 = P3[j];
    d13[j] = p1 - p3;
    e1f[j] = (double)P2[j] - p3;
    e1s[j] = (double)P4[j] - p1;
  }
  // first: cross(p2 - p3, p1 - p3); second: cross(p4 - p1, p3 - p1) = -cross(e1s, d13).
  // Products and differences rounded separately (numpy's np.cross, no FMA contraction): a
  // triangle with two coincident vertices has an exactly zero cross product -> NaN normal,
  // as in the reference (a contracted FMA leaves the rounding error of one product).
  normalise_fast(dsub(dmul(e1f[1], d13[2]), dmul(e1f[2], d13[1])),
                 dsub(dmul(e1f[2], d13[0]), dmul(e1f[0], d13[2])),
                 dsub(dmul(e1f[0], d13[1]), dmul(e1f[1], d13[0])), n);
  normalise_fast(dsub(dmul(e1s[2], d13[1]), dmul(e1s[1], d13[2])),
                 dsub(dmul(e1s[0], d13[2]), dmul(e1s[2], d13[0])),
                 dsub(dmul(e1s[1], d13[0]), dmul(e1s[0], d13[1])), n + 3);
}


// the 4 pack planes (in shared memory, or the global packed FC arrays of the fused
// pipeline): one quad = (triangle 0, triangle 1) lane pairs, 48 B
struct Planes {
  float4* c0;
  float2* c1;
  float4* n0;
  float2* n1;
};
template <int H>
__device__ __forceinline__ Planes planes_at(float* base) {
  using T = BilTile<H>;
  return Planes{reinterpret_cast<float4*>(base), reinterpret_cast<float2*>(base + T::P_C1),
                reinterpret_cast<float4*>(base + T::P_N0),
                reinterpret_cast<float2*>(base + T::P_N1)};
}

// pack one quad: n' = n*sqrt(B); `cs` are the centroids already scaled (c' = c*sqrt(A));
// a triangle with a NaN normal or centroid is encoded as n' = 0, c' = 1e18 (its weight
// to / from any valid triangle underflows to exactly 0).  One NaN test per triangle: on
// the sum of its six values (an infinite value either yields NaN or a zero weight) -- or,
// for normals computed here from the points (FC), on one component: such a normal is NaN
// in all three or in none, and a NaN vertex (NaN centroid) makes it NaN.
template <bool FC>
__device__ __forceinline__ void pack_quad(const Planes& P, int q, const float* n,
                                          const float* cs, float sB) {
  float c2[2][3], n2[2][3];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float t = FC ? n[3 * k]
                       : ((n[3 * k] + n[3 * k + 1]) + (n[3 * k + 2] + cs[3 * k])) +
                             (cs[3 * k + 1] + cs[3 * k + 2]);
    const bool ok = !isnan(t);
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      n2[k][j] = ok ? n[3 * k + j] * sB : 0.f;
      c2[k][j] = ok ? cs[3 * k + j] : 1e18f;
    }
  }
  P.c0[q] = make_float4(c2[0][0], c2[1][0], c2[0][1], c2[1][1]);
  P.c1[q] = make_float2(c2[0][2], c2[1][2]);
  P.n0[q] = make_float4(n2[0][0], n2[1][0], n2[0][1], n2[1][1]);
  P.n1[q] = make_float2(n2[0][2], n2[1][2]);
}

// a quad as 6 packed (tri 0, tri 1) registers: LDS.128 + LDS.64 + LDS.128 + LDS.64
struct Quad2 {
  f2_t cx, cy, cz, nx, ny, nz;
};
__device__ __forceinline__ Quad2 load_quad2(const Planes& P, int q) {
  const ulonglong2 a = reinterpret_cast<const ulonglong2*>(P.c0)[q];
  const f2_t cz = reinterpret_cast<const f2_t*>(P.c1)[q];
  const ulonglong2 b = reinterpret_cast<const ulonglong2*>(P.n0)[q];
  const f2_t nz = reinterpret_cast<const f2_t*>(P.n1)[q];
  return Quad2{a.x, a.y, cz, b.x, b.y, nz};
}

// an own triangle, NEGATED (so differences are packed adds with a broadcast operand)
struct OwnTri {
  float cx, cy, cz, nx, ny, nz;
};
__device__ __forceinline__ OwnTri own_tri(const Quad2& q, int k) {
  auto lane = [&](f2_t r) { return k == 0 ? f2lo(r) : f2hi(r); };
  return OwnTri{-lane(q.cx), -lane(q.cy), -lane(q.cz), -lane(q.nx), -lane(q.ny), -lane(q.nz)};
}

// |x'_j - x'_i|^2 for the two triangles j of a neighbour quad against own triangle i
__device__ __forceinline__ f2_t dist2(const OwnTri& t, const Quad2& nb) {
  const f2_t dx = add2(nb.cx, bc2(t.cx)), dy = add2(nb.cy, bc2(t.cy)), dz = add2(nb.cz, bc2(t.cz));
  const f2_t ex = add2(nb.nx, bc2(t.nx)), ey = add2(nb.ny, bc2(t.ny)), ez = add2(nb.nz, bc2(t.nz));
  f2_t s = mul2(dx, dx);
  s = fma2(dy, dy, s);
  s = fma2(dz, dz, s);
  s = fma2(ex, ex, s);
  s = fma2(ey, ey, s);
  return fma2(ez, ez, s);
}

// Weigh one thread's two quads: a = pack row R0, b = R0 + 1, pack column C.  res holds
// the filtered unit normals where upd[o][k]; qa / qb are the thread's own packed quads.
template <int H>
__device__ __forceinline__ void bil_weigh(const Planes& P, int R0, int C, float sB, Quad2& qa,
                                          Quad2& qb, float res[2][6], bool upd[2][2]) {
  using T = BilTile<H>;
  qa = load_quad2(P, R0 * T::QW + C);
  qb = load_quad2(P, (R0 + 1) * T::QW + C);
  const OwnTri own[2][2] = {{own_tri(qa, 0), own_tri(qa, 1)}, {own_tri(qb, 0), own_tri(qb, 1)}};
  f2_t acc[2][2][3];  // [own quad][own triangle][x, y, z] x (kk = 0, kk = 1) lanes
#pragma unroll
  for (int o = 0; o < 2; ++o)
#pragma unroll
    for (int k = 0; k < 2; ++k) acc[o][k][0] = acc[o][k][1] = acc[o][k][2] = 0ull;

  // (1) pairs inside the thread, weighed once: w(i,j) = w(j,i).
  //   intra-quad (tri 0, tri 1) of a and of b: one scalar weight each
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const Quad2& q = o == 0 ? qa : qb;
    const OwnTri& t0 = own[o][0];
    const OwnTri& t1 = own[o][1];
    const float dx = t1.cx - t0.cx, dy = t1.cy - t0.cy, dz = t1.cz - t0.cz;
    const float ex = t1.nx - t0.nx, ey = t1.ny - t0.ny, ez = t1.nz - t0.nz;
    float e = dx * dx;
    e = fmaf(dy, dy, e);
    e = fmaf(dz, dz, e);
    e = fmaf(ex, ex, e);
    e = fmaf(ey, ey, e);
    e = fmaf(ez, ez, e);
    const float w = ex2_approx(-e);
    // tri 1 <- tri 0 into lane kk = 0, tri 0 <- tri 1 into lane kk = 1: one scalar FMA per
    // component (the other lane is untouched)
    auto lo_fma = [&](f2_t n, f2_t& a) { a = f2(fmaf(f2lo(n), w, f2lo(a)), f2hi(a)); };
    auto hi_fma = [&](f2_t n, f2_t& a) { a = f2(f2lo(a), fmaf(f2hi(n), w, f2hi(a))); };
    lo_fma(q.nx, acc[o][1][0]);
    lo_fma(q.ny, acc[o][1][1]);
    lo_fma(q.nz, acc[o][1][2]);
    hi_fma(q.nx, acc[o][0][0]);
    hi_fma(q.ny, acc[o][0][1]);
    hi_fma(q.nz, acc[o][0][2]);
  }
  //   vertical a-b: a's triangle k against b's pair (lanes kk), shared with b
  {
    f2_t wv[2];
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const f2_t sd = dist2(own[0][k], qb);
      wv[k] = f2(ex2_approx(-f2lo(sd)), ex2_approx(-f2hi(sd)));
      acc[0][k][0] = fma2(qb.nx, wv[k], acc[0][k][0]);
      acc[0][k][1] = fma2(qb.ny, wv[k], acc[0][k][1]);
      acc[0][k][2] = fma2(qb.nz, wv[k], acc[0][k][2]);
    }
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {  // b's triangle kk <- a's pair (lanes k)
      const f2_t w = kk == 0 ? f2(f2lo(wv[0]), f2lo(wv[1])) : f2(f2hi(wv[0]), f2hi(wv[1]));
      acc[1][kk][0] = fma2(qa.nx, w, acc[1][kk][0]);
      acc[1][kk][1] = fma2(qa.ny, w, acc[1][kk][1]);
      acc[1][kk][2] = fma2(qa.nz, w, acc[1][kk][2]);
    }
  }

  // (2) every other quad of the two windows
#pragma unroll
  for (int dr = -H; dr <= H + 1; ++dr) {
#pragma unroll
    for (int dc = -H; dc <= H; ++dc) {
      if (dc == 0 && (dr == 0 || dr == 1)) continue;  // a and b themselves: (1)
      const Quad2 nb = load_quad2(P, (R0 + dr) * T::QW + C + dc);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int du = dr - o;
        if (du < -H || du > H) continue;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const f2_t sd = dist2(own[o][k], nb);
          const f2_t w = f2(ex2_approx(-f2lo(sd)), ex2_approx(-f2hi(sd)));
          acc[o][k][0] = fma2(nb.nx, w, acc[o][k][0]);
          acc[o][k][1] = fma2(nb.ny, w, acc[o][k][1]);
          acc[o][k][2] = fma2(nb.nz, w, acc[o][k][2]);
        }
      }
    }
  }

  // underflow-safe normalisation: n = m/|m|, m = acc'/s; |acc| > 1e-30 <=> |m| s > 1e-30 sB.
  // wsum is not accumulated: wsum == 0 implies acc == 0, so the reference's
  // `wsum > 0 and |acc| > 1e-30` (_native.pyx:352-360) is just |acc| > 1e-30, here
  // |acc'| > 1e-30 sqrt(B) evaluated underflow-safely as s * |acc'/s|, s = max |acc'_i|
  const float thr = 1e-30f * sB;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float* r = &res[o][3 * k];
      const bool valid = own[o][k].cx != -1e18f;  // not the pack sentinel
      const float ax = f2lo(acc[o][k][0]) + f2hi(acc[o][k][0]);
      const float ay = f2lo(acc[o][k][1]) + f2hi(acc[o][k][1]);
      const float az = f2lo(acc[o][k][2]) + f2hi(acc[o][k][2]);
      upd[o][k] = false;
      r[0] = r[1] = r[2] = 0.f;
      // |acc'|^2 inside [2^-120, 2^120] (the usual case): normalise directly, and |acc'| >=
      // 2^-60 > thr, so the triangle moves.  Outside (rare): rescale by max |acc'_i| first.
      // MUFU rsqrt + one Newton step (~1 ulp, like IEEE sqrt + divide, whose slow-path
      // checks cost ~8 % of the kernel's instructions).
      const float d2 = fmaf(az, az, fmaf(ay, ay, ax * ax));
      if (valid && d2 >= 7.5231638e-37f && d2 <= 1.329228e36f) {
        float il = rsqrt_approx(d2);
        il = il * fmaf(-0.5f * d2, il * il, 1.5f);
        r[0] = ax * il;
        r[1] = ay * il;
        r[2] = az * il;
        upd[o][k] = true;
      } else {
        const float sc = fmaxf(fabsf(ax), fmaxf(fabsf(ay), fabsf(az)));
        if (valid && sc > 0.f) {
          const float is = rcp_approx(sc);  // a common scale: cancels in the normalisation
          const float mx = ax * is, my = ay * is, mz = az * is;
          const float l2 = mx * mx + my * my + mz * mz;  // in [1, 3]
          float il = rsqrt_approx(l2);
          il = il * fmaf(-0.5f * l2, il * il, 1.5f);
          if (l2 * il * sc > thr) {
            r[0] = mx * il;
            r[1] = my * il;
            r[2] = mz * il;
            upd[o][k] = true;
          }
        }
      }
    }
  }
}

// the fused pipeline's packed FC arrays in global memory (per frame, row-major quads):
// C0 / N0 float4 [Mq][Nq], C1 / N1 float2 [Mq][Nq2] (Nq2 = Nq rounded up to even)
struct PackedG {  // the packed normal planes N0 / N1 of the fused pipeline
  float4* n0;
  float2* n1;
  long long s4, s2;    // row strides in quads (Nq, Nq2)
  long long f4, f2s;   // frame strides in quads
};

__device__ __forceinline__ void store_packed_n(const PackedG& g, int f, int u, int v,
                                               const float* res, const bool* upd,
                                               const Quad2& own, float sB) {
  // n' of the next iteration: the filtered normal * sqrt(B); unchanged -> the input n'
  // (exactly, already scaled); invalid (sentinel) -> 0
  float n[6];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const float inx = k == 0 ? f2lo(own.nx) : f2hi(own.nx);
    const float iny = k == 0 ? f2lo(own.ny) : f2hi(own.ny);
    const float inz = k == 0 ? f2lo(own.nz) : f2hi(own.nz);
    n[3 * k] = upd[k] ? res[3 * k] * sB : inx;
    n[3 * k + 1] = upd[k] ? res[3 * k + 1] * sB : iny;
    n[3 * k + 2] = upd[k] ? res[3 * k + 2] * sB : inz;
  }
  g.n0[f * g.f4 + (long long)u * g.s4 + v] = make_float4(n[0], n[3], n[1], n[4]);
  g.n1[f * g.f2s + (long long)u * g.s2 + v] = make_float2(n[2], n[5]);
}

__device__ __forceinline__ void scatter_mesh(const BilArgs& a, int f, int u, int v,
                                             const float* r) {
  const int Nq = a.N - 1;
  const long long g = 2ll * ((long long)u * Nq + v);
  const longlong2 tm = *reinterpret_cast<const longlong2*>(a.trimap + f * a.tm_fs + g);
  auto put = [&](auto* dst) {
    if (tm.x >= 0 && tm.x < a.n_out) {
      dst[3 * tm.x] = r[0];
      dst[3 * tm.x + 1] = r[1];
      dst[3 * tm.x + 2] = r[2];
    }
    if (tm.y >= 0 && tm.y < a.n_out) {
      dst[3 * tm.y] = r[3];
      dst[3 * tm.y + 1] = r[4];
      dst[3 * tm.y + 2] = r[5];
    }
  };
  if (a.out_mesh64)  // uniform: the mixed front end's float64 normals
    put(a.out_mesh64 + f * a.out_fs);
  else
    put(a.out_mesh + f * a.out_fs);
}

// PACKOUT (mode 0, fused pipeline with >= 2 iterations): besides filtering, write the
// packed centroid planes (constant for all later iterations) and the packed filtered
// normals, so the later iterations (bilateral_packed_kernel) skip the pack phase.
template <int H, int MODE, bool SCATTER, bool PACKOUT>
__global__ void __launch_bounds__(kBilNT, bil_min_blocks(H))
    bilateral_kernel(const __grid_constant__ CUtensorMap tpts, const __grid_constant__ CUtensorMap tnrm,
                     const __grid_constant__ CUtensorMap tcen, const __grid_constant__ CUtensorMap tout,
                     BilArgs a, PackedG pg) {
  using T = BilTile<H>;
  static_assert(!PACKOUT || (MODE != kNormalsBuf && !SCATTER), "PACKOUT: mode 0 / 2 / 3, no scatter");
  static_assert(MODE != kFromPoints64 || PACKOUT, "mode 3 is the fused pipeline's iteration 1");
  constexpr bool P64 = MODE == kFromPoints64;
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp;
  float* p = reinterpret_cast<float*>(smem_aligned_base(smem_raw, &barp));
  float* pts_s = nullptr;
  float* nrm_s = nullptr;
  float* cen_s = nullptr;
  if (MODE != kNormalsCentBuf) { pts_s = p; p += (P64 ? 2 : 1) * T::PTS_F; }
  if (MODE != kFromPoints && !P64) { nrm_s = p; p += T::FC_F; }
  const double* pts_d = reinterpret_cast<const double*>(pts_s);  // mode 3: the f64 point box
  if (MODE == kNormalsCentBuf) { cen_s = p; p += 2 * T::FC_F; }  // float64 centroid tile
  const double* cen_d = reinterpret_cast<const double*>(cen_s);
  const Planes P = planes_at<H>(p);
  p += T::PACK_F;
  float* out_s = (MODE == kFromPoints) ? p : nrm_s;  // modes 1/2: aliases the FC tile
  uint64_t& bar = *barp;

  const int Mq = a.M - 1, Nq = a.N - 1;
  const int q0 = blockIdx.x * kBilTQW;   // first interior quad column
  const int u0 = blockIdx.y * kBilTQH;   // first interior quad row
  const int f = blockIdx.z;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    uint32_t bytes = 0;
    if (MODE != kNormalsCentBuf) bytes += T::PW * 3 * T::PH * (P64 ? 8 : 4);
    if (MODE != kFromPoints && !P64) bytes += T::QW * 6 * T::QH * 4;
    if (MODE == kNormalsCentBuf) bytes += T::QW * 6 * T::QH * 8;
    mbar_expect_tx(&bar, bytes);
    if (MODE != kNormalsCentBuf) tma_load_3d(pts_s, &tpts, &bar, (q0 - T::LP) * 3, u0 - H, f);
    if (MODE != kFromPoints && !P64) tma_load_3d(nrm_s, &tnrm, &bar, (q0 - T::LQ) * 6, u0 - H, f);
    if (MODE == kNormalsCentBuf) tma_load_3d(cen_s, &tcen, &bar, (q0 - T::LQ) * 6, u0 - H, f);
  }
  __syncthreads();  // barrier initialised (and its loads issued) before anyone waits
  const float sA = a.sA, sB = a.sB, sA3 = a.sA * (1.0f / 3.0f);
  const int tx = threadIdx.x % kBilTQW, ty = threadIdx.x / kBilTQW;
  const int R0 = kQPT * ty + H, C = tx + T::LQ;  // pack position of the thread's quad 0
  mbar_wait(&bar, 0);
  // tile origin: the box's centre value, or (rare, e.g. NaN there) the first finite one;
  // every thread reads the same shared value, so the fallback branch is uniform
  __shared__ int s_first;
  float3 o;
  double3 od;  // MODE 2: float64 centroids, origin and differences in fp64
  if constexpr (MODE == kNormalsCentBuf) {
    const double* cp = cen_d + ((T::QH / 2) * T::QW + T::QW / 2) * 6;
    od = make_double3(cp[0], cp[1], cp[2]);
    if (!(isfinite(od.x) && isfinite(od.y) && isfinite(od.z)))
      od = tile_origin<kBilNT>(cen_d, T::QW * T::QH * 2, 3, &s_first);
  } else if constexpr (P64) {
    // the same origin mode 2 takes from the FC arrays: the centroid of the box's centre
    // quad's triangle 0, else the first finite box centroid in (quad, triangle) order
    double c[3];
    fc64_centroid_t<H>(pts_d, T::QH / 2, T::QW / 2, 0, c);
    od = make_double3(c[0], c[1], c[2]);
    if (!(isfinite(od.x) && isfinite(od.y) && isfinite(od.z))) {
      if (threadIdx.x == 0) s_first = 0x7fffffff;
      __syncthreads();
      for (int i = threadIdx.x; i < T::QW * T::QH * 2; i += kBilNT) {
        fc64_centroid_t<H>(pts_d, (i / 2) / T::QW, (i / 2) % T::QW, i % 2, c);
        if (isfinite(c[0]) && isfinite(c[1]) && isfinite(c[2])) {
          atomicMin(&s_first, i);
          break;
        }
      }
      __syncthreads();
      const int i = s_first;
      if (i == 0x7fffffff) {
        od = make_double3(0.0, 0.0, 0.0);
      } else {
        fc64_centroid_t<H>(pts_d, (i / 2) / T::QW, (i / 2) % T::QW, i % 2, c);
        od = make_double3(c[0], c[1], c[2]);
      }
    }
  } else {
    const float* cp = pts_s + ((T::PH / 2) * T::PW + T::PW / 2) * 3;
    o = make_float3(cp[0], cp[1], cp[2]);
    if (!finite3f(o.x, o.y, o.z)) o = tile_origin<kBilNT>(pts_s, T::PW * T::PH, 3, &s_first);
  }

  // ---- pack every quad the weighing reads into the planes (scaled + sentinel-encoded)
  if constexpr (PACKOUT && T::CW < T::QW) {  // unread padding columns of the stored window: 0
    constexpr int PADW = T::QW - T::CW;
    for (int i = threadIdx.x; i < T::QH * PADW; i += kBilNT) {
      const int r = i / PADW, j = i % PADW, q = r * T::QW + (j < T::CB ? j : T::CW + j);
      P.c0[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      P.c1[q] = make_float2(0.f, 0.f);
    }
  }
  auto pack_at = [&](int r, int c) {
    const int q = r * T::QW + c;
    float n[6], cc[6];  // cc: scaled centroids c' = c * sqrt(A)
    if (MODE == kNormalsCentBuf) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        n[j] = nrm_s[q * 6 + j];
        const double oj = j % 3 == 0 ? od.x : (j % 3 == 1 ? od.y : od.z);
        cc[j] = (float)((cen_d[q * 6 + j] - oj) * (double)sA);
      }
    } else if constexpr (P64) {
      // fc_rows_kernel<true>'s arithmetic (mixed FC data), bit for bit, from the box
      const double* P1 = pts_d + (r * T::PW + c + T::PSHIFT) * 3;
      const double* P2 = P1 + 3;
      const double* P4 = P1 + T::PW * 3;
      const double* P3 = P4 + 3;
      const double* tri[2][3] = {{P3, P2, P1}, {P1, P4, P3}};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const double *A = tri[k][0], *B = tri[k][1], *Cc = tri[k][2];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double oj = j == 0 ? od.x : (j == 1 ? od.y : od.z);
          const double cen = mixed_centroid(A[j], B[j], Cc[j]);
          cc[3 * k + j] = (float)((cen - oj) * (double)sA);
        }
        double nx, ny, nz;
        fast_unit_normal_f64(A, B, Cc, nx, ny, nz);
        n[3 * k] = (float)nx;
        n[3 * k + 1] = (float)ny;
        n[3 * k + 2] = (float)nz;
      }
    } else {
      const float* P1 = pts_s + (r * T::PW + c + T::PSHIFT) * 3;
      const float* P2 = P1 + 3;
      const float* P4 = P1 + T::PW * 3;
      const float* P3 = P4 + 3;
      // triangles (p3, p2, p1) and (p1, p4, p3) share p1 + p3; relative to the tile origin
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float oj = j == 0 ? o.x : (j == 1 ? o.y : o.z);
        const float s13 = (P1[j] - oj) + (P3[j] - oj);
        cc[j] = (s13 + (P2[j] - oj)) * sA3;
        cc[3 + j] = (s13 + (P4[j] - oj)) * sA3;
      }
      if (MODE == kFromPoints) {
        fc_normals_quad(P1, P2, P3, P4, n);
      } else {
#pragma unroll
        for (int j = 0; j < 6; ++j) n[j] = nrm_s[q * 6 + j];
      }
      if (MODE == kFromPoints && !PACKOUT) {  // raw normals of interior quads: "unchanged"
        const int ir = r - H, ic = c - T::LQ;
        if (ir >= 0 && ir < kBilTQH && ic >= 0 && ic < kBilTQW) {
#pragma unroll
          for (int j = 0; j < 6; ++j) out_s[(ir * kBilTQW + ic) * 6 + j] = n[j];
        }
      }
    }
    pack_quad<MODE == kFromPoints>(P, q, n, cc, sB);
  };
  // a warp packs 32 consecutive quads of one row (no row wrap inside a warp: conflict-free
  // point loads and plane stores), then the last warps the 2H leftover columns of each row
  static_assert(T::CW >= kBilTQW && kBilTQW == 32, "row segments of one warp");
  for (int r = threadIdx.x / 32; r < T::QH; r += kBilNT / 32) pack_at(r, T::CB + threadIdx.x % 32);
  constexpr int LW = T::CW - kBilTQW;
  for (int j = kBilNT - 1 - threadIdx.x; j < T::QH * LW; j += kBilNT)
    pack_at(j / LW, T::CB + kBilTQW + j % LW);
  __syncthreads();
  if (PACKOUT && threadIdx.x == 0) {  // the tile's centroid window, for iterations 2..B
    char* win = a.cwin + (((long long)f * a.gy + blockIdx.y) * a.gx + blockIdx.x) * a.wstride;
    fence_proxy_async_smem();
    bulk_store(win, P.c0, T::NQ * 16);
    bulk_store(win + T::NQ * 16, P.c1, T::NQ * 8);
    tma_store_commit();
  }

  static_assert(kQPT == 2, "bil_weigh handles 2 quads per thread");
  Quad2 qa, qb;
  float res[2][6];
  bool upd[2][2];
  bil_weigh<H>(P, R0, C, sB, qa, qb, res, upd);

  if constexpr (PACKOUT) {
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const int u = u0 + kQPT * ty + o, v = q0 + tx;
      if (u < Mq && v < Nq) {
        const Quad2& q = o == 0 ? qa : qb;
        store_packed_n(pg, f, u, v, res[o], upd[o], q, sB);
      }
    }
    if (threadIdx.x == 0) tma_store_wait_read();  // the window left shared memory
  } else {
#pragma unroll
  for (int o = 0; o < kQPT; ++o) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!upd[o][k]) {  // unchanged (missing / isolated / |acc| <= 1e-30): the input normal
        float* r = &res[o][3 * k];
        const float* n = (MODE == kFromPoints)
                             ? out_s + ((kQPT * ty + o) * kBilTQW + tx) * 6 + 3 * k
                             : nrm_s + ((R0 + o) * T::QW + C) * 6 + 3 * k;
        r[0] = n[0];
        r[1] = n[1];
        r[2] = n[2];
      }
    }
  }

  if (SCATTER) {
#pragma unroll
    for (int o = 0; o < kQPT; ++o) {
      const int u = u0 + kQPT * ty + o, v = q0 + tx;
      if (u < Mq && v < Nq) scatter_mesh(a, f, u, v, res[o]);
    }
  } else {
    __syncthreads();  // every thread has read its raw normals (out tile aliases them)
#pragma unroll
    for (int o = 0; o < kQPT; ++o) {
      float* dst = out_s + ((kQPT * ty + o) * kBilTQW + tx) * 6;
#pragma unroll
      for (int j = 0; j < 6; ++j) dst[j] = res[o][j];
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_3d(&tout, out_s, q0 * 6, u0, f);
      tma_store_commit_and_wait();
    }
  }
  }  // !PACKOUT
}

// Iterations 2..B of the fused pipeline: the packed planes (constant centroids from
// iteration 1, the previous iteration's packed normals) arrive by four TMA boxes straight
// into the shared-memory planes -- no pack phase, no barrier after the load.  Off-grid
// halo quads are zero-filled by TMA: their n' = 0, so whatever their weight, they add
// nothing.  Unchanged outputs are the input n' exactly (scaled domain); the final scatter
// unscales (n'/sqrt(B): <= 1 ulp of the unit normal; NaN for the sentinel).
template <int H, bool SCATTER>
__global__ void __launch_bounds__(kBilNT, bil_min_blocks(H))
    bilateral_packed_kernel(const __grid_constant__ CUtensorMap tc0,
                            const __grid_constant__ CUtensorMap tc1,
                            const __grid_constant__ CUtensorMap tn0,
                            const __grid_constant__ CUtensorMap tn1, BilArgs a, PackedG out) {
  using T = BilTile<H>;
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp;
  float* p = reinterpret_cast<float*>(smem_aligned_base(smem_raw, &barp));
  const Planes P = planes_at<H>(p);
  uint64_t& bar = *barp;
  const int Mq = a.M - 1, Nq = a.N - 1;
  const int q0 = blockIdx.x * kBilTQW;
  const int u0 = blockIdx.y * kBilTQH;
  const int f = blockIdx.z;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, T::QW * T::QH * 48);
    const int x = q0 - T::LQ, y = u0 - H;
    const char* win = a.cwin + (((long long)f * a.gy + blockIdx.y) * a.gx + blockIdx.x) * a.wstride;
    bulk_load(P.c0, win, T::NQ * 16, &bar);
    bulk_load(P.c1, win + T::NQ * 16, T::NQ * 8, &bar);
    tma_load_3d(P.n0, &tn0, &bar, x * 4, y, f);
    tma_load_3d(P.n1, &tn1, &bar, x * 2, y, f);
  }
  __syncthreads();  // barrier initialised (and its loads issued) before anyone waits
  const float sB = a.sB;
  const int tx = threadIdx.x % kBilTQW, ty = threadIdx.x / kBilTQW;
  const int R0 = kQPT * ty + H, C = tx + T::LQ;
  mbar_wait(&bar, 0);

  Quad2 qa, qb;
  float res[2][6];
  bool upd[2][2];
  bil_weigh<H>(P, R0, C, sB, qa, qb, res, upd);

#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int u = u0 + kQPT * ty + o, v = q0 + tx;
    if (u >= Mq || v >= Nq) continue;
    const Quad2& q = o == 0 ? qa : qb;
    if (SCATTER) {
      // unchanged triangles return this iteration's input normal, held here only as
      // n' = fl(n * sqrt(B)).  A valid triangle no iteration has moved (isolated, or
      // |acc| <= 1e-30 throughout -- the usual case) has n = its FC normal: rebuilt from
      // the points with iteration 1's arithmetic and accepted when it reproduces n'
      // exactly; otherwise n' / sqrt(B) (<= 1 ulp).  Rare path (global point loads).
      const float inv = 1.0f / sB;
      bool rebuild = false;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (!upd[o][k]) {
          const bool valid = (k == 0 ? f2lo(q.cx) : f2hi(q.cx)) != 1e18f;  // not a sentinel
          const float qn = __int_as_float(0x7fc00000);
          res[o][3 * k] = valid ? (k == 0 ? f2lo(q.nx) : f2hi(q.nx)) * inv : qn;
          res[o][3 * k + 1] = valid ? (k == 0 ? f2lo(q.ny) : f2hi(q.ny)) * inv : qn;
          res[o][3 * k + 2] = valid ? (k == 0 ? f2lo(q.nz) : f2hi(q.nz)) * inv : qn;
          rebuild |= valid;
        }
      }
      if (rebuild && a.pts != nullptr) {  // rare: a valid triangle left unchanged (FC-array
                                          // input: no points, n' / sqrt(B) stays)
        const float* P1 = a.pts + f * a.pts_fs + (long long)u * a.pitch + 3 * v;
        float raw[6];
        fc_normals_quad(P1, P1 + 3, P1 + a.pitch + 3, P1 + a.pitch, raw);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const float n0 = k == 0 ? f2lo(q.nx) : f2hi(q.nx);
          const float n1 = k == 0 ? f2lo(q.ny) : f2hi(q.ny);
          const float n2 = k == 0 ? f2lo(q.nz) : f2hi(q.nz);
          const float* rk = raw + 3 * k;
          if (!upd[o][k] && (k == 0 ? f2lo(q.cx) : f2hi(q.cx)) != 1e18f &&
              rk[0] * sB == n0 && rk[1] * sB == n1 && rk[2] * sB == n2) {
            res[o][3 * k] = rk[0];
            res[o][3 * k + 1] = rk[1];
            res[o][3 * k + 2] = rk[2];
          }
        }
      }
      scatter_mesh(a, f, u, v, res[o]);
    } else {
      store_packed_n(out, f, u, v, res[o], upd[o], q, sB);
    }
  }
}

template <int H, int MODE, bool SCATTER, bool PACKOUT = false>
int launch_bil(const CUtensorMap& tp, const CUtensorMap& tn, const CUtensorMap& tc,
               const CUtensorMap& to, const BilArgs& a, int F, cudaStream_t st,
               const PackedG& pg = PackedG{}) {
  constexpr int smem = bil_smem_bytes<H, MODE>();
  static std::atomic<unsigned long long> attr_mask{0};
  if (const int rc = ensure_smem_attr(bilateral_kernel<H, MODE, SCATTER, PACKOUT>, smem, attr_mask))
    return rc;
  const int Mq = a.M - 1, Nq = a.N - 1;
  dim3 grid((Nq + kBilTQW - 1) / kBilTQW, (Mq + kBilTQH - 1) / kBilTQH, F);
  bilateral_kernel<H, MODE, SCATTER, PACKOUT><<<grid, kBilNT, smem, st>>>(tp, tn, tc, to, a, pg);
  return check_launch("bilateral_kernel");
}

template <int H, bool SCATTER>
int launch_packed(const CUtensorMap* maps, const BilArgs& a, int F, const PackedG& out,
                  cudaStream_t st) {
  using T = BilTile<H>;
  constexpr int smem = T::PACK_F * 4 + kSmemSlack;
  static std::atomic<unsigned long long> attr_mask{0};
  if (const int rc = ensure_smem_attr(bilateral_packed_kernel<H, SCATTER>, smem, attr_mask))
    return rc;
  const int Mq = a.M - 1, Nq = a.N - 1;
  dim3 grid((Nq + kBilTQW - 1) / kBilTQW, (Mq + kBilTQH - 1) / kBilTQH, F);
  bilateral_packed_kernel<H, SCATTER><<<grid, kBilNT, smem, st>>>(maps[0], maps[1], maps[2],
                                                                   maps[3], a, out);
  return check_launch("bilateral_packed_kernel");
}

template <int H>
int launch_any(int mode, bool scatter, const CUtensorMap& tp, const CUtensorMap& tn,
               const CUtensorMap& tc, const CUtensorMap& to, const BilArgs& a, int F,
               cudaStream_t st) {
  switch (mode) {
    case kFromPoints:
      return scatter ? launch_bil<H, kFromPoints, true>(tp, tn, tc, to, a, F, st)
                     : launch_bil<H, kFromPoints, false>(tp, tn, tc, to, a, F, st);
    case kNormalsBuf:
      return scatter ? launch_bil<H, kNormalsBuf, true>(tp, tn, tc, to, a, F, st)
                     : launch_bil<H, kNormalsBuf, false>(tp, tn, tc, to, a, F, st);
    default:
      return scatter ? launch_bil<H, kNormalsCentBuf, true>(tp, tn, tc, to, a, F, st)
                     : launch_bil<H, kNormalsCentBuf, false>(tp, tn, tc, to, a, F, st);
  }
}

int launch_h(int h, int mode, bool scatter, const CUtensorMap& tp, const CUtensorMap& tn,
             const CUtensorMap& tc, const CUtensorMap& to, const BilArgs& a, int F,
             cudaStream_t st) {
  switch (h) {
    case 1: return launch_any<1>(mode, scatter, tp, tn, tc, to, a, F, st);
    case 2: return launch_any<2>(mode, scatter, tp, tn, tc, to, a, F, st);
    case 3: return launch_any<3>(mode, scatter, tp, tn, tc, to, a, F, st);
    case 4: return launch_any<4>(mode, scatter, tp, tn, tc, to, a, F, st);
    default: return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  }
}

int launch_packout_h(int h, const CUtensorMap& tp, const BilArgs& a, int F, const PackedG& pg,
                     cudaStream_t st) {
  switch (h) {
    case 1: return launch_bil<1, kFromPoints, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 2: return launch_bil<2, kFromPoints, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 3: return launch_bil<3, kFromPoints, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 4: return launch_bil<4, kFromPoints, false, true>(tp, tp, tp, tp, a, F, st, pg);
    default: return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  }
}

// iteration 1 of the fused pipeline from FC arrays (fp32 normals + f64 centroids: the
// mixed-precision front end)
int launch_packout_arrays_h(int h, const CUtensorMap& tn, const CUtensorMap& tc,
                            const BilArgs& a, int F, const PackedG& pg, cudaStream_t st) {
  switch (h) {
    case 1: return launch_bil<1, kNormalsCentBuf, false, true>(tn, tn, tc, tn, a, F, st, pg);
    case 2: return launch_bil<2, kNormalsCentBuf, false, true>(tn, tn, tc, tn, a, F, st, pg);
    case 3: return launch_bil<3, kNormalsCentBuf, false, true>(tn, tn, tc, tn, a, F, st, pg);
    case 4: return launch_bil<4, kNormalsCentBuf, false, true>(tn, tn, tc, tn, a, F, st, pg);
    default: return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  }
}

// iteration 1 of the fused pipeline from the f64 point grid (the mixed front end, even N)
int launch_packout_pts64_h(int h, const CUtensorMap& tp, const BilArgs& a, int F,
                           const PackedG& pg, cudaStream_t st) {
  switch (h) {
    case 1: return launch_bil<1, kFromPoints64, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 2: return launch_bil<2, kFromPoints64, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 3: return launch_bil<3, kFromPoints64, false, true>(tp, tp, tp, tp, a, F, st, pg);
    case 4: return launch_bil<4, kFromPoints64, false, true>(tp, tp, tp, tp, a, F, st, pg);
    default: return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  }
}

int launch_packed_h(int h, bool scatter, const CUtensorMap* maps, const BilArgs& a, int F,
                    const PackedG& out, cudaStream_t st) {
  switch (h) {
    case 1: return scatter ? launch_packed<1, true>(maps, a, F, out, st)
                           : launch_packed<1, false>(maps, a, F, out, st);
    case 2: return scatter ? launch_packed<2, true>(maps, a, F, out, st)
                           : launch_packed<2, false>(maps, a, F, out, st);
    case 3: return scatter ? launch_packed<3, true>(maps, a, F, out, st)
                           : launch_packed<3, false>(maps, a, F, out, st);
    case 4: return scatter ? launch_packed<4, true>(maps, a, F, out, st)
                           : launch_packed<4, false>(maps, a, F, out, st);
    default: return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  }
}

// OPCFE_BILATERAL_PACKED=0 disables the packed-plane path of the fused pipeline (A/B)
static const bool g_bil_packed = [] {
  const char* v = std::getenv("OPCFE_BILATERAL_PACKED");
  return v == nullptr || v[0] != '0';
}();

// OPCFE_MIXED_FUSED_FC=0 keeps the separate FC-data pass of the mixed front end (A/B)
static const bool g_mixed_fused_fc = [] {
  const char* v = std::getenv("OPCFE_MIXED_FUSED_FC");
  return v == nullptr || v[0] != '0';
}();

int box_q(int h) { return ((((h + 1) / 2 * 2) + kBilTQW + h + 1) / 2) * 2; }
int box_p(int h) { return ((((h + 3) / 4 * 4) + kBilTQW + h + 1 + 3) / 4) * 4; }

}  // namespace

bool bilateral_fc_in_iteration1(int N, int iters) {
  return g_mixed_fused_fc && g_bil_packed && N % 2 == 0 && iters >= 2;
}

// bytes of one tile's packed centroid window (C0 float4 + C1 float2 per box quad), 128-B rounded
size_t centroid_window_bytes(int h) {
  const int QW = box_q(h), QH = kBilTQH + 2 * h;
  return ((size_t)QW * QH * 24 + 127) / 128 * 128;
}
size_t bilateral_buf_c_bytes(int F, int M, int N, int ksize) {
  const size_t tiles = (size_t)((N - 1 + kBilTQW - 1) / kBilTQW) * ((M - 1 + kBilTQH - 1) / kBilTQH);
  return (size_t)F * tiles * centroid_window_bytes(ksize / 2);
}

int bilateral(const float* pts, int F, int M, int N, int pitch, const float* normals_in,
              const double* centroids_in, float sigma_length, float sigma_angle, int ksize,
              int iters, float* buf_a, float* buf_b, float* out_fc, const int64_t* trimap,
              float* out_mesh, long long out_rows, cudaStream_t st, float* buf_c,
              double* out_mesh64, const double* pts64) {
  if (F < 1 || M < 2 || N < 2 || iters < 1 || ksize < 3 || (ksize % 2) == 0)
    return fail(ERR_INVALID, "bilateral: bad shape or parameters");
  if (!(sigma_length > 0.f) || !(sigma_angle > 0.f))
    return fail(ERR_INVALID, "bilateral: sigma scales must be positive");
  const int h = ksize / 2;
  if (h > 4) return fail(ERR_UNSUPPORTED, "bilateral: kernel_size > 9 is not compiled in");
  // input forms: FC arrays (normals + centroids) | point grid | point grid + FC normals
  // to continue from (centroids from the grid: the fused pipeline's iterations 2..B)
  const bool from_arrays = normals_in != nullptr && centroids_in != nullptr;
  const bool resume = normals_in != nullptr && centroids_in == nullptr;
  // pts64: the mixed front end's FC data computed inside the fused iteration 1 from the
  // f64 grid (even N: 16-B rows; >= 2 iterations with the packed-window buffer)
  const bool from_p64 = pts64 != nullptr;
  if (from_p64 && (from_arrays || resume || N % 2 || iters < 2 || buf_c == nullptr ||
                   !g_bil_packed || (out_mesh == nullptr && out_mesh64 == nullptr)))
    return fail(ERR_INVALID, "bilateral: f64-grid input needs even N and the fused pipeline");
  if (!from_arrays && !from_p64 && (pts == nullptr || pitch < 3 * N || pitch % 4))
    return fail(ERR_INVALID, "bilateral: point grid (pitch multiple of 4 floats) required");
  const bool scatter = out_mesh != nullptr || out_mesh64 != nullptr;
  if (scatter && trimap == nullptr) return fail(ERR_INVALID, "bilateral: scatter needs trimap");
  if (!scatter && out_fc == nullptr) return fail(ERR_INVALID, "bilateral: no output given");
  if ((iters > 1 && !buf_a) || (iters > 2 && !buf_b))
    return fail(ERR_INVALID, "bilateral: ping-pong buffers required");

  const int Mq = M - 1, Nq = N - 1;
  const int fcp = fc_pitch(N);
  const uint64_t fc_fs = (uint64_t)Mq * fcp;
  const int QW = box_q(h), QH = kBilTQH + 2 * h;
  const int PW = box_p(h), PH = QH + 1;
  const int SW = kBilTQW, SH = kBilTQH;  // store box
  // kernel parameters need a valid encoding even where a mode ignores the map
  CUtensorMap m_pts, m_nin, m_cin, ld_a, st_a, ld_b, st_b, st_fin;
  int rc;
  auto fc_load = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, QW * 6, QH);
  };
  auto fc_store = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, SW * 6, SH);
  };
  if (from_p64) {
    if ((rc = make_tmap_3d(&m_pts, pts64, true, 3ull * N, M, F, 3ull * N, 3ull * N * M, PW * 3,
                           PH)))
      return rc;
    m_nin = m_cin = m_pts;
  } else if (from_arrays) {
    if ((rc = fc_load(&m_nin, normals_in))) return rc;
    // float64 centroids, contiguous [F][Mq][Nq][2][3] (rows of 6 Nq doubles: 16-B multiples)
    if ((rc = make_tmap_3d(&m_cin, centroids_in, true, 6ull * Nq, Mq, F, 6ull * Nq,
                           6ull * Nq * Mq, QW * 6, QH)))
      return rc;
    m_pts = m_nin;
  } else {
    if ((rc = make_tmap_3d(&m_pts, pts, false, 3ull * N, M, F, pitch, (uint64_t)M * pitch,
                           PW * 3, PH)))
      return rc;
    m_nin = m_cin = m_pts;
    if (resume && (rc = fc_load(&m_nin, normals_in))) return rc;
  }
  if (!scatter) {
    if ((rc = fc_store(&st_fin, out_fc))) return rc;
  } else {
    st_fin = m_pts;
  }
  if (buf_a && ((rc = fc_load(&ld_a, buf_a)) || (rc = fc_store(&st_a, buf_a)))) return rc;
  if (buf_b && ((rc = fc_load(&ld_b, buf_b)) || (rc = fc_store(&st_b, buf_b)))) return rc;

  BilArgs a;
  a.M = M;
  a.N = N;
  a.F = F;
  a.sA = (float)std::sqrt(1.4426950408889634 / (2.0 * (double)sigma_length * sigma_length));
  a.sB = (float)std::sqrt(1.4426950408889634 / (2.0 * (double)sigma_angle * sigma_angle));
  a.trimap = trimap;
  a.tm_fs = 2ll * Mq * Nq;
  a.out_mesh = out_mesh;
  a.out_mesh64 = out_mesh64;
  a.out_fs = 3ll * out_rows;
  a.n_out = out_rows;
  a.pts = pts;
  a.pitch = pitch;
  a.pts_fs = (long long)M * pitch;
  a.gx = (Nq + kBilTQW - 1) / kBilTQW;
  a.gy = (Mq + kBilTQH - 1) / kBilTQH;
  a.wstride = (long long)centroid_window_bytes(h);
  a.cwin = reinterpret_cast<char*>(buf_c);

  // Fused pipeline with >= 2 iterations and a third buffer: iteration 1 writes the packed
  // planes (centroids once into C, normals into A); iterations 2..B read them by TMA with
  // no pack phase (bilateral_packed_kernel), ping-ponging A / B; the last one scatters.
  if (buf_c != nullptr && g_bil_packed && !resume && scatter && iters >= 2) {
    const long long Nq2 = (Nq + 1) & ~1ll;
    auto planes_of = [&](float* b) {
      PackedG g;
      g.n0 = reinterpret_cast<float4*>(b);
      g.n1 = reinterpret_cast<float2*>(b + 4ll * F * Mq * Nq);
      g.s4 = Nq;
      g.s2 = Nq2;
      g.f4 = (long long)Mq * Nq;
      g.f2s = (long long)Mq * Nq2;
      return g;
    };
    const PackedG ga = planes_of(buf_a);  // normals; centroids: per-tile windows in buf_c
    const PackedG gb = buf_b ? planes_of(buf_b) : ga;
    auto maps_of = [&](const PackedG& g, CUtensorMap* m4, CUtensorMap* m2) {
      int r = make_tmap_3d(m4, g.n0, false, 4ull * Nq, Mq, F, 4ull * Nq, 4ull * Mq * Nq,
                           QW * 4, QH, true);
      if (!r) r = make_tmap_3d(m2, g.n1, false, 2ull * Nq, Mq, F, 2ull * Nq2, 2ull * Mq * Nq2,
                               QW * 2, QH, true);
      return r;
    };
    CUtensorMap mna[2], mnb[2];
    if ((rc = maps_of(ga, &mna[0], &mna[1])) || (rc = maps_of(gb, &mnb[0], &mnb[1]))) return rc;
    // iteration 1: centroid windows -> buf_c, normals -> A
    if ((rc = from_p64      ? launch_packout_pts64_h(h, m_pts, a, F, ga, st)
              : from_arrays ? launch_packout_arrays_h(h, m_nin, m_cin, a, F, ga, st)
                            : launch_packout_h(h, m_pts, a, F, ga, st)))
      return rc;
    for (int it = 1; it < iters; ++it) {
      const bool last = it == iters - 1;
      const bool from_a = (it % 2) == 1;
      const CUtensorMap* nin = from_a ? mna : mnb;
      const CUtensorMap maps[4] = {nin[0], nin[1], nin[0], nin[1]};  // [0], [1] unused
      if ((rc = launch_packed_h(h, last, maps, a, F, from_a ? gb : ga, st))) return rc;
    }
    return OK;
  }

  // it0 reads (points | arrays) and writes A; it_k reads A/B and writes B/A; the last
  // iteration scatters to mesh order (trimap) or stores to out_fc.
  const CUtensorMap* src_n = &m_nin;
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    const int mode = from_arrays ? kNormalsCentBuf
                                 : ((it == 0 && !resume) ? kFromPoints : kNormalsBuf);
    const CUtensorMap* dst = last ? &st_fin : ((it % 2 == 0) ? &st_a : &st_b);
    rc = launch_h(h, mode, last && scatter, m_pts, *src_n, m_cin, *dst, a, F, st);
    if (rc) return rc;
    src_n = (it % 2 == 0) ? &ld_a : &ld_b;
  }
  return OK;
}

}  // namespace opcfe
