// Strict (fp64) front-end kernels: the reference's own arithmetic, in its own operation
// order, on the reference's own float64 layouts -- any odd kernel size.
//
//   laplacian_f64   _kernels.laplacian_filter (_native.pyx:225-284; _fallback.py:82-117)
//                   bit-identical to the reference: IEEE dmul / dadd / sqrt / div, no FMA
//                   contraction (the reference is built with -ffp-contract=off,
//                   setup.py:24-26), neighbours in the same du-outer / dv-inner order.
//   bilateral_f64   _kernels.bilateral_iterate (_native.pyx:287-364; _fallback.py:120-166)
//                   + the trimap gather of bilateral_filter_opc (smoothing.py:108-114):
//                   same accumulation order; fp64 throughout, FMA-contracted products and
//                   an own exp (exp_neg, ~2 ulp), so each weight is within a few ulp of
//                   the reference's -- its own two backends differ by ~1 ulp already
//                   (SURVEY.md App. A.5); chained C4 result within 1.5e-14.
//   batched helpers the strict front end needs: FC data, triangle normals and l_max
//   flags over F frames with per-frame live counts.
//
// Layouts (the reference's): grids (F, M, N, 3) f64 contiguous; FC arrays
// (F, M-1, N-1, 2, 3) f64 contiguous.  One thread per output point / quad; a CTA stages
// its tile + halo in shared memory (planar, one plane per component) when it fits,
// otherwise (huge kernels) the neighbours are read through L1 from global memory.
// FP64-pipe bound: ~64 DFMA/clk/SM, IEEE sqrt + div ~2.7 pairs/clk/SM, exp ~2.9/clk/SM
// (dev/probes/fp64_probe.cu on B200).
#include "common.cuh"
#include "opcfe_internal.h"

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace opcfe {

namespace {

constexpr int kSTW = 32;  // tile width (points / quads) = one warp
constexpr int kSTH = 8;   // tile height (rows) = warps per CTA
constexpr int kSNT = kSTW * kSTH;
constexpr int kSmemMax = 200 * 1024;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000LL); }
constexpr double kSentinel = 1e200;
  // centroid of a skipped neighbour: |dc|^2 = inf -> w = 0

// exp(x) for the bilateral weights, x <= 0 (global-memory path: the exponent
// -dc2/(2 sl^2) - dn2/(2 sa^2)).  Cody-Waite reduction x = n ln2 + r, |r| <= ln2/2,
// degree-13 Taylor polynomial (truncation < 2e-16 relative): within ~2 ulp of the correctly
// rounded value (the reference's libm exp is within 1 ulp; its two backends differ by as
// much).  x < -708 returns 0 (a weight < 1e-307 is invisible: the reference's |acc| >
// 1e-30 test leaves a triangle whose weights are all that small unchanged, and next to
// any larger weight it is below the last ulp); NaN passes through (poisons the sum, as in
// the reference).
__constant__ double kExpC[14] = {
    1.0, 1.0, 1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040, 1.0 / 40320,
    1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800, 1.0 / 479001600, 1.0 / 6227020800.0};
__device__ __forceinline__ double exp_neg(double x) {
  if (x < -708.0) return 0.0;
  const double n = rint(x * 1.4426950408889634);
  double r = fma(n, -6.93147180369123816490e-01, x);   // ln2 hi (Cody-Waite split)
  r = fma(n, -1.90821492927058770002e-10, r);          // ln2 lo
  double p = kExpC[13];
#pragma unroll
  for (int k = 12; k >= 0; --k) p = fma(p, r, kExpC[k]);
  return p * __hiloint2double(((int)n + 1023) << 20, 0);
}

__device__ __forceinline__ void exp_table_init(double* T) {  // T[j] = 2^(j/32)
  const int t = threadIdx.y * blockDim.x + threadIdx.x;
  if (t < 32) T[t] = exp2((double)t / 32.0);
}

// 2^(y/32) for y <= 0 (the shared-memory path, whose features are prescaled so that the
// weight is 2^(-t/32), t = |dc'|^2 + |dn'|^2): y = 32 m + j + f with n = rint(y), f = y - n
// EXACT (|f| <= 1/2, no Cody-Waite split), j = n & 31, m = n >> 5; the result is
// T[j] * 2^m * e^(f ln2/32) with T[j] = 2^(j/32) from a 32-entry shared table (2^m folded
// into T[j]'s exponent bits: one integer add) and a degree-6 polynomial in f (truncation
// < 4e-18) by Estrin's scheme (dependency depth 4).  Branch-free: y below -32704 (weight
// < 2^-1022) selects 0; NaN propagates.  ~2 ulp.
__constant__ double kExp2C[7] = {  // (ln2/32)^k / k!
    1.0, 0.02166084939249829, 0.00023459619820224677, 1.6938509724371819e-06,
    9.172562701824643e-09, 3.9737099845494154e-11, 1.4345655584131932e-13};
__device__ __forceinline__ double exp2_32(double y, const double* T) {
  const double n = rint(y);
  const double f = y - n;                                   // exact
  const int ni = (int)n;
  const double f2 = f * f;
  const double a = fma(kExp2C[1], f, kExp2C[0]);
  const double b = fma(kExp2C[3], f, kExp2C[2]);
  const double c = fma(kExp2C[5], f, kExp2C[4]);
  const double ab = fma(b, f2, a);
  const double cd = fma(kExp2C[6], f2, c);
  const double p = fma(cd, f2 * f2, ab);
  const double t = T[ni & 31];
  const double s = __hiloint2double(__double2hiint(t) + ((ni >> 5) << 20), __double2loint(t));
  return y < -32704.0 ? 0.0 : p * s;
}

// ------------------------------------------------------------------ Laplacian
// in/out: [F][M][N][3].  HC > 0: compile-time half width; HC == 0: runtime h.
// SMEM: the tile + halo is staged in three planes of (kSTH+2h) x (kSTW+2h) doubles;
// out-of-grid cells hold NaN (the reference skips them; a NaN distance is skipped too).
template <int HC, bool SMEM>
__global__ void __launch_bounds__(kSNT, 5) laplacian_f64_kernel(const double* __restrict__ in,
                                                             double* __restrict__ out, int M,
                                                             int N, int h_rt, double lam) {
  const int h = HC > 0 ? HC : h_rt;
  const int f = blockIdx.z;
  const long long fs = 3ll * M * N;
  const double* src = in + f * fs;
  double* dst = out + f * fs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int u = blockIdx.y * kSTH + ty, v = blockIdx.x * kSTW + tx;
  extern __shared__ double sm[];
  const int bw = kSTW + 2 * h, bh = kSTH + 2 * h, plane = bw * bh;
  if (SMEM) {  // one box point per thread and step: 3 loads, 3 planar stores
    const int u0 = blockIdx.y * kSTH - h, v0 = blockIdx.x * kSTW - h;
    for (int q = threadIdx.y * kSTW + threadIdx.x; q < plane; q += kSNT) {
      const int r = q / bw, c = q - r * bw;
      const int uu = u0 + r, vv = v0 + c;
      double x = qnan(), y = qnan(), z = qnan();
      if (uu >= 0 && uu < M && vv >= 0 && vv < N) {
        const double* g = src + ((long long)uu * N + vv) * 3;
        x = __ldg(g);
        y = __ldg(g + 1);
        z = __ldg(g + 2);
      }
      sm[q] = x;
      sm[plane + q] = y;
      sm[2 * plane + q] = z;
    }
    __syncthreads();
  }
  if (u >= M || v >= N) return;
  const long long o = ((long long)u * N + v) * 3;
  double px, py, pz;
  if (SMEM) {
    const int c = (ty + h) * bw + tx + h;
    px = sm[c];
    py = sm[plane + c];
    pz = sm[2 * plane + c];
  } else {
    px = src[o];
    py = src[o + 1];
    pz = src[o + 2];
  }
  // outer ring copied for any kernel size (_native.pyx:240-241); NaN centre kept (:245-249)
  if (u == 0 || u == M - 1 || v == 0 || v == N - 1 || px != px || py != py || pz != pz) {
    dst[o] = px;
    dst[o + 1] = py;
    dst[o + 2] = pz;
    return;
  }
  double wsum = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
  for (int du = -h; du <= h; ++du) {
    const int uu = u + du;
    if (!SMEM && (uu < 0 || uu >= M)) continue;
#pragma unroll
    for (int dv = -h; dv <= h; ++dv) {
      if (du == 0 && dv == 0) continue;
      const int vv = v + dv;
      double qx, qy, qz;
      if (SMEM) {
        const int c = (ty + h + du) * bw + tx + h + dv;
        qx = sm[c];
        qy = sm[plane + c];
        qz = sm[2 * plane + c];
      } else {
        if (vv < 0 || vv >= N) continue;
        const double* q = src + ((long long)uu * N + vv) * 3;
        qx = __ldg(q);
        qy = __ldg(q + 1);
        qz = __ldg(q + 2);
      }
      const double dx = dsub(qx, px), dy = dsub(qy, py), dz = dsub(qz, pz);
      const double dist = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
      if (!(dist > 0.0)) continue;  // NaN or <= 0 (:265-266)
      const double w = __drcp_rn(dist);  // correctly rounded 1/dist == the reference's 1.0/dist
      ax = dadd(ax, dmul(dx, w));
      ay = dadd(ay, dmul(dy, w));
      az = dadd(az, dmul(dz, w));
      wsum = dadd(wsum, w);
    }
  }
  if (wsum > 0.0) {
    const double s = __ddiv_rn(lam, wsum);
    px = dadd(px, dmul(s, ax));
    py = dadd(py, dmul(s, ay));
    pz = dadd(pz, dmul(s, az));
  }
  dst[o] = px;
  dst[o + 1] = py;
  dst[o + 2] = pz;
}

// k = 3, even N (16-B row stride of the f64 grid): the same arithmetic as
// laplacian_f64_kernel<1, true>, with the tile + halo arriving by ONE TMA 3-D box load
// (NaN out-of-bounds fill) instead of per-thread global loads, then transposed in shared
// memory into the conflict-free planar layout.  The box starts 2 points left of the tile
// (a 16-B aligned start: 2 x 24 B) and is 36 points wide.
// RPT rows per thread: the tile is 32 x (8 RPT) points, thread (tx, ty) computes rows ty,
// ty + 8, ... (independent chains; the halo and the staging amortised over RPT times the
// points).  The smoothed tile is staged in the (then dead) raw box and leaves by one TMA
// store (the grid edge clipped by the tensor map) instead of 24-B-strided scalar stores.
// MIXED (precision "mixed"): the pair weight 1/dist is rsqrt(|d|^2) (MUFU.RSQ64H + Newton,
// ~1 ulp) instead of an IEEE sqrt and an IEEE division, and the sums are FMA-contracted:
// float64 vertices within a few ulp per pass of the reference's, not bit-exact.
// SRC = float: the first pass of a float32 source reads its fp32 box directly (the
// widening to f64 is exact, so the results are those of an f64 copy of the source) --
// no separate conversion pass; the box then starts 4 points left (16-B rule for 12-B
// points) and the output tile gets its own room.
template <typename SRC>
__host__ __device__ constexpr int lap_box_lpad() { return sizeof(SRC) == 8 ? 2 : 4; }
template <int RPT, typename SRC>
__host__ __device__ constexpr int lap_raw_doubles() {
  constexpr int BXW = kSTW + 2 * lap_box_lpad<SRC>(), BXH = kSTH * RPT + 2;
  constexpr int raw = (BXW * 3 * BXH * (int)sizeof(SRC) + 127) / 128 * 128 / 8;
  constexpr int out = (kSTW * 3 * kSTH * RPT * 8 + 127) / 128 * 128 / 8;
  return raw > out ? raw : out;
}
template <int RPT, bool MIXED, typename SRC = double>
__global__ void __launch_bounds__(kSNT, 5) laplacian_f64_tma_kernel(
    const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int M,
    int N, double lam, uint32_t* __restrict__ vmask) {
  constexpr int TH = kSTH * RPT;
  constexpr int LPAD = lap_box_lpad<SRC>();
  constexpr int BXW = kSTW + 2 * LPAD, BXH = TH + 2;  // TMA box (points)
  constexpr int RAWF = lap_raw_doubles<RPT, SRC>();
  constexpr int BW = kSTW + 2, PL = BW * BXH;
  static_assert(kSTW * 3 * TH <= RAWF, "the output tile reuses the raw box");
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp;
  double* raw = reinterpret_cast<double*>(smem_aligned_base(smem_raw, &barp));
  const SRC* raw_s = reinterpret_cast<const SRC*>(raw);
  double* sm = raw + RAWF;
  uint64_t& bar = *barp;
  const int f = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * kSTW + tx;
  const int u0 = blockIdx.y * TH, v0 = blockIdx.x * kSTW;
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    mbar_expect_tx(&bar, BXW * 3 * BXH * (int)sizeof(SRC));
    tma_load_3d(raw, &tin, &bar, (v0 - LPAD) * 3, u0 - 1, f);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  for (int q = tid; q < PL; q += kSNT) {  // AoS box (r, c + LPAD - 1) -> planes (r, c)
    const int r = q / BW, c = q - r * BW;
    const SRC* p = raw_s + (r * BXW + c + LPAD - 1) * 3;
    sm[q] = (double)p[0];
    sm[PL + q] = (double)p[1];
    sm[2 * PL + q] = (double)p[2];
  }
  __syncthreads();  // raw is dead from here: the output tile [TH][32][3]
  const int v = v0 + tx;
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int ty_k = ty + k * kSTH, u = u0 + ty_k;
    const int c0 = (ty_k + 1) * BW + tx + 1;
    double px = sm[c0], py = sm[PL + c0], pz = sm[2 * PL + c0];
    if (vmask != nullptr) {  // pass 1: the grid's validity bits (iteration-invariant), one
                             // word per warp row segment (off-grid lanes read NaN: 0)
      const unsigned bits = __ballot_sync(0xffffffffu, isfinite(px) && isfinite(py) && isfinite(pz));
      if (tx == 0 && u < M) vmask[((long long)f * M + u) * ((N + 31) / 32) + blockIdx.x] = bits;
    }
    if (u > 0 && u < M - 1 && v > 0 && v < N - 1 && px == px && py == py && pz == pz) {
      double wsum = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
      for (int du = -1; du <= 1; ++du) {
#pragma unroll
        for (int dv = -1; dv <= 1; ++dv) {
          if (du == 0 && dv == 0) continue;
          const int c = c0 + du * BW + dv;
          if constexpr (MIXED) {
            const double dx = sm[c] - px, dy = sm[PL + c] - py, dz = sm[2 * PL + c] - pz;
            const double d2 = fma(dz, dz, fma(dy, dy, dx * dx));
            if (d2 > 0.0) {  // NaN / coincident: skipped (:265-266)
              const double w = rsqrt(d2);
              ax = fma(dx, w, ax);
              ay = fma(dy, w, ay);
              az = fma(dz, w, az);
              wsum += w;
            }
          } else {
            const double dx = dsub(sm[c], px), dy = dsub(sm[PL + c], py),
                         dz = dsub(sm[2 * PL + c], pz);
            const double dist = __dsqrt_rn(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
            if (!(dist > 0.0)) continue;  // NaN or <= 0 (:265-266)
            const double w = __drcp_rn(dist);
            ax = dadd(ax, dmul(dx, w));
            ay = dadd(ay, dmul(dy, w));
            az = dadd(az, dmul(dz, w));
            wsum = dadd(wsum, w);
          }
        }
      }
      if (wsum > 0.0) {
        if constexpr (MIXED) {
          const double s = lam / wsum;
          px = fma(s, ax, px);
          py = fma(s, ay, py);
          pz = fma(s, az, pz);
        } else {
          const double s = __ddiv_rn(lam, wsum);
          px = dadd(px, dmul(s, ax));
          py = dadd(py, dmul(s, ay));
          pz = dadd(pz, dmul(s, az));
        }
      }
    }
    double* o = raw + (ty_k * kSTW + tx) * 3;  // ring / NaN / off-grid cells: the input value
    o[0] = px;
    o[1] = py;
    o[2] = pz;
  }
  fence_proxy_async_smem();
  __syncthreads();
  if (tid == 0) {
    tma_store_3d(&tout, raw, v0 * 3, u0, f);
    tma_store_commit_and_wait();
  }
}

// ------------------------------------------------------------------ bilateral
// centroids, normals: [F][Mq][Nq][2][3].  Output: FC layout (out_fc) or, with trimap,
// mesh order out_mesh[f][trimap[gid]] (OUT = double or float).  Shared planes (SMEM):
// 12 of (kSTH+2h) x (kSTW+2h) doubles: centroid xyz and normal xyz of triangles 0 / 1.
struct Bil64Args {
  const double* cen;
  const double* nin;
  double* nout;          // FC output (nullable when scattering)
  const int64_t* trimap; // [F][G] (scatter)
  void* out_mesh;        // [F][out_rows][3]
  long long out_rows;
  int Mq, Nq, h;
  double inv2sc, inv2ss;
  double sC, sN;          // sqrt(32 log2(e) inv2sc), sqrt(32 log2(e) inv2ss): prescaled path
};

// Global-memory path (windows too large for shared memory): neighbours read through L1,
// the reference's own operation order, exp_neg.
template <typename OUT>
__global__ void __launch_bounds__(kSNT) bilateral_f64_kernel(Bil64Args a) {
  const int h = a.h;
  const int Mq = a.Mq, Nq = a.Nq;
  const int f = blockIdx.z;
  const long long fs = 6ll * Mq * Nq;
  const double* cen = a.cen + f * fs;
  const double* nrm = a.nin + f * fs;
  const int u = blockIdx.y * kSTH + threadIdx.y, v = blockIdx.x * kSTW + threadIdx.x;
  if (u >= Mq || v >= Nq) return;
  const long long qo = ((long long)u * Nq + v) * 6;
  for (int k = 0; k < 2; ++k) {
    const double cx = cen[qo + 3 * k], cy = cen[qo + 3 * k + 1], cz = cen[qo + 3 * k + 2];
    const double nx = nrm[qo + 3 * k], ny = nrm[qo + 3 * k + 1], nz = nrm[qo + 3 * k + 2];
    double rx = nx, ry = ny, rz = nz;  // NaN centre: kept (:313-318)
    if (!(nx != nx || ny != ny || nz != nz)) {
      double wsum = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
      for (int du = -h; du <= h; ++du) {
        const int uu = u + du;
        if (uu < 0 || uu >= Mq) continue;
        for (int dv = -h; dv <= h; ++dv) {
          const int vv = v + dv;
          if (vv < 0 || vv >= Nq) continue;
          for (int kk = 0; kk < 2; ++kk) {
            if (du == 0 && dv == 0 && kk == k) continue;
            const long long o = ((long long)uu * Nq + vv) * 6 + 3 * kk;
            const double mx = __ldg(nrm + o), my = __ldg(nrm + o + 1), mz = __ldg(nrm + o + 2);
            if (mx != mx || my != my || mz != mz) continue;  // (:337-338)
            double dx = dsub(__ldg(cen + o), cx), dy = dsub(__ldg(cen + o + 1), cy),
                   dz = dsub(__ldg(cen + o + 2), cz);
            const double dc2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
            dx = dsub(mx, nx);
            dy = dsub(my, ny);
            dz = dsub(mz, nz);
            const double dn2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
            const double w = exp_neg(dsub(dmul(-dc2, a.inv2sc), dmul(dn2, a.inv2ss)));
            ax = dadd(ax, dmul(mx, w));
            ay = dadd(ay, dmul(my, w));
            az = dadd(az, dmul(mz, w));
            wsum = dadd(wsum, w);
          }
        }
      }
      const double norm = __dsqrt_rn(dadd(dadd(dmul(ax, ax), dmul(ay, ay)), dmul(az, az)));
      if (wsum > 0.0 && norm > 1e-30) {  // (:352-360)
        rx = __ddiv_rn(ax, norm);
        ry = __ddiv_rn(ay, norm);
        rz = __ddiv_rn(az, norm);
      }
    }
    if (a.trimap != nullptr) {
      const long long G = 2ll * Mq * Nq;
      const long long t = a.trimap[f * G + 2ll * ((long long)u * Nq + v) + k];
      if (t >= 0 && t < a.out_rows) {
        OUT* o = static_cast<OUT*>(a.out_mesh) + (f * a.out_rows + t) * 3;
        o[0] = (OUT)rx;
        o[1] = (OUT)ry;
        o[2] = (OUT)rz;
      }
    } else {
      double* o = a.nout + f * fs + qo + 3 * k;
      o[0] = rx;
      o[1] = ry;
      o[2] = rz;
    }
  }
}

// Shared-memory path (any window that fits): the tile + halo is staged once, then every
// box triangle is PRESCALED in place -- c' = (c - o) sC with o a centroid of the tile
// (tile-relative: c - o is exact for nearby values, so the scaling's rounding scales with
// the tile extent, not the distance from the coordinate origin), n' = n sN -- so that the
// weight is 2^(-t/32) with t = |c'_j - c'_i|^2 + |n'_j - n'_i|^2: exp2_32 needs no
// Cody-Waite reduction and the exponent no scaling products.  Neighbours the reference
// skips (NaN normal, off the grid) become sentinels (n' = 0, c' = 1e200: t = inf, w = 0):
// no per-pair test.  wsum is not accumulated: wsum > 0 is implied by |acc| > 1e-30
// (a NaN weight makes both tests false), here |acc'| > 1e-30 sN.  Products are
// FMA-contracted and sums reordered relative to the reference -- results within a few
// ulp (the 1e-13 bar of the strict tests).
// SYM (h == 1): each unordered pair's weight is computed once -- w(i,j) = w(j,i) exactly in
// the reference too (|x_j - x_i|^2 == |x_i - x_j|^2 bit for bit) -- by the thread owning
// the "forward" quad of the pair (offsets (0,+1), (+1,-1), (+1,0), (+1,+1) and the
// intra-quad pair), which accumulates its side at once and hands the weight to the
// receiving thread through shared memory (16 weights per quad); pairs whose forward quad
// lies in the halo are weighed by the receiver itself.  41 % fewer fp64 operations per
// output triangle for 32 KB more shared memory.
// TMA (with SYM): the centroid and normal boxes arrive by two TMA loads (NaN out-of-bounds
// fill == off-grid) into the weight-exchange region (free until after staging), and the
// staging pass transforms them from shared memory instead of global loads.
template <int HC, bool VEC, bool SYM, typename OUT, bool TMA = false>
__global__ void __launch_bounds__(kSNT, SYM ? 3 : 4)
    bilateral_f64s_kernel(Bil64Args a, const __grid_constant__ CUtensorMap tc,
                          const __grid_constant__ CUtensorMap tn) {
  static_assert(!SYM || HC == 1, "the symmetric schedule is written for kernel size 3");
  static_assert(!TMA || SYM, "TMA staging is written for the kernel-size-3 layout");
  const int h = HC > 0 ? HC : a.h;
  const int Mq = a.Mq, Nq = a.Nq;
  const int f = blockIdx.z;
  const long long fs = 6ll * Mq * Nq;
  const double* cen = a.cen + f * fs;
  const double* nrm = a.nin + f * fs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * kSTW + tx;
  const int u = blockIdx.y * kSTH + ty, v = blockIdx.x * kSTW + tx;
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp = nullptr;
  double* const sm = TMA ? reinterpret_cast<double*>(smem_aligned_base(smem_raw, &barp))
                         : reinterpret_cast<double*>(smem_raw);
  __shared__ double expT[32];
  __shared__ double s_o[3];
  __shared__ int s_first;
  exp_table_init(expT);
  const int bw = kSTW + 2 * h, bh = kSTH + 2 * h, plane = bw * bh;
  // plane index: (k * 2 + {0 centroid, 1 normal}) * 3 + comp
  const int u0 = blockIdx.y * kSTH - h, v0 = blockIdx.x * kSTW - h;
  const double sC = a.sC, sN = a.sN;
  // tile origin o: the tile's centre quad's triangle-0 centroid (read by every thread;
  // one L1 line), so staging can prescale on the fly; a non-finite centre (rare: a NaN
  // there) stages raw values first and picks the first finite centroid of the box
  const int cu = min(blockIdx.y * kSTH + kSTH / 2, Mq - 1), cv = min(blockIdx.x * kSTW + kSTW / 2, Nq - 1);
  const double* co = cen + ((long long)cu * Nq + cv) * 6;
  double o[3] = {co[0], co[1], co[2]};
  const bool direct = isfinite(o[0]) && isfinite(o[1]) && isfinite(o[2]);
  // one box quad per thread and step: its 12 doubles (centroids, normals of both
  // triangles; 2 x 48 contiguous bytes, 16-B loads when aligned) -> 12 planar slots.
  // Skipped neighbours (NaN normal, off the grid) become sentinels: n' = 0, c' = 1e200
  // (t = inf -> w = 0): no per-pair test in the loop.
  double* const rawc = sm + 12 * plane;  // TMA boxes [bh][bw * 6] (the W region)
  double* const rawn = rawc + 2048;
  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(barp, 1);
      fence_mbar_init();
      mbar_expect_tx(barp, 2 * bw * 6 * bh * 8);
      tma_load_3d(rawc, &tc, barp, v0 * 6, u0, f);
      tma_load_3d(rawn, &tn, barp, v0 * 6, u0, f);
    }
    __syncthreads();
    mbar_wait(barp, 0);
  }
  for (int q = tid; q < plane; q += kSNT) {
    const int r = q / bw, c = q - r * bw;
    const int uu = u0 + r, vv = v0 + c;
    double cv6[6], nv6[6];
    if constexpr (TMA) {
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const double2 x = reinterpret_cast<const double2*>(rawc + q * 6)[j];
        const double2 y = reinterpret_cast<const double2*>(rawn + q * 6)[j];
        cv6[2 * j] = x.x;
        cv6[2 * j + 1] = x.y;
        nv6[2 * j] = y.x;
        nv6[2 * j + 1] = y.y;
      }
    } else if (uu >= 0 && uu < Mq && vv >= 0 && vv < Nq) {
      const long long off = ((long long)uu * Nq + vv) * 6;
      if (VEC) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double2 x = __ldg(reinterpret_cast<const double2*>(cen + off) + j);
          const double2 y = __ldg(reinterpret_cast<const double2*>(nrm + off) + j);
          cv6[2 * j] = x.x;
          cv6[2 * j + 1] = x.y;
          nv6[2 * j] = y.x;
          nv6[2 * j + 1] = y.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          cv6[j] = __ldg(cen + off + j);
          nv6[j] = __ldg(nrm + off + j);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < 6; ++j) cv6[j] = nv6[j] = qnan();
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      double* cb = sm + (k * 2) * 3 * plane + q;
      double* nb = cb + 3 * plane;
      const double* cc = cv6 + 3 * k;
      const double* nn = nv6 + 3 * k;
      if (!direct) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          cb[d * plane] = cc[d];
          nb[d * plane] = nn[d];
        }
      } else if (isnan(nn[0]) || isnan(nn[1]) || isnan(nn[2])) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          cb[d * plane] = kSentinel;
          nb[d * plane] = 0.0;
        }
      } else {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          cb[d * plane] = (cc[d] - o[d]) * sC;
          nb[d * plane] = nn[d] * sN;
        }
      }
    }
  }
  if (!direct) {  // uniform over the CTA: the rare NaN-centre tile
    if (tid == 0) s_first = 0x7fffffff;
    __syncthreads();
    auto finite_c = [&](int i) {  // box triangle i = k * plane + cell
      const int k = i >= plane, cell = i - k * plane;
      const double* cb = sm + (k * 2) * 3 * plane + cell;
      return isfinite(cb[0]) && isfinite(cb[plane]) && isfinite(cb[2 * plane]);
    };
    for (int i = tid; i < 2 * plane; i += kSNT)
      if (finite_c(i)) {
        atomicMin(&s_first, i);
        break;
      }
    __syncthreads();
    if (tid == 0) {
      const int i = s_first;
      const int k = i >= plane, cell = i - k * plane;
      for (int d = 0; d < 3; ++d)
        s_o[d] = i == 0x7fffffff ? 0.0 : sm[((k * 2) * 3 + d) * plane + cell];
    }
    __syncthreads();
    for (int i = tid; i < 2 * plane; i += kSNT) {
      const int k = i >= plane, cell = i - k * plane;
      double* cb = sm + (k * 2) * 3 * plane + cell;
      double* nb = cb + 3 * plane;
      if (isnan(nb[0]) || isnan(nb[plane]) || isnan(nb[2 * plane])) {
        nb[0] = nb[plane] = nb[2 * plane] = 0.0;
        cb[0] = cb[plane] = cb[2 * plane] = kSentinel;
      } else {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          cb[d * plane] = (cb[d * plane] - s_o[d]) * sC;
          nb[d * plane] *= sN;
        }
      }
    }
  }
  __syncthreads();
  // prescaled weight of the pair (own triangle: centroid ci, normal ni; box cell / kk)
  auto tri = [&](int cell, int kk, double* cc, double* nn) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      cc[d] = sm[((kk * 2) * 3 + d) * plane + cell];
      nn[d] = sm[((kk * 2 + 1) * 3 + d) * plane + cell];
    }
  };
  auto weight = [&](const double* ci, const double* ni, const double* cj, const double* nj) {
    const double ex = cj[0] - ci[0], ey = cj[1] - ci[1], ez = cj[2] - ci[2];
    const double fx = nj[0] - ni[0], fy = nj[1] - ni[1], fz = nj[2] - ni[2];
    double t = ex * ex;
    t = fma(ey, ey, t);
    t = fma(ez, ez, t);
    t = fma(fx, fx, t);
    t = fma(fy, fy, t);
    t = fma(fz, fz, t);
    return exp2_32(-t, expT);
  };
  const int c0 = (ty + h) * bw + tx + h;
  double oc[2][3], on[2][3];
  tri(c0, 0, oc[0], on[0]);
  tri(c0, 1, oc[1], on[1]);
  double acc[2][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
  if constexpr (SYM) {
    double* W = sm + 12 * plane;  // [16][kSNT]: weights for the receiving thread
    constexpr int FD[4][2] = {{0, 1}, {1, -1}, {1, 0}, {1, 1}};
    {  // intra-quad pair
      const double w = weight(oc[0], on[0], oc[1], on[1]);
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        acc[0][d] = fma(on[1][d], w, acc[0][d]);
        acc[1][d] = fma(on[0][d], w, acc[1][d]);
      }
    }
#pragma unroll
    for (int di = 0; di < 4; ++di) {  // forward pairs: weigh, keep own side, hand over
      const int du = FD[di][0], dv = FD[di][1];
      const int rty = ty + du, rtx = tx + dv;
      const bool recv = rty < kSTH && rtx >= 0 && rtx < kSTW;
      const int rtid = rty * kSTW + rtx;
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        double cj[3], nj[3];
        tri(c0 + du * bw + dv, kk, cj, nj);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const double w = weight(oc[k], on[k], cj, nj);
#pragma unroll
          for (int d = 0; d < 3; ++d) acc[k][d] = fma(nj[d], w, acc[k][d]);
          if (recv) W[(di * 4 + k * 2 + kk) * kSNT + rtid] = w;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int di = 0; di < 4; ++di) {  // backward pairs: handed over, or (halo) weighed here
      const int du = FD[di][0], dv = FD[di][1];
      const int sty = ty - du, stx = tx - dv;
      const bool from_w = sty >= 0 && stx >= 0 && stx < kSTW;
#pragma unroll
      for (int ks = 0; ks < 2; ++ks) {
        double cj[3], nj[3];
        tri(c0 - du * bw - dv, ks, cj, nj);
#pragma unroll
        for (int kr = 0; kr < 2; ++kr) {
          const double w = from_w ? W[(di * 4 + ks * 2 + kr) * kSNT + tid]
                                  : weight(oc[kr], on[kr], cj, nj);
#pragma unroll
          for (int d = 0; d < 3; ++d) acc[kr][d] = fma(nj[d], w, acc[kr][d]);
        }
      }
    }
  }
  if (u >= Mq || v >= Nq) return;
  const long long qo = ((long long)u * Nq + v) * 6;
  const double thr = 1e-30 * sN;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double cx = oc[k][0], cy = oc[k][1], cz = oc[k][2];
    const double nx = on[k][0], ny = on[k][1], nz = on[k][2];
    double ax = acc[k][0], ay = acc[k][1], az = acc[k][2];
    bool moved = false;
    if (cx != kSentinel) {
      if constexpr (!SYM) {
#pragma unroll
        for (int du = -h; du <= h; ++du) {
#pragma unroll
          for (int dv = -h; dv <= h; ++dv) {
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              if (du == 0 && dv == 0 && kk == k) continue;
              const int c = (ty + h + du) * bw + tx + h + dv;
              const double mx = sm[((kk * 2 + 1) * 3 + 0) * plane + c];
              const double my = sm[((kk * 2 + 1) * 3 + 1) * plane + c];
              const double mz = sm[((kk * 2 + 1) * 3 + 2) * plane + c];
              const double qx = sm[((kk * 2) * 3 + 0) * plane + c];
              const double qy = sm[((kk * 2) * 3 + 1) * plane + c];
              const double qz = sm[((kk * 2) * 3 + 2) * plane + c];
              const double ex = qx - cx, ey = qy - cy, ez = qz - cz;
              const double fx = mx - nx, fy = my - ny, fz = mz - nz;
              double t = ex * ex;
              t = fma(ey, ey, t);
              t = fma(ez, ez, t);
              t = fma(fx, fx, t);
              t = fma(fy, fy, t);
              t = fma(fz, fz, t);
              const double w = exp2_32(-t, expT);
              ax = fma(mx, w, ax);
              ay = fma(my, w, ay);
              az = fma(mz, w, az);
            }
          }
        }
      }
      const double norm = sqrt(fma(az, az, fma(ay, ay, ax * ax)));
      moved = norm > thr;  // (:352-360); NaN -> unchanged
      if (moved) {
        ax /= norm;
        ay /= norm;
        az /= norm;
      }
    }
    if (!moved) {  // unchanged (NaN / isolated / |acc| <= 1e-30): the input normal exactly
      ax = nrm[qo + 3 * k];
      ay = nrm[qo + 3 * k + 1];
      az = nrm[qo + 3 * k + 2];
    }
    if (a.trimap != nullptr) {
      const long long G = 2ll * Mq * Nq;
      const long long t = a.trimap[f * G + 2ll * ((long long)u * Nq + v) + k];
      if (t >= 0 && t < a.out_rows) {
        OUT* o = static_cast<OUT*>(a.out_mesh) + (f * a.out_rows + t) * 3;
        o[0] = (OUT)ax;
        o[1] = (OUT)ay;
        o[2] = (OUT)az;
      }
    } else {
      double* o = a.nout + f * fs + qo + 3 * k;
      o[0] = ax;
      o[1] = ay;
      o[2] = az;
    }
  }
}

// ------------------------------------------------------------------ batched helpers
// FC data (smoothing.py:61-88) of F frames: [F][M][N][3] -> [F][Mq][Nq][2][3], bit-exact.
__global__ void fc_data_f64_kernel(const double* __restrict__ opc, int M, int N,
                                   double* __restrict__ cen, double* __restrict__ nrm) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int Nq = N - 1;
  const long long Q = (long long)(M - 1) * Nq;
  if (q >= Q) return;
  const int f = blockIdx.y;
  const int u = (int)(q / Nq), v = (int)(q % Nq);
  const double* p1 = opc + (long long)f * M * N * 3 + ((long long)u * N + v) * 3;
  const double* p2 = p1 + 3;
  const double* p4 = p1 + (long long)N * 3;
  const double* p3 = p4 + 3;
  const double* tri[2][3] = {{p3, p2, p1}, {p1, p4, p3}};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double *A = tri[k][0], *B = tri[k][1], *C = tri[k][2];
    double* co = cen + (f * Q + q) * 6 + 3 * k;
    double* no = nrm + (f * Q + q) * 6 + 3 * k;
#pragma unroll
    for (int j = 0; j < 3; ++j) co[j] = centroid_f64(A[j], B[j], C[j]);
    unit_normal_f64(A[0], A[1], A[2], B[0], B[1], B[2], C[0], C[1], C[2], no[0], no[1], no[2]);
  }
}

// FC data for the MIXED front end: the reference's f64 centroids and FC normals (bit-exact,
// as fc_data_f64), the normals rounded to fp32 straight into the padded FC rows the fp32
// bilateral reads (fc_pitch floats per quad row) -- one pass instead of fc_data_f64 +
// staging.  (An fp32 normalisation of the fp64 cross product, ~2 ulp instead of 0.5, put
// one C4 triangle of the chain at 1.5e-5: the normals are rounded from the exact ones.)
__global__ void fc_mixed_kernel(const double* __restrict__ opc, int M, int N,
                                double* __restrict__ cen, float* __restrict__ nrm32, int fcp) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int Nq = N - 1;
  const long long Q = (long long)(M - 1) * Nq;
  if (q >= Q) return;
  const int f = blockIdx.y;
  const int u = (int)(q / Nq), v = (int)(q % Nq);
  const double* p1 = opc + (long long)f * M * N * 3 + ((long long)u * N + v) * 3;
  const double* p2 = p1 + 3;
  const double* p4 = p1 + (long long)N * 3;
  const double* p3 = p4 + 3;
  const double* tri[2][3] = {{p3, p2, p1}, {p1, p4, p3}};
  float* no = nrm32 + ((long long)f * (M - 1) + u) * fcp + 6 * v;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double *A = tri[k][0], *B = tri[k][1], *C = tri[k][2];
    double* co = cen + (f * Q + q) * 6 + 3 * k;
#pragma unroll
    for (int j = 0; j < 3; ++j) co[j] = centroid_f64(A[j], B[j], C[j]);
    double nx, ny, nz;
    unit_normal_f64(A[0], A[1], A[2], B[0], B[1], B[2], C[0], C[1], C[2], nx, ny, nz);
    no[3 * k] = (float)nx;
    no[3 * k + 1] = (float)ny;
    no[3 * k + 2] = (float)nz;
  }
}

// OPCFE_FC_FAST=0 keeps the IEEE-exact FC arithmetic in the mixed FC data (A/B)
static const bool g_fc_fast_host = [] {
  const char* v = std::getenv("OPCFE_FC_FAST");
  return v == nullptr || v[0] != '0';
}();

// FC data, row-segment form (fc_data_f64 / fc_mixed for every shape): a warp owns 32
// consecutive quads of one row.  Each lane loads its two points (u, v), (u + 1, v); the
// right-hand pair comes from the next lane by shuffles (lane 31 loads its own).  The
// arithmetic is fc_data_f64_kernel's (bit-identical); the outputs -- 6 f64 centroids and
// 6 normals per quad, f64 or fp32 (MIXED: padded FC rows) -- are staged in shared memory
// and written as contiguous 16-B / 8-B runs instead of 48-B-strided scalar stores (4x the
// DRAM sectors through L2 in the per-quad kernel).
template <bool MIXED>
__global__ void __launch_bounds__(256) fc_rows_kernel(const double* __restrict__ opc, int M, int N,
                                                     double* __restrict__ cen, void* __restrict__ nrm,
                                                     int fcp, bool fast) {
  __shared__ __align__(16) double s_cen[8][32 * 6];
  __shared__ __align__(16) double s_nrm[8][32 * 6];  // MIXED: floats in the first half
  const int lane = threadIdx.x, w = threadIdx.y;
  const int Nq = N - 1, Mq = M - 1;
  const int u = blockIdx.y * 8 + w;
  const int v0 = blockIdx.x * 32, v = v0 + lane;
  const int f = blockIdx.z;
  if (u >= Mq) return;  // warp-uniform
  const int nseg = min(32, Nq - v0);
  const double* row0 = opc + ((long long)f * M + u) * N * 3;
  const double* row1 = row0 + (long long)N * 3;
  double a[3], b[3];  // (u, v), (u + 1, v)
  if (v < N) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      a[j] = __ldg(row0 + 3ll * v + j);
      b[j] = __ldg(row1 + 3ll * v + j);
    }
  }
  double a2[3], b2[3];  // (u, v + 1), (u + 1, v + 1)
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    a2[j] = __shfl_down_sync(0xffffffffu, a[j], 1);
    b2[j] = __shfl_down_sync(0xffffffffu, b[j], 1);
  }
  if (lane == 31 && v + 1 < N) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      a2[j] = __ldg(row0 + 3ll * (v + 1) + j);
      b2[j] = __ldg(row1 + 3ll * (v + 1) + j);
    }
  }
  if (lane < nseg) {
    // p1 = (u, v), p2 = (u, v + 1), p3 = (u + 1, v + 1), p4 = (u + 1, v): (p3, p2, p1), (p1, p4, p3)
    const double* tri[2][3] = {{b2, a2, a}, {a, b, b2}};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const double *A = tri[k][0], *B = tri[k][1], *C = tri[k][2];
      double nx, ny, nz;
      if (MIXED && fast) {
        // the fp32 bilateral reads these through fp32 (normals) / tile-relative fp32
        // (centroids): a 1-ulp fp64 rsqrt and a product by 1/3 change nothing there but
        // the rare double rounding, at a fraction of the IEEE divisions' cost
#pragma unroll
        for (int j = 0; j < 3; ++j)
          s_cen[w][lane * 6 + 3 * k + j] = mixed_centroid(A[j], B[j], C[j]);
        fast_unit_normal_f64(A, B, C, nx, ny, nz);
      } else {
#pragma unroll
        for (int j = 0; j < 3; ++j) s_cen[w][lane * 6 + 3 * k + j] = centroid_f64(A[j], B[j], C[j]);
        unit_normal_f64(A[0], A[1], A[2], B[0], B[1], B[2], C[0], C[1], C[2], nx, ny, nz);
      }
      if (MIXED) {
        float* sn = reinterpret_cast<float*>(s_nrm[w]) + lane * 6 + 3 * k;
        sn[0] = (float)nx;
        sn[1] = (float)ny;
        sn[2] = (float)nz;
      } else {
        double* sn = s_nrm[w] + lane * 6 + 3 * k;
        sn[0] = nx;
        sn[1] = ny;
        sn[2] = nz;
      }
    }
  }
  __syncwarp();
  const long long qb = (long long)f * Mq * Nq + (long long)u * Nq + v0;  // first quad of the run
  double2* gc = reinterpret_cast<double2*>(cen + qb * 6);
  const double2* sc = reinterpret_cast<const double2*>(s_cen[w]);
  for (int i = lane; i < nseg * 3; i += 32) gc[i] = sc[i];
  if (MIXED) {
    float2* gn = reinterpret_cast<float2*>(static_cast<float*>(nrm) +
                                           ((long long)f * Mq + u) * fcp + 6ll * v0);
    const float2* sn = reinterpret_cast<const float2*>(s_nrm[w]);
    for (int i = lane; i < nseg * 3; i += 32) gn[i] = sn[i];
  } else {
    double2* gn = reinterpret_cast<double2*>(static_cast<double*>(nrm) + qb * 6);
    const double2* sn = reinterpret_cast<const double2*>(s_nrm[w]);
    for (int i = lane; i < nseg * 3; i += 32) gn[i] = sn[i];
  }
}

// mesh normals / l_max flags of F frames: frame f's triangles are rows f*G .. f*G+n_tri[f]
// of `tris` (vertex indices local to the frame), points [F][P][3] f64.
template <typename OUT>
__global__ void tri_extras_f64_kernel(const double* __restrict__ pts, long long P,
                                      const int64_t* __restrict__ tris, long long G,
                                      const int64_t* __restrict__ n_tri, OUT* __restrict__ normals,
                                      double l2_thr, uint8_t* __restrict__ flag) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int f = blockIdx.y;
  if (t >= n_tri[f]) return;
  const long long row = f * G + t;
  const double* base = pts + f * P * 3;
  const double* A = base + tris[3 * row] * 3;
  const double* B = base + tris[3 * row + 1] * 3;
  const double* C = base + tris[3 * row + 2] * 3;
  if (normals != nullptr) {
    double nx, ny, nz;
    unit_normal_f64(A[0], A[1], A[2], B[0], B[1], B[2], C[0], C[1], C[2], nx, ny, nz);
    normals[3 * row] = (OUT)nx;
    normals[3 * row + 1] = (OUT)ny;
    normals[3 * row + 2] = (OUT)nz;
  }
  if (flag != nullptr)
    flag[row] = (uint8_t)longest_edge_exceeds(edge_len2_f64(A[0], A[1], A[2], B[0], B[1], B[2]),
                                              edge_len2_f64(B[0], B[1], B[2], C[0], C[1], C[2]),
                                              edge_len2_f64(C[0], C[1], C[2], A[0], A[1], A[2]),
                                              l2_thr);
}

inline unsigned nblk(long long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

template <typename K>
int set_smem(K kern, int smem) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess)
      return fail(ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  }
  return OK;
}

int lap_smem(int h) { return 3 * (kSTW + 2 * h) * (kSTH + 2 * h) * (int)sizeof(double); }
int bil_smem(int h) { return 12 * (kSTW + 2 * h) * (kSTH + 2 * h) * (int)sizeof(double); }

template <int HC, bool SMEM>
int lap_launch(const double* in, double* out, int F, int M, int N, int h, double lam,
               cudaStream_t st) {
  const int smem = SMEM ? lap_smem(h) : 0;
  int rc;
  if ((rc = set_smem(laplacian_f64_kernel<HC, SMEM>, smem))) return rc;
  dim3 grid((N + kSTW - 1) / kSTW, (M + kSTH - 1) / kSTH, F);
  laplacian_f64_kernel<HC, SMEM><<<grid, dim3(kSTW, kSTH), smem, st>>>(in, out, M, N, h, lam);
  return check_launch("laplacian_f64_kernel");
}

template <int RPT, bool MIXED, typename SRC = double>
int lap_tma_launch_t(const SRC* in, long long in_rs, long long in_fs, double* out, int F, int M,
                     int N, double lam, cudaStream_t st, uint32_t* vmask = nullptr) {
  constexpr int TH = kSTH * RPT, BXH = TH + 2;
  constexpr int RAWF = lap_raw_doubles<RPT, SRC>();
  CUtensorMap mi, mo;
  int rc;
  if ((rc = make_tmap_3d(&mi, in, sizeof(SRC) == 8, 3ull * N, M, F, (uint64_t)in_rs,
                         (uint64_t)in_fs, (kSTW + 2 * lap_box_lpad<SRC>()) * 3, BXH)) ||
      (rc = make_tmap_3d(&mo, out, true, 3ull * N, M, F, 3ull * N, 3ull * N * M, kSTW * 3, TH)))
    return rc;
  constexpr int smem = (RAWF + 3 * (kSTW + 2) * BXH) * (int)sizeof(double) + kSmemSlack;
  static std::atomic<unsigned long long> attr_mask{0};
  auto kern = laplacian_f64_tma_kernel<RPT, MIXED, SRC>;
  if ((rc = ensure_smem_attr(kern, smem, attr_mask))) return rc;
  dim3 grid((N + kSTW - 1) / kSTW, (M + TH - 1) / TH, F);
  kern<<<grid, dim3(kSTW, kSTH), smem, st>>>(mi, mo, M, N, lam, vmask);
  return check_launch("laplacian_f64_tma_kernel");
}

// three rows per thread (32 x 24-point tiles): strict 6.74 ms per 10 C4 passes x 16 frames
// against 6.79 (two rows) and 7.07 (one); mixed 4.49 against 4.56 / 4.85 (four rows, 3
// CTAs / SM: 5.26)
int lap_tma_launch(const double* in, double* out, int F, int M, int N, double lam,
                   cudaStream_t st, uint32_t* vmask) {
  return lap_tma_launch_t<3, false>(in, 3ll * N, 3ll * N * M, out, F, M, N, lam, st, vmask);
}

int lap_mixed_launch(const double* in, double* out, int F, int M, int N, double lam,
                     cudaStream_t st, uint32_t* vmask) {
  return lap_tma_launch_t<3, true>(in, 3ll * N, 3ll * N * M, out, F, M, N, lam, st, vmask);
}

// OPCFE_BIL64_TMA=0 keeps the per-thread staging of the strict k = 3 bilateral (A/B)
static const bool g_bil64_tma = [] {
  const char* v = std::getenv("OPCFE_BIL64_TMA");
  return v == nullptr || v[0] != '0';
}();

template <int HC, bool SMEM, typename OUT>
int bil_launch(const Bil64Args& a, int F, cudaStream_t st) {
  dim3 grid((a.Nq + kSTW - 1) / kSTW, (a.Mq + kSTH - 1) / kSTH, F);
  int rc;
  if constexpr (SMEM) {
    int smem = bil_smem(a.h);
    const bool vec = (reinterpret_cast<uintptr_t>(a.cen) | reinterpret_cast<uintptr_t>(a.nin)) % 16 == 0;
    constexpr bool kSym = HC == 1;
    CUtensorMap tc{}, tn{};
    if constexpr (kSym) {
      if (vec && g_bil64_tma) {  // 48-B quads: the FC rows are 16-B multiples for any Nq
        const int bw = kSTW + 2, bh = kSTH + 2;
        if ((rc = make_tmap_3d(&tc, a.cen, true, 6ull * a.Nq, a.Mq, F, 6ull * a.Nq,
                               6ull * a.Nq * a.Mq, bw * 6, bh)) ||
            (rc = make_tmap_3d(&tn, a.nin, true, 6ull * a.Nq, a.Mq, F, 6ull * a.Nq,
                               6ull * a.Nq * a.Mq, bw * 6, bh)))
          return rc;
        smem += 16 * kSNT * (int)sizeof(double) + kSmemSlack;
        auto kern = bilateral_f64s_kernel<HC, true, true, OUT, true>;
        if ((rc = set_smem(kern, smem))) return rc;
        kern<<<grid, dim3(kSTW, kSTH), smem, st>>>(a, tc, tn);
        return check_launch("bilateral_f64s_kernel");
      }
    }
    auto kern = vec ? bilateral_f64s_kernel<HC, true, kSym, OUT>
                    : bilateral_f64s_kernel<HC, false, kSym, OUT>;
    if (kSym) smem += 16 * kSNT * (int)sizeof(double);
    if ((rc = set_smem(kern, smem))) return rc;
    kern<<<grid, dim3(kSTW, kSTH), smem, st>>>(a, tc, tn);
    return check_launch("bilateral_f64s_kernel");
  } else {
    bilateral_f64_kernel<OUT><<<grid, dim3(kSTW, kSTH), 0, st>>>(a);
    return check_launch("bilateral_f64_kernel");
  }
}

template <typename OUT>
int bil_dispatch(const Bil64Args& a, int F, cudaStream_t st) {
  if (a.h == 1) return bil_launch<1, true, OUT>(a, F, st);
  if (a.h == 2) return bil_launch<2, true, OUT>(a, F, st);
  if (bil_smem(a.h) <= kSmemMax) return bil_launch<0, true, OUT>(a, F, st);
  return bil_launch<0, false, OUT>(a, F, st);
}

}  // namespace

// OPCFE_LAP64_TMA=0 keeps the per-thread staging for every N (A/B)
static const bool g_lap_tma = [] {
  const char* v = std::getenv("OPCFE_LAP64_TMA");
  return v == nullptr || v[0] != '0';
}();

int laplacian_f64(const double* in, double* out, double* tmp, int F, int M, int N, double lam,
                  int ksize, int iters, cudaStream_t st, uint32_t* vmask) {
  if (F < 1 || M < 1 || N < 1 || iters < 1 || ksize < 3 || (ksize % 2) == 0 || !in || !out)
    return fail(ERR_INVALID, "laplacian_f64: bad shape or parameters");
  if (iters > 1 && tmp == nullptr) return fail(ERR_INVALID, "laplacian_f64: tmp buffer required");
  if (in == out || (iters > 1 && in == tmp))
    return fail(ERR_INVALID, "laplacian_f64: input must not alias the output or the ping-pong buffer");
  const int h = ksize / 2;
  // ping-pong so that the last pass lands in `out`
  bool to_out = (iters % 2) == 1;
  const double* src = in;
  for (int it = 0; it < iters; ++it) {
    double* dst = to_out ? out : tmp;
    int rc;
    // k = 3 with a 16-B f64 row stride (N even): TMA-staged; otherwise per-thread loads
    if (h == 1 && N % 2 == 0 && g_lap_tma)
      rc = lap_tma_launch(src, dst, F, M, N, lam, st, it == 0 ? vmask : nullptr);
    else if (h == 1) rc = lap_launch<1, true>(src, dst, F, M, N, h, lam, st);
    else if (h == 2) rc = lap_launch<2, true>(src, dst, F, M, N, h, lam, st);
    else if (lap_smem(h) <= kSmemMax) rc = lap_launch<0, true>(src, dst, F, M, N, h, lam, st);
    else rc = lap_launch<0, false>(src, dst, F, M, N, h, lam, st);
    if (rc) return rc;
    src = dst;
    to_out = !to_out;
  }
  return OK;
}

// OPCFE_LAP64_FROM32=0 keeps the separate fp32 -> f64 conversion pass (A/B)
static const bool g_lap_from32 = [] {
  const char* v = std::getenv("OPCFE_LAP64_FROM32");
  return v == nullptr || v[0] != '0';
}();

bool laplacian64_mask_fused(int N, int ksize) { return g_lap_tma && ksize == 3 && N % 2 == 0; }

bool laplacian64_from32_ok(const float* in, int N, long long rs, int ksize) {
  return g_lap_from32 && g_lap_tma && ksize == 3 && N % 2 == 0 && (rs * 4) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(in) % 16 == 0;
}

int laplacian64_from32(const float* in, long long rs, long long fs, double* out, double* tmp,
                       int F, int M, int N, double lam, int ksize, int iters, bool mixed,
                       cudaStream_t st, uint32_t* vmask) {
  if (!laplacian64_from32_ok(in, N, rs, ksize) || F < 1 || M < 1 || iters < 1 || !in || !out ||
      (iters > 1 && !tmp))
    return fail(ERR_INVALID, "laplacian64_from32: unsupported shape or arguments");
  // pass 1 straight from the fp32 source; passes 2..L on the f64 grid (ping-pong as
  // laplacian_f64: the last pass lands in `out`)
  double* dst = (iters % 2) == 1 ? out : tmp;
  int rc = mixed ? lap_tma_launch_t<3, true, float>(in, rs, fs, dst, F, M, N, lam, st, vmask)
                 : lap_tma_launch_t<3, false, float>(in, rs, fs, dst, F, M, N, lam, st, vmask);
  const long long g_rs = 3ll * N, g_fs = 3ll * N * M;
  for (int it = 1; it < iters && rc == OK; ++it) {
    const double* src = dst;
    dst = dst == out ? tmp : out;
    rc = mixed ? lap_tma_launch_t<3, true>(src, g_rs, g_fs, dst, F, M, N, lam, st)
               : lap_tma_launch_t<3, false>(src, g_rs, g_fs, dst, F, M, N, lam, st);
  }
  return rc;
}

int laplacian_mixed(const double* in, double* out, double* tmp, int F, int M, int N, double lam,
                    int ksize, int iters, cudaStream_t st, uint32_t* vmask) {
  // the fp32-pair kernel covers k = 3 with a 16-B f64 row stride; otherwise the strict
  // kernels (exact, so within every bound the mixed mode promises)
  if (!(ksize == 3 && N % 2 == 0 && g_lap_tma))
    return laplacian_f64(in, out, tmp, F, M, N, lam, ksize, iters, st, vmask);
  if (F < 1 || M < 1 || N < 1 || iters < 1 || !in || !out)
    return fail(ERR_INVALID, "laplacian_mixed: bad shape or parameters");
  if (iters > 1 && tmp == nullptr) return fail(ERR_INVALID, "laplacian_mixed: tmp buffer required");
  if (in == out || (iters > 1 && in == tmp))
    return fail(ERR_INVALID, "laplacian_mixed: input must not alias the output or the ping-pong buffer");
  bool to_out = (iters % 2) == 1;
  const double* src = in;
  for (int it = 0; it < iters; ++it) {
    double* dst = to_out ? out : tmp;
    int rc;
    if ((rc = lap_mixed_launch(src, dst, F, M, N, lam, st, it == 0 ? vmask : nullptr))) return rc;
    src = dst;
    to_out = !to_out;
  }
  return OK;
}

int bilateral_f64(const double* centroids, const double* normals_in, int F, int Mq, int Nq,
                  double sigma_length, double sigma_angle, int ksize, int iters, double* buf_a,
                  double* buf_b, double* out_fc, const int64_t* trimap, void* out_mesh,
                  bool out_f32, long long out_rows, cudaStream_t st) {
  if (F < 1 || Mq < 1 || Nq < 1 || iters < 1 || ksize < 3 || (ksize % 2) == 0 || !centroids ||
      !normals_in)
    return fail(ERR_INVALID, "bilateral_f64: bad shape or parameters");
  if (!(sigma_length > 0.0) || !(sigma_angle > 0.0))
    return fail(ERR_INVALID, "bilateral_f64: sigma scales must be positive");
  const bool scatter = out_mesh != nullptr;
  if (scatter && trimap == nullptr) return fail(ERR_INVALID, "bilateral_f64: scatter needs trimap");
  if (!scatter && out_fc == nullptr) return fail(ERR_INVALID, "bilateral_f64: no output given");
  if ((iters > 1 && !buf_a) || (iters > 2 && !buf_b))
    return fail(ERR_INVALID, "bilateral_f64: ping-pong buffers required");
  Bil64Args a;
  a.cen = centroids;
  a.Mq = Mq;
  a.Nq = Nq;
  a.h = ksize / 2;
  // the reference's constants, same operation order (_native.pyx:295-296)
  a.inv2sc = 1.0 / (2.0 * sigma_length * sigma_length);
  a.inv2ss = 1.0 / (2.0 * sigma_angle * sigma_angle);
  a.sC = std::sqrt(32.0 * 1.4426950408889634 * a.inv2sc);
  a.sN = std::sqrt(32.0 * 1.4426950408889634 * a.inv2ss);
  a.out_rows = out_rows;
  const double* src = normals_in;
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    a.nin = src;
    a.nout = last ? out_fc : ((it % 2 == 0) ? buf_a : buf_b);
    a.trimap = (last && scatter) ? trimap : nullptr;
    a.out_mesh = (last && scatter) ? out_mesh : nullptr;
    const int rc = (last && scatter && out_f32) ? bil_dispatch<float>(a, F, st)
                                                : bil_dispatch<double>(a, F, st);
    if (rc) return rc;
    src = a.nout;
  }
  return OK;
}

// OPCFE_FC_ROWS=0 keeps the per-quad FC-data kernels (A/B)
static const bool g_fc_rows = [] {
  const char* v = std::getenv("OPCFE_FC_ROWS");
  return v == nullptr || v[0] != '0';
}();

int fc_data_f64(const double* opc, int F, int M, int N, double* cen, double* nrm,
                cudaStream_t st) {
  if (F < 1 || M < 2 || N < 2) return fail(ERR_INVALID, "organized cloud must be at least 2 x 2");
  if (g_fc_rows && reinterpret_cast<uintptr_t>(cen) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(nrm) % 16 == 0) {
    dim3 grid((N - 1 + 31) / 32, (M - 1 + 7) / 8, F);
    fc_rows_kernel<false><<<grid, dim3(32, 8), 0, st>>>(opc, M, N, cen, nrm, 0, false);
    return check_launch("fc_rows_kernel");
  }
  const long long Q = (long long)(M - 1) * (N - 1);
  fc_data_f64_kernel<<<dim3(nblk(Q, 256), F), 256, 0, st>>>(opc, M, N, cen, nrm);
  return check_launch("fc_data_f64_kernel");
}

int fc_mixed(const double* opc, int F, int M, int N, double* cen, float* nrm32, int fcp,
             cudaStream_t st) {
  if (F < 1 || M < 2 || N < 2) return fail(ERR_INVALID, "organized cloud must be at least 2 x 2");
  if (g_fc_rows && reinterpret_cast<uintptr_t>(cen) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(nrm32) % 16 == 0 && fcp % 4 == 0) {
    dim3 grid((N - 1 + 31) / 32, (M - 1 + 7) / 8, F);
    fc_rows_kernel<true><<<grid, dim3(32, 8), 0, st>>>(opc, M, N, cen, nrm32, fcp,
                                                          g_fc_fast_host);
    return check_launch("fc_rows_kernel");
  }
  const long long Q = (long long)(M - 1) * (N - 1);
  fc_mixed_kernel<<<dim3(nblk(Q, 256), F), 256, 0, st>>>(opc, M, N, cen, nrm32, fcp);
  return check_launch("fc_mixed_kernel");
}

int tri_extras_f64(const double* pts, int F, int M, int N, const int64_t* tris,
                   const int64_t* n_tri, void* normals, bool normals_f32, double l_max,
                   uint8_t* flag, cudaStream_t st) {
  if (!normals && !flag) return OK;
  const long long G = 2ll * (M - 1) * (N - 1);
  const long long P = (long long)M * N;
  const double thr = sq_threshold(l_max);
  dim3 grid(nblk(G, 256), F);
  if (normals_f32)
    tri_extras_f64_kernel<float><<<grid, 256, 0, st>>>(pts, P, tris, G, n_tri,
                                                       static_cast<float*>(normals), thr, flag);
  else
    tri_extras_f64_kernel<double><<<grid, 256, 0, st>>>(pts, P, tris, G, n_tri,
                                                        static_cast<double*>(normals), thr, flag);
  return check_launch("tri_extras_f64_kernel");
}

}  // namespace opcfe
