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
// B200 mapping (issue-bound kernel: ~14 FP32 ops + 1 MUFU per directed pair, 34 pairs
// per quad at k=3, against 60 B of HBM traffic per quad):
//   * one CTA = 32 x 16 quads, 256 threads, each thread 2 vertically adjacent quads
//     (both triangles of each), so a neighbour record loaded from shared memory feeds
//     up to 4 output triangles;
//   * tile + halo arrive by TMA 3-D box loads with NaN out-of-bounds fill (== the
//     reference's "off-grid neighbours are skipped"): the point tile (centroids are
//     recomputed from points every iteration: 12 B/point instead of 24 B/quad of
//     stored centroids) and, after iteration 1, the previous normal tile;
//   * a pack step turns each halo quad into 3 float4 planes (conflict-free LDS.128):
//     per triangle n' = n*sqrt(B), c' = c*sqrt(A) with B, A the exponent scales
//     pre-multiplied by log2(e), so  w = ex2(-(|c'_i - c'_j|^2 + |n'_i - n'_j|^2)).
//     Missing / NaN-normal triangles carry n' = 0, c' = 1e18, so their weight to any
//     valid triangle underflows to exactly 0: no per-pair NaN test;
//   * iteration 1 computes FC normals with fp64 edges + cross product (no cancellation
//     on slivers) and an fp32 normalisation;
//   * the |acc| > 1e-30 test is evaluated underflow-safely as |acc/wsum| * wsum
//     (SURVEY.md 8c); accumulation order per triangle is the reference's (du, dv, kk).
#include "common.cuh"
#include "opcfe_internal.h"

#include <cmath>
#include <algorithm>
#include <cstdlib>

namespace opcfe {

namespace {

// kernel_size 3 runs the direct kernel by default; OPCFE_BILATERAL_SYM=1 selects the
// pair-symmetric persistent kernel below (half the weights, but 121 registers -> 2 CTAs
// per SM; measured 3.24 vs 2.77 ms per 8 x 1080p x 5 iterations on B200, kept for A/B).
static const bool g_bil_direct = std::getenv("OPCFE_BILATERAL_SYM") == nullptr;
// OPCFE_BILATERAL_WS=1 selects the warp-specialised persistent kernel (A/B: measured
// 2.85 vs 2.43 ms for the direct kernel at 4 CTAs/SM, 8 x 1080p x 5 iterations)
static const bool g_bil_ws = std::getenv("OPCFE_BILATERAL_WS") != nullptr;

constexpr int kBilTQW = 32;  // interior quads per tile row (= one warp)
constexpr int kBilTQH = 16;  // interior quad rows per tile (2 per thread)
constexpr int kBilNT = 256;
// resident CTAs per SM the register budget targets: k = 3 fits 4 x 55 KB of smem (64
// registers), larger windows are smem-limited to 3 (80 registers)
constexpr int bil_min_blocks(int h) { return h == 1 ? 4 : 3; }

enum BilMode : int {
  kFromPoints = 0,     // iteration 1: normals + centroids from the point grid
  kNormalsBuf = 1,     // normals from the previous iteration, centroids from points
  kNormalsCentBuf = 2  // normals and centroids from FC arrays (drop-in bilateral_iterate)
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
  static constexpr int PTS_F = ((PW * 3 * PH) + 31) / 32 * 32;
  static constexpr int FC_F = ((QW * 6 * QH) + 31) / 32 * 32;
  static constexpr int PACK_F = 12 * NQ;  // 3 float4 planes (pack_quad)
  static constexpr int OUT_F = kBilTQW * 6 * kBilTQH;
  static_assert(QW * 6 <= 256 && PW * 3 <= 256 && PH <= 256, "TMA box extent must be <= 256");
  static_assert((QW * 6) % 4 == 0, "FC box rows must be 16-B multiples");
  static_assert(FC_F >= OUT_F, "out tile aliases the FC normal tile");
};

// out tile: its own region in mode 0; aliases the (dead after packing) FC tile otherwise
template <int H, int MODE>
constexpr int bil_smem_bytes() {
  using T = BilTile<H>;
  return (((MODE != kNormalsCentBuf) ? T::PTS_F : 0) + ((MODE != kFromPoints) ? T::FC_F : 0) +
          ((MODE == kNormalsCentBuf) ? T::FC_F : 0) + T::PACK_F +
          ((MODE == kFromPoints) ? T::OUT_F : 0)) *
             4 +
         kSmemSlack;
}

struct BilArgs {
  int M, N;          // point grid (Mq = M-1, Nq = N-1 quads)
  int F;             // frames (persistent kernels walk tiles of all frames)
  float sA, sB;      // sqrt(log2(e)/(2 sl^2)), sqrt(log2(e)/(2 sa^2))
  const int64_t* trimap;  // scatter mode: per frame [G]
  long long tm_fs;
  float* out_mesh;   // scatter destination: per frame [cap][3]
  long long out_fs;  // floats per frame
  long long n_out;   // rows per frame available in out_mesh (bounds check)
  const float* raw_n;  // this launch's input FC normals (modes 1, 2): "unchanged" outputs
  int raw_pitch;       // floats per FC quad row
  long long raw_fs;    // floats per frame
};

// FC normal for the bilateral input: edges and cross product in fp64 (exact edge
// differences of fp32 vertices; no cancellation on slivers), normalisation in fp32.
// |n - float32(reference)| ~ 1e-7, far inside the 1e-5 contract, at a fraction of the
// cost of the correctly rounded fp64 divide/sqrt used where bit-exact normals are
// returned (gridops.cu).
__device__ __forceinline__ void unit_normal_fast(const float* pa, const float* pb, const float* pc,
                                                 float* n) {
  const double e1x = (double)pb[0] - pa[0], e1y = (double)pb[1] - pa[1], e1z = (double)pb[2] - pa[2];
  const double e2x = (double)pc[0] - pa[0], e2y = (double)pc[1] - pa[1], e2z = (double)pc[2] - pa[2];
  const double x = e1y * e2z - e1z * e2y;
  const double y = e1z * e2x - e1x * e2z;
  const double z = e1x * e2y - e1y * e2x;
  const double s = x * x + y * y + z * z;
  if (s > 0.0 && s < 1e300) {
    const float fx = (float)x, fy = (float)y, fz = (float)z;
    // rescale into fp32 range before squaring (tiny triangles: |x| ~ 1e-20)
    const float sc = fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz)));
    const float is = 1.0f / sc;
    const float gx = fx * is, gy = fy * is, gz = fz * is;
    const float r = 1.0f / sqrtf(gx * gx + gy * gy + gz * gz);
    n[0] = gx * r;
    n[1] = gy * r;
    n[2] = gz * r;
  } else {
    n[0] = n[1] = n[2] = __int_as_float(0x7fc00000);
  }
}

struct Tri {
  float nx, ny, nz, cx, cy, cz;
};

// log2 of the weight between two packed triangles: -(|dc'|^2 + |dn'|^2).  Both terms
// from differences: the dot form |n_i|^2 + |n_j|^2 - 2 n_i.n_j cancels catastrophically
// for near-parallel normals (measured 4.6e-5 after 5 iterations at 1080p, > 1e-5).
__device__ __forceinline__ float neg_log2w(const Tri& i, const Tri& j) {
  const float dx = j.cx - i.cx, dy = j.cy - i.cy, dz = j.cz - i.cz;
  const float ex = j.nx - i.nx, ey = j.ny - i.ny, ez = j.nz - i.nz;
  float e = -(dx * dx);
  e = fmaf(-dy, dy, e);
  e = fmaf(-dz, dz, e);
  e = fmaf(-ex, ex, e);
  e = fmaf(-ey, ey, e);
  return fmaf(-ez, ez, e);
}

// pack one quad (both triangles) into 3 float4 planes (conflict-free LDS.128):
//   P0 = (n0'xyz, c0'x)  P1 = (c0'yz, n1'xy)  P2 = (n1'z, c1'xyz)
// n' = n*sqrt(B), c' = c*sqrt(A); a triangle with a NaN normal or centroid is encoded as
// n' = 0, c' = 1e18 (its weight to / from any valid triangle underflows to exactly 0).
__device__ __forceinline__ void pack_quad(float4* pk, int nq, int q, const float* n,
                                          const float* cc, float sA, float sB) {
  float v[12];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const bool ok = !(isnan(n[3 * k]) || isnan(n[3 * k + 1]) || isnan(n[3 * k + 2]) ||
                      isnan(cc[3 * k]) || isnan(cc[3 * k + 1]) || isnan(cc[3 * k + 2]));
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      v[6 * k + j] = ok ? n[3 * k + j] * sB : 0.f;
      v[6 * k + 3 + j] = ok ? cc[3 * k + j] * sA : 1e18f;
    }
  }
  pk[q] = make_float4(v[0], v[1], v[2], v[3]);
  pk[nq + q] = make_float4(v[4], v[5], v[6], v[7]);
  pk[2 * nq + q] = make_float4(v[8], v[9], v[10], v[11]);
}

__device__ __forceinline__ void load_quad(const float4* pk, int nq, int q, Tri* t) {
  const float4 a0 = pk[q], a1 = pk[nq + q], a2 = pk[2 * nq + q];
  t[0] = Tri{a0.x, a0.y, a0.z, a0.w, a1.x, a1.y};
  t[1] = Tri{a1.z, a1.w, a2.x, a2.y, a2.z, a2.w};
}

template <int H, int MODE, bool SCATTER>
__global__ void __launch_bounds__(kBilNT, bil_min_blocks(H))
    bilateral_kernel(const __grid_constant__ CUtensorMap tpts, const __grid_constant__ CUtensorMap tnrm,
                     const __grid_constant__ CUtensorMap tcen, const __grid_constant__ CUtensorMap tout,
                     BilArgs a) {
  using T = BilTile<H>;
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp;
  float* p = reinterpret_cast<float*>(smem_aligned_base(smem_raw, &barp));
  float* pts_s = nullptr;
  float* nrm_s = nullptr;
  float* cen_s = nullptr;
  if (MODE != kNormalsCentBuf) { pts_s = p; p += T::PTS_F; }
  if (MODE != kFromPoints) { nrm_s = p; p += T::FC_F; }
  if (MODE == kNormalsCentBuf) { cen_s = p; p += T::FC_F; }
  float4* pk = reinterpret_cast<float4*>(p);  // 3 planes, see pack_quad
  p += T::PACK_F;
  float* out_s = (MODE == kFromPoints) ? p : nrm_s;
  uint64_t& bar = *barp;

  const int Mq = a.M - 1, Nq = a.N - 1;
  const int q0 = blockIdx.x * kBilTQW;   // first interior quad column
  const int u0 = blockIdx.y * kBilTQH;   // first interior quad row
  const int f = blockIdx.z;

  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t bytes = 0;
    if (MODE != kNormalsCentBuf) bytes += T::PW * 3 * T::PH * 4;
    if (MODE != kFromPoints) bytes += T::QW * 6 * T::QH * 4;
    if (MODE == kNormalsCentBuf) bytes += T::QW * 6 * T::QH * 4;
    mbar_expect_tx(&bar, bytes);
    if (MODE != kNormalsCentBuf) tma_load_3d(pts_s, &tpts, &bar, (q0 - T::LP) * 3, u0 - H, f);
    if (MODE != kFromPoints) tma_load_3d(nrm_s, &tnrm, &bar, (q0 - T::LQ) * 6, u0 - H, f);
    if (MODE == kNormalsCentBuf) tma_load_3d(cen_s, &tcen, &bar, (q0 - T::LQ) * 6, u0 - H, f);
  }
  mbar_wait(&bar, 0);

  const float sA = a.sA, sB = a.sB;
  // ---- pack every halo quad into the 4 planes (scaled + sentinel-encoded)
  for (int q = threadIdx.x; q < T::NQ; q += kBilNT) {
    const int r = q / T::QW, c = q % T::QW;
    float n[6], cc[6];
    if (MODE == kNormalsCentBuf) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        n[j] = nrm_s[q * 6 + j];
        cc[j] = cen_s[q * 6 + j];
      }
    } else {
      const float* P1 = pts_s + (r * T::PW + c + T::PSHIFT) * 3;
      const float* P2 = P1 + 3;
      const float* P4 = P1 + T::PW * 3;
      const float* P3 = P4 + 3;
      const float* tri[2][3] = {{P3, P2, P1}, {P1, P4, P3}};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float *pa = tri[k][0], *pb = tri[k][1], *pc = tri[k][2];
#pragma unroll
        for (int j = 0; j < 3; ++j) cc[3 * k + j] = ((pa[j] + pb[j]) + pc[j]) * (1.0f / 3.0f);
        if (MODE == kFromPoints) unit_normal_fast(pa, pb, pc, n + 3 * k);
      }
      if (MODE == kNormalsBuf) {
#pragma unroll
        for (int j = 0; j < 6; ++j) n[j] = nrm_s[q * 6 + j];
      }
      if (MODE == kFromPoints) {  // raw normals of interior quads: the "unchanged" output
        const int ir = r - H, ic = c - T::LQ;
        if (ir >= 0 && ir < kBilTQH && ic >= 0 && ic < kBilTQW) {
#pragma unroll
          for (int j = 0; j < 6; ++j) out_s[(ir * kBilTQW + ic) * 6 + j] = n[j];
        }
      }
    }
    pack_quad(pk, T::NQ, q, n, cc, sA, sB);
  }
  __syncthreads();

  // ---- two vertically adjacent interior quads per thread
  const int tx = threadIdx.x % kBilTQW, ty = threadIdx.x / kBilTQW;  // ty in [0, 8)
  const int R0 = 2 * ty + H, C = tx + T::LQ;                         // pack pos of quad 0
  float raw[2][6];  // unchanged-output fallback (the caller's normals)
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const float* src = (MODE == kFromPoints) ? out_s + ((2 * ty + o) * kBilTQW + tx) * 6
                                             : nrm_s + ((R0 + o) * T::QW + C) * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) raw[o][j] = src[j];
  }
  Tri own[2][2];
#pragma unroll
  for (int o = 0; o < 2; ++o) load_quad(pk, T::NQ, (R0 + o) * T::QW + C, own[o]);
  float acc[2][2][4];  // [own quad][triangle][x, y, z, wsum]
#pragma unroll
  for (int o = 0; o < 2; ++o)
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[o][k][j] = 0.f;

#pragma unroll
  for (int dr = -H; dr <= H + 1; ++dr) {
#pragma unroll
    for (int dc = -H; dc <= H; ++dc) {
      Tri nb[2];
      load_quad(pk, T::NQ, (R0 + dr) * T::QW + C + dc, nb);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int du = dr - o;
        if (du < -H || du > H) continue;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            if (du == 0 && dc == 0 && kk == k) continue;
            const float w = ex2_approx(neg_log2w(own[o][k], nb[kk]));
            acc[o][k][0] = fmaf(nb[kk].nx, w, acc[o][k][0]);
            acc[o][k][1] = fmaf(nb[kk].ny, w, acc[o][k][1]);
            acc[o][k][2] = fmaf(nb[kk].nz, w, acc[o][k][2]);
          }
        }
      }
    }
  }

  // underflow-safe normalisation: n = m/|m|, m = acc'/wsum; |acc| > 1e-30 <=> |m| wsum > 1e-30 sB
  const float thr = 1e-30f * sB;
  float res[2][6];
#pragma unroll
  for (int o = 0; o < 2; ++o) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float* r = &res[o][3 * k];
      const float* n = &raw[o][3 * k];
      r[0] = n[0];
      r[1] = n[1];
      r[2] = n[2];
      const bool valid = !(isnan(n[0]) || isnan(n[1]) || isnan(n[2]));
      // wsum is not accumulated: wsum == 0 implies acc == 0, so the reference's
      // `wsum > 0 and |acc| > 1e-30` (_native.pyx:352-360) is just |acc| > 1e-30, here
      // |acc'| > 1e-30 sqrt(B) evaluated underflow-safely as s * |acc'/s|, s = max |acc'_i|
      const float ax = acc[o][k][0], ay = acc[o][k][1], az = acc[o][k][2];
      const float s = fmaxf(fabsf(ax), fmaxf(fabsf(ay), fabsf(az)));
      if (valid && s > 0.f) {
        const float is = rcp_approx(s);  // a common scale: cancels in the normalisation
        const float mx = ax * is, my = ay * is, mz = az * is;
        // IEEE sqrt + reciprocal (~1.5 ulp): the stored normals feed the next iteration's
        // weights, so rounding here compounds over the iterations
        const float len = sqrtf(mx * mx + my * my + mz * mz);
        if (len * s > thr) {
          const float il = 1.0f / len;
          r[0] = mx * il;
          r[1] = my * il;
          r[2] = mz * il;
        }
      }
    }
  }

  if (SCATTER) {
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      const int u = u0 + 2 * ty + o, v = q0 + tx;
      if (u < Mq && v < Nq) {
        const long long g = 2ll * ((long long)u * Nq + v);
        const longlong2 tm = *reinterpret_cast<const longlong2*>(a.trimap + f * a.tm_fs + g);
        float* dst = a.out_mesh + f * a.out_fs;
        if (tm.x >= 0 && tm.x < a.n_out) {
          dst[3 * tm.x] = res[o][0];
          dst[3 * tm.x + 1] = res[o][1];
          dst[3 * tm.x + 2] = res[o][2];
        }
        if (tm.y >= 0 && tm.y < a.n_out) {
          dst[3 * tm.y] = res[o][3];
          dst[3 * tm.y + 1] = res[o][4];
          dst[3 * tm.y + 2] = res[o][5];
        }
      }
    }
  } else {
    if (MODE != kFromPoints) __syncthreads();  // out tile aliases the FC tile read above
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      float* dst = out_s + ((2 * ty + o) * kBilTQW + tx) * 6;
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
}

template <int H, int MODE, bool SCATTER>
int launch_bil(const CUtensorMap& tp, const CUtensorMap& tn, const CUtensorMap& tc,
               const CUtensorMap& to, const BilArgs& a, int F, cudaStream_t st) {
  constexpr int smem = bil_smem_bytes<H, MODE>();
  static unsigned long long attr_mask = 0;
  ensure_smem_attr(bilateral_kernel<H, MODE, SCATTER>, smem, attr_mask);
  const int Mq = a.M - 1, Nq = a.N - 1;
  dim3 grid((Nq + kBilTQW - 1) / kBilTQW, (Mq + kBilTQH - 1) / kBilTQH, F);
  bilateral_kernel<H, MODE, SCATTER><<<grid, kBilNT, smem, st>>>(tp, tn, tc, to, a);
  return check_launch("bilateral_kernel");
}

// ============================================================================
// Warp-specialised persistent kernel (default).  The direct kernel above loses ~30 % of
// its issue slots to CTA-phase bubbles: TMA wait at CTA start, the pack phase's last
// partial round in front of a __syncthreads, the store at the end (ncu: 74 % issue-
// active).  Here each persistent CTA has
//   * 4 PRODUCER warps: wait for the TMA tile, pack it (pre-scaled, sentinel-encoded,
//     3 float4 planes) into one of TWO pack buffers, release it through an mbarrier
//     ("full"), and immediately TMA-load the next tile into the (now dead) input tiles;
//   * 8 CONSUMER warps: wait "full", weigh and accumulate 2 quads per thread, release the
//     pack ("empty"), and TMA-store / scatter the results,
// so packing and loading tile i+1 overlap the compute of tile i.  The input tiles are
// dead once packed, so consumers never see them: an output left unchanged (missing /
// isolated / |acc| <= 1e-30) re-reads its input normal from global memory (modes 1, 2)
// or is n'/sqrt(B) (<= 1 ulp of the FC normal; NaN where c' carries the sentinel).
// ============================================================================
constexpr int kWsCons = kBilNT;          // consumer threads (8 warps)
constexpr int kWsProd = 128;             // producer threads (4 warps)
constexpr int kWsThreads = kWsCons + kWsProd;

template <int H, int MODE>
constexpr int ws_smem_bytes() {
  using T = BilTile<H>;
  return (((MODE != kNormalsCentBuf) ? T::PTS_F : 0) + ((MODE != kFromPoints) ? T::FC_F : 0) +
          ((MODE == kNormalsCentBuf) ? T::FC_F : 0) + 2 * T::PACK_F + T::OUT_F) *
             4 +
         64 + kSmemSlack;
}

template <int H, int MODE, bool SCATTER>
__global__ void __launch_bounds__(kWsThreads, 2)
    bilateral_ws_kernel(const __grid_constant__ CUtensorMap tpts,
                        const __grid_constant__ CUtensorMap tnrm,
                        const __grid_constant__ CUtensorMap tcen,
                        const __grid_constant__ CUtensorMap tout, BilArgs a) {
  using T = BilTile<H>;
  constexpr int NQ = T::NQ;
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* tma_bar;
  float* p = reinterpret_cast<float*>(smem_aligned_base(smem_raw, &tma_bar));
  float* pts_s = nullptr;
  float* nrm_s = nullptr;
  float* cen_s = nullptr;
  if (MODE != kNormalsCentBuf) { pts_s = p; p += T::PTS_F; }
  if (MODE != kFromPoints) { nrm_s = p; p += T::FC_F; }
  if (MODE == kNormalsCentBuf) { cen_s = p; p += T::FC_F; }
  float4* const packs = reinterpret_cast<float4*>(p);  // 2 buffers x 3 planes x NQ
  p += 2 * T::PACK_F;
  float* out_s = p;
  p += T::OUT_F;
  uint64_t* full = reinterpret_cast<uint64_t*>(p);  // [2]
  uint64_t* empty = full + 2;                       // [2]

  const int Mq = a.M - 1, Nq = a.N - 1;
  const int tiles_x = (Nq + kBilTQW - 1) / kBilTQW, tiles_y = (Mq + kBilTQH - 1) / kBilTQH;
  const int n_tiles = tiles_x * tiles_y * a.F;
  auto tile_origin = [&](int tile, int& q0, int& u0, int& f) {
    q0 = (tile % tiles_x) * kBilTQW;
    u0 = ((tile / tiles_x) % tiles_y) * kBilTQH;
    f = tile / (tiles_x * tiles_y);
  };
  auto issue = [&](int tile) {
    int q0, u0, f;
    tile_origin(tile, q0, u0, f);
    uint32_t bytes = 0;
    if (MODE != kNormalsCentBuf) bytes += T::PW * 3 * T::PH * 4;
    if (MODE != kFromPoints) bytes += T::QW * 6 * T::QH * 4;
    if (MODE == kNormalsCentBuf) bytes += T::QW * 6 * T::QH * 4;
    mbar_expect_tx(tma_bar, bytes);
    if (MODE != kNormalsCentBuf) tma_load_3d(pts_s, &tpts, tma_bar, (q0 - T::LP) * 3, u0 - H, f);
    if (MODE != kFromPoints) tma_load_3d(nrm_s, &tnrm, tma_bar, (q0 - T::LQ) * 6, u0 - H, f);
    if (MODE == kNormalsCentBuf) tma_load_3d(cen_s, &tcen, tma_bar, (q0 - T::LQ) * 6, u0 - H, f);
  };
  if (threadIdx.x == 0) {
    mbar_init(tma_bar, 1);
    mbar_init(&full[0], kWsProd);
    mbar_init(&full[1], kWsProd);
    mbar_init(&empty[0], kWsCons);
    mbar_init(&empty[1], kWsCons);
    fence_mbar_init();
  }
  __syncthreads();
  const float sA = a.sA, sB = a.sB;

  if (threadIdx.x >= kWsCons) {
    // ------------------------------------------------------------ producer warps
    const int pt = threadIdx.x - kWsCons;
    if (pt == 0 && (int)blockIdx.x < n_tiles) issue(blockIdx.x);
    int it = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
      const int s = it & 1;
      float4* pk = packs + s * 3 * NQ;
      mbar_wait(tma_bar, it & 1);                              // input tile landed
      if (it >= 2) mbar_wait(&empty[s], ((it >> 1) - 1) & 1);  // pack s released
      for (int q = pt; q < NQ; q += kWsProd) {
        const int r = q / T::QW, c = q % T::QW;
        float n[6], cc[6];
        if (MODE == kNormalsCentBuf) {
#pragma unroll
          for (int j = 0; j < 6; ++j) {
            n[j] = nrm_s[q * 6 + j];
            cc[j] = cen_s[q * 6 + j];
          }
        } else {
          const float* P1 = pts_s + (r * T::PW + c + T::PSHIFT) * 3;
          const float* P2 = P1 + 3;
          const float* P4 = P1 + T::PW * 3;
          const float* P3 = P4 + 3;
          const float* tri[2][3] = {{P3, P2, P1}, {P1, P4, P3}};
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const float *pa = tri[k][0], *pb = tri[k][1], *pc = tri[k][2];
#pragma unroll
            for (int j = 0; j < 3; ++j) cc[3 * k + j] = ((pa[j] + pb[j]) + pc[j]) * (1.0f / 3.0f);
            if (MODE == kFromPoints) unit_normal_fast(pa, pb, pc, n + 3 * k);
          }
          if (MODE == kNormalsBuf) {
#pragma unroll
            for (int j = 0; j < 6; ++j) n[j] = nrm_s[q * 6 + j];
          }
        }
        pack_quad(pk, NQ, q, n, cc, sA, sB);
      }
      named_bar_sync(2, kWsProd);  // every producer is done reading the input tiles
      if (pt == 0 && tile + (int)gridDim.x < n_tiles) issue(tile + gridDim.x);
      mbar_arrive(&full[s]);
    }
    return;
  }

  // -------------------------------------------------------------- consumer warps
  const int tx = threadIdx.x % kBilTQW, ty = threadIdx.x / kBilTQW;  // ty in [0, 8)
  const int R0 = 2 * ty + H, C = tx + T::LQ;                         // pack pos of quad 0
  const float inv_sB = 1.0f / sB;
  const float thr = 1e-30f * sB;
  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int s = it & 1;
    const float4* pk = packs + s * 3 * NQ;
    int q0, u0, f;
    tile_origin(tile, q0, u0, f);
    mbar_wait(&full[s], (it >> 1) & 1);
    auto load2 = [&](int q, Tri* t) { load_quad(pk, NQ, q, t); };
    Tri own[2][2];
    load2(R0 * T::QW + C, own[0]);
    load2((R0 + 1) * T::QW + C, own[1]);
    float acc[2][2][3];
#pragma unroll
    for (int o = 0; o < 2; ++o)
#pragma unroll
      for (int k = 0; k < 2; ++k) acc[o][k][0] = acc[o][k][1] = acc[o][k][2] = 0.f;
#pragma unroll
    for (int dr = -H; dr <= H + 1; ++dr) {
#pragma unroll
      for (int dc = -H; dc <= H; ++dc) {
        Tri nb[2];
        load2((R0 + dr) * T::QW + C + dc, nb);
#pragma unroll
        for (int o = 0; o < 2; ++o) {
          const int du = dr - o;
          if (du < -H || du > H) continue;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              if (du == 0 && dc == 0 && kk == k) continue;
              const float w = ex2_approx(neg_log2w(own[o][k], nb[kk]));
              acc[o][k][0] = fmaf(nb[kk].nx, w, acc[o][k][0]);
              acc[o][k][1] = fmaf(nb[kk].ny, w, acc[o][k][1]);
              acc[o][k][2] = fmaf(nb[kk].nz, w, acc[o][k][2]);
            }
          }
        }
      }
    }
    mbar_arrive(&empty[s]);  // pack s may be refilled (all reads above are done)

    float res[2][6];
#pragma unroll
    for (int o = 0; o < 2; ++o) {
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        float* r = &res[o][3 * k];
        const Tri& t = own[o][k];
        const bool valid = t.cx != 1e18f;
        // |acc| > 1e-30 (wsum > 0 implied), underflow-safe: s * |acc/s|, s = max |acc_i|
        const float ax = acc[o][k][0], ay = acc[o][k][1], az = acc[o][k][2];
        const float sc = fmaxf(fabsf(ax), fmaxf(fabsf(ay), fabsf(az)));
        bool upd = false;
        if (valid && sc > 0.f) {
          const float is = rcp_approx(sc);
          const float mx = ax * is, my = ay * is, mz = az * is;
          const float len = sqrtf(mx * mx + my * my + mz * mz);
          if (len * sc > thr) {
            const float il = 1.0f / len;
            r[0] = mx * il;
            r[1] = my * il;
            r[2] = mz * il;
            upd = true;
          }
        }
        if (!upd) {  // unchanged (rare): the input normal as given
          if (MODE == kFromPoints) {
            // n'/sqrt(B) (<= 1 ulp of the FC normal); invalid <=> NaN normal in this mode
            r[0] = valid ? t.nx * inv_sB : __int_as_float(0x7fc00000);
            r[1] = valid ? t.ny * inv_sB : __int_as_float(0x7fc00000);
            r[2] = valid ? t.nz * inv_sB : __int_as_float(0x7fc00000);
          } else {
            const int u = u0 + 2 * ty + o, v = q0 + tx;
            r[0] = r[1] = r[2] = __int_as_float(0x7fc00000);
            if (u < Mq && v < Nq) {
              const float* g = a.raw_n + f * a.raw_fs + (long long)u * a.raw_pitch + 6 * v + 3 * k;
              r[0] = g[0];
              r[1] = g[1];
              r[2] = g[2];
            }
          }
        }
      }
    }
    if (SCATTER) {
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int u = u0 + 2 * ty + o, v = q0 + tx;
        if (u < Mq && v < Nq) {
          const long long g = 2ll * ((long long)u * Nq + v);
          const longlong2 tm = *reinterpret_cast<const longlong2*>(a.trimap + f * a.tm_fs + g);
          float* dst = a.out_mesh + f * a.out_fs;
          if (tm.x >= 0 && tm.x < a.n_out) {
            dst[3 * tm.x] = res[o][0];
            dst[3 * tm.x + 1] = res[o][1];
            dst[3 * tm.x + 2] = res[o][2];
          }
          if (tm.y >= 0 && tm.y < a.n_out) {
            dst[3 * tm.y] = res[o][3];
            dst[3 * tm.y + 1] = res[o][4];
            dst[3 * tm.y + 2] = res[o][5];
          }
        }
      }
    } else {
      if (threadIdx.x == 0) tma_store_wait_read();  // previous out tile has left smem
      named_bar_sync(1, kWsCons);
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        float* dst = out_s + ((2 * ty + o) * kBilTQW + tx) * 6;
#pragma unroll
        for (int j = 0; j < 6; ++j) dst[j] = res[o][j];
      }
      fence_proxy_async_smem();
      named_bar_sync(1, kWsCons);
      if (threadIdx.x == 0) {
        tma_store_3d(&tout, out_s, q0 * 6, u0, f);
        tma_store_commit();
      }
    }
  }
  if (threadIdx.x == 0) tma_store_wait_read();
}

template <int H, int MODE, bool SCATTER>
int launch_ws(const CUtensorMap& tp, const CUtensorMap& tn, const CUtensorMap& tc,
              const CUtensorMap& to, const BilArgs& a, int F, cudaStream_t st) {
  constexpr int smem = ws_smem_bytes<H, MODE>();
  static unsigned long long attr_mask = 0;
  ensure_smem_attr(bilateral_ws_kernel<H, MODE, SCATTER>, smem, attr_mask);
  static int resident = 0, sms = 0;
  if (resident == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, bilateral_ws_kernel<H, MODE, SCATTER>,
                                                  kWsThreads, smem);
    if (resident < 1) resident = 1;
  }
  const int Mq = a.M - 1, Nq = a.N - 1;
  const long long tiles = (long long)((Nq + kBilTQW - 1) / kBilTQW) *
                          ((Mq + kBilTQH - 1) / kBilTQH) * F;
  const int grid = (int)std::min<long long>(tiles, (long long)sms * resident);  // persistent
  bilateral_ws_kernel<H, MODE, SCATTER><<<grid, kWsThreads, smem, st>>>(tp, tn, tc, to, a);
  return check_launch("bilateral_ws_kernel");
}

template <int H>
int launch_any(int mode, bool scatter, const CUtensorMap& tp, const CUtensorMap& tn,
               const CUtensorMap& tc, const CUtensorMap& to, const BilArgs& a, int F,
               cudaStream_t st) {
  if (g_bil_ws) {
    switch (mode) {
      case kFromPoints:
        return scatter ? launch_ws<H, kFromPoints, true>(tp, tn, tc, to, a, F, st)
                       : launch_ws<H, kFromPoints, false>(tp, tn, tc, to, a, F, st);
      case kNormalsBuf:
        return scatter ? launch_ws<H, kNormalsBuf, true>(tp, tn, tc, to, a, F, st)
                       : launch_ws<H, kNormalsBuf, false>(tp, tn, tc, to, a, F, st);
      default:
        return scatter ? launch_ws<H, kNormalsCentBuf, true>(tp, tn, tc, to, a, F, st)
                       : launch_ws<H, kNormalsCentBuf, false>(tp, tn, tc, to, a, F, st);
    }
  }
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

int box_q(int h) { return ((((h + 1) / 2 * 2) + kBilTQW + h + 1) / 2) * 2; }
int box_p(int h) { return ((((h + 3) / 4 * 4) + kBilTQW + h + 1 + 3) / 4) * 4; }

// ============================================================================
// kernel_size 3: pair-symmetric kernel.  w(i,j) = w(j,i), so every unordered
// triangle pair is weighed ONCE and shared between its two triangles:
//   * a warp = 32 consecutive quad columns (lanes 0 and 31 are halo columns that
//     compute but do not output: 30 outputs / warp), 2 quad rows per warp, 8 warps
//     stacked vertically: tile = 30 x 16 quads;
//   * each lane weighs, for its 2 quads: the 2 intra-quad pairs, the vertical pair
//     between its quads, the 4 quad pairs with the right column (16 weights, handed to
//     lane+1 with one shuffle each) and the 3 quad pairs with the row below (12 weights,
//     handed to the warp below through shared memory); the top warp weighs its row
//     above itself.  17 weights per quad instead of 34;
//   * accumulation of a triangle's 17 neighbours happens as weights arrive, so the
//     summation order differs from the reference's (du, dv, kk) by a few ulp.
// ============================================================================
constexpr int kSymW = 32;                 // lanes = columns incl. 2 halo columns
constexpr int kSymOut = kSymW - 2;        // output columns per tile
constexpr int kSymRows = 16;              // output rows per tile
constexpr int kSymQW = kSymW + 2;         // pack / FC box columns: q0-2 .. q0+31
constexpr int kSymQH = kSymRows + 2;      // pack / FC box rows: u0-1 .. u0+16
constexpr int kSymNQ = kSymQW * kSymQH;
constexpr int kSymPW = 40;                // point box columns (>= 35 + alignment shift 2)
constexpr int kSymPH = kSymQH + 1;
constexpr int kSymPtsF = ((kSymPW * 3 * kSymPH) + 31) / 32 * 32;
constexpr int kSymFcF = ((kSymQW * 6 * kSymQH) + 31) / 32 * 32;
constexpr int kSymPackF = 16 * kSymNQ;
constexpr int kSymOutF = kSymOut * 6 * kSymRows;
constexpr int kSymXchF = 8 * 32 * 12;     // down-side weights handed to the next warp
static_assert(kSymFcF >= kSymOutF, "out tile aliases the FC tile");

template <int MODE>
constexpr int sym_smem_bytes() {  // 2 input stages + pack + [own out tile] + exchange + 2 bars
  return (2 * (((MODE != kNormalsCentBuf) ? kSymPtsF : 0) + ((MODE != kFromPoints) ? kSymFcF : 0) +
               ((MODE == kNormalsCentBuf) ? kSymFcF : 0)) +
          kSymPackF + ((MODE == kFromPoints) ? kSymOutF : 0) + kSymXchF) *
             4 +
         16 + kSmemSlack;
}

struct Tri6 {
  float nx, ny, nz, cx, cy, cz;
};

__device__ __forceinline__ float sym_w(const Tri6& i, const Tri6& j) {
  const float dx = j.cx - i.cx, dy = j.cy - i.cy, dz = j.cz - i.cz;
  const float ex = j.nx - i.nx, ey = j.ny - i.ny, ez = j.nz - i.nz;
  float e = -(dx * dx);
  e = fmaf(-dy, dy, e);
  e = fmaf(-dz, dz, e);
  e = fmaf(-ex, ex, e);
  e = fmaf(-ey, ey, e);
  return ex2_approx(fmaf(-ez, ez, e));
}

struct Acc {
  float x = 0.f, y = 0.f, z = 0.f, w = 0.f;
  __device__ __forceinline__ void add(float nx, float ny, float nz, float wt) {
    x = fmaf(nx, wt, x);
    y = fmaf(ny, wt, y);
    z = fmaf(nz, wt, z);
    w += wt;
  }
};

template <int MODE, bool SCATTER>
__global__ void __launch_bounds__(256, 2)
    bilateral_sym_kernel(const __grid_constant__ CUtensorMap tpts,
                         const __grid_constant__ CUtensorMap tnrm,
                         const __grid_constant__ CUtensorMap tcen,
                         const __grid_constant__ CUtensorMap tout, BilArgs a) {
  extern __shared__ __align__(16) char smem_raw[];
  uint64_t* barp;
  float* p = reinterpret_cast<float*>(smem_aligned_base(smem_raw, &barp));
  // two input stages (double buffering), one pack, one exchange area
  float* pts_st[2] = {nullptr, nullptr};
  float* nrm_st[2] = {nullptr, nullptr};
  float* cen_st[2] = {nullptr, nullptr};
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    if (MODE != kNormalsCentBuf) { pts_st[s] = p; p += kSymPtsF; }
    if (MODE != kFromPoints) { nrm_st[s] = p; p += kSymFcF; }
    if (MODE == kNormalsCentBuf) { cen_st[s] = p; p += kSymFcF; }
  }
  float4* pk = reinterpret_cast<float4*>(p);  // planes: [0] n0' [1] c0' [2] n1' [3] c1'
  p += kSymPackF;
  float* out_own = nullptr;
  if (MODE == kFromPoints) { out_own = p; p += kSymOutF; }
  float4* xch = reinterpret_cast<float4*>(p);  // [warp][lane][3] float4
  p += kSymXchF;
  uint64_t* bars = reinterpret_cast<uint64_t*>(p);  // 2 stage barriers

  const int Mq = a.M - 1, Nq = a.N - 1;
  const int tiles_x = (Nq + kSymOut - 1) / kSymOut, tiles_y = (Mq + kSymRows - 1) / kSymRows;
  const int n_tiles = tiles_x * tiles_y * a.F;
  auto issue = [&](int tile, int s) {  // TMA loads of `tile` into stage s (thread 0)
    const int tx = tile % tiles_x, rest = tile / tiles_x;
    const int tq0 = tx * kSymOut, tu0 = (rest % tiles_y) * kSymRows, tf = rest / tiles_y;
    const int tsh = (tq0 - 2) & 3;
    uint32_t bytes = 0;
    if (MODE != kNormalsCentBuf) bytes += kSymPW * 3 * kSymPH * 4;
    if (MODE != kFromPoints) bytes += kSymQW * 6 * kSymQH * 4;
    if (MODE == kNormalsCentBuf) bytes += kSymQW * 6 * kSymQH * 4;
    mbar_expect_tx(&bars[s], bytes);
    if (MODE != kNormalsCentBuf)
      tma_load_3d(pts_st[s], &tpts, &bars[s], (tq0 - 2 - tsh) * 3, tu0 - 1, tf);
    if (MODE != kFromPoints) tma_load_3d(nrm_st[s], &tnrm, &bars[s], (tq0 - 2) * 6, tu0 - 1, tf);
    if (MODE == kNormalsCentBuf)
      tma_load_3d(cen_st[s], &tcen, &bars[s], (tq0 - 2) * 6, tu0 - 1, tf);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
    if ((int)blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  }
  __syncthreads();

  // persistent loop: tile i of this CTA computes while tile i+1's inputs stream in
  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
  const int s = it & 1;
  if (threadIdx.x == 0) {
    tma_store_wait_read();  // the previous tile's out tile (aliases stage s^1 / out_own)
    if (tile + (int)gridDim.x < n_tiles) issue(tile + gridDim.x, s ^ 1);
  }
  __syncthreads();
  const int q0 = (tile % tiles_x) * kSymOut;   // first output quad column (even)
  const int u0 = ((tile / tiles_x) % tiles_y) * kSymRows;
  const int f = tile / (tiles_x * tiles_y);
  const int pshift = (q0 - 2) & 3;             // point box starts on a 16-B boundary
  const float* pts_s = pts_st[s];
  float* nrm_s = nrm_st[s];
  const float* cen_s = cen_st[s];
  float* out_s = (MODE == kFromPoints) ? out_own : nrm_s;
  mbar_wait(&bars[s], (it >> 1) & 1);

  const float sA = a.sA, sB = a.sB;
  for (int q = threadIdx.x; q < kSymNQ; q += 256) {
    const int r = q / kSymQW, c = q % kSymQW;
    float n[6], cc[6];
    if (MODE == kNormalsCentBuf) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        n[j] = nrm_s[q * 6 + j];
        cc[j] = cen_s[q * 6 + j];
      }
    } else {
      const float* P1 = pts_s + (r * kSymPW + c + pshift) * 3;
      const float* P2 = P1 + 3;
      const float* P4 = P1 + kSymPW * 3;
      const float* P3 = P4 + 3;
      const float* tri[2][3] = {{P3, P2, P1}, {P1, P4, P3}};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float *pa = tri[k][0], *pb = tri[k][1], *pc = tri[k][2];
#pragma unroll
        for (int j = 0; j < 3; ++j) cc[3 * k + j] = ((pa[j] + pb[j]) + pc[j]) * (1.0f / 3.0f);
        if (MODE == kFromPoints) unit_normal_fast(pa, pb, pc, n + 3 * k);
      }
      if (MODE == kNormalsBuf) {
#pragma unroll
        for (int j = 0; j < 6; ++j) n[j] = nrm_s[q * 6 + j];
      }
      if (MODE == kFromPoints) {
        const int ir = r - 1, ic = c - 2;
        if (ir >= 0 && ir < kSymRows && ic >= 0 && ic < kSymOut) {
#pragma unroll
          for (int j = 0; j < 6; ++j) out_s[(ir * kSymOut + ic) * 6 + j] = n[j];
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const bool ok = !(isnan(n[3 * k]) || isnan(n[3 * k + 1]) || isnan(n[3 * k + 2]) ||
                        isnan(cc[3 * k]) || isnan(cc[3 * k + 1]) || isnan(cc[3 * k + 2]));
      pk[(2 * k) * kSymNQ + q] = ok ? make_float4(n[3 * k] * sB, n[3 * k + 1] * sB,
                                                  n[3 * k + 2] * sB, 0.f)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      pk[(2 * k + 1) * kSymNQ + q] = ok ? make_float4(cc[3 * k] * sA, cc[3 * k + 1] * sA,
                                                      cc[3 * k + 2] * sA, 0.f)
                                        : make_float4(1e18f, 1e18f, 1e18f, 0.f);
    }
  }
  __syncthreads();

  const int lane = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int R0 = 2 * ty + 1, C = lane + 1;   // pack position of this lane's first quad
  auto tri6 = [&](int q, int k) {
    const float4 n4 = pk[(2 * k) * kSymNQ + q], c4 = pk[(2 * k + 1) * kSymNQ + q];
    return Tri6{n4.x, n4.y, n4.z, c4.x, c4.y, c4.z};
  };
  auto nrm3 = [&](int q, int k) { return pk[(2 * k) * kSymNQ + q]; };

  float raw[2][6];
  const bool out_lane = lane >= 1 && lane <= kSymOut;
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const int ir = 2 * ty + o, ic = lane - 1;
    const float* src = (MODE == kFromPoints)
                           ? out_s + (ir * kSymOut + (out_lane ? ic : 0)) * 6
                           : nrm_s + ((R0 + o) * kSymQW + C) * 6;
#pragma unroll
    for (int j = 0; j < 6; ++j) raw[o][j] = src[j];
  }

  const int q0p = R0 * kSymQW + C, q1p = q0p + kSymQW;  // own quads
  Tri6 own[2][2] = {{tri6(q0p, 0), tri6(q0p, 1)}, {tri6(q1p, 0), tri6(q1p, 1)}};
  Acc acc[2][2];
  // intra-quad pairs
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    const float w = sym_w(own[o][0], own[o][1]);
    acc[o][0].add(own[o][1].nx, own[o][1].ny, own[o][1].nz, w);
    acc[o][1].add(own[o][0].nx, own[o][0].ny, own[o][0].nz, w);
  }
  // vertical pair between the lane's two quads
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const float w = sym_w(own[0][k], own[1][kk]);
      acc[0][k].add(own[1][kk].nx, own[1][kk].ny, own[1][kk].nz, w);
      acc[1][kk].add(own[0][k].nx, own[0][k].ny, own[0][k].nz, w);
    }
  // right column: weigh, keep own share, hand the weights to lane+1 (its left column)
#pragma unroll
  for (int ob = 0; ob < 2; ++ob) {
    const int rq = (R0 + ob) * kSymQW + C + 1;   // right quad in row R0+ob
    const int lq = rq - 2;                        // left quad, same row
    const Tri6 rt[2] = {tri6(rq, 0), tri6(rq, 1)};
    const float4 ln[2] = {nrm3(lq, 0), nrm3(lq, 1)};
#pragma unroll
    for (int oa = 0; oa < 2; ++oa) {
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          // pair (own quad oa tri k) - (right quad in row ob tri kk)
          const float w = sym_w(own[oa][k], rt[kk]);
          acc[oa][k].add(rt[kk].nx, rt[kk].ny, rt[kk].nz, w);
          // the same pair seen from lane+1: (its left quad in row oa, tri k) - (its
          // own quad ob, tri kk); receive lane-1's weight for (left oa,k) - (own ob,kk)
          const float wl = __shfl_up_sync(0xffffffffu, w, 1);
          // here: left quad in row R0+oa; its normal is needed -> from the pack
          const float4 lno = nrm3((R0 + oa) * kSymQW + C - 1, k);
          acc[ob][kk].add(lno.x, lno.y, lno.z, wl);
        }
    }
    (void)ln;
  }
  // row below: weigh (own quad 1) - (quads below at columns C-1, C, C+1)
  float4* xout = xch + (ty * 32 + lane) * 3;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int dq = (R0 + 2) * kSymQW + C - 1 + d;
    const Tri6 dt[2] = {tri6(dq, 0), tri6(dq, 1)};
    float w4[4];
#pragma unroll
    for (int k = 0; k < 2; ++k)
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const float w = sym_w(own[1][k], dt[kk]);
        acc[1][k].add(dt[kk].nx, dt[kk].ny, dt[kk].nz, w);
        w4[2 * k + kk] = w;
      }
    xout[d] = make_float4(w4[0], w4[1], w4[2], w4[3]);
  }
  // row above
  if (ty == 0) {  // top warp: its row above is the halo row, weigh it here
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int uq = (R0 - 1) * kSymQW + C - 1 + d;
      const Tri6 ut[2] = {tri6(uq, 0), tri6(uq, 1)};
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const float w = sym_w(ut[k], own[0][kk]);
          acc[0][kk].add(ut[k].nx, ut[k].ny, ut[k].nz, w);
        }
    }
  }
  __syncthreads();
  if (ty > 0) {
    // warp ty-1's lane at column C-1+d weighed (its quad 1 = our up quad at column
    // C-1+d) - (quad below at column C-1+d + (2-d) - 1 ... ) ; we are its d' = 2-d entry
    const float4* xin = xch + ((ty - 1) * 32) * 3;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int sl = min(max(lane - 1 + d, 0), 31);   // sender lane (column C-1+d)
      const float4 w = xin[sl * 3 + (2 - d)];
      const int uq = (R0 - 1) * kSymQW + C - 1 + d;
      const float4 un0 = nrm3(uq, 0), un1 = nrm3(uq, 1);
      // w = (U0B0, U0B1, U1B0, U1B1), U = up quad (sender's quad 1), B = our quad 0
      acc[0][0].add(un0.x, un0.y, un0.z, w.x);
      acc[0][1].add(un0.x, un0.y, un0.z, w.y);
      acc[0][0].add(un1.x, un1.y, un1.z, w.z);
      acc[0][1].add(un1.x, un1.y, un1.z, w.w);
    }
  }

  const float thr = 1e-30f * sB;
  float res[2][6];
#pragma unroll
  for (int o = 0; o < 2; ++o) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float* r = &res[o][3 * k];
      const float* n = &raw[o][3 * k];
      r[0] = n[0];
      r[1] = n[1];
      r[2] = n[2];
      const bool valid = !(isnan(n[0]) || isnan(n[1]) || isnan(n[2]));
      const float ws = acc[o][k].w;
      if (valid && ws > 0.f) {
        const float iw = rcp_approx(ws);
        const float mx = acc[o][k].x * iw, my = acc[o][k].y * iw, mz = acc[o][k].z * iw;
        const float len = sqrtf(mx * mx + my * my + mz * mz);
        if (len * ws > thr) {
          const float il = 1.0f / len;
          r[0] = mx * il;
          r[1] = my * il;
          r[2] = mz * il;
        }
      }
    }
  }

  if (SCATTER) {
    if (out_lane) {
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        const int u = u0 + 2 * ty + o, v = q0 + lane - 1;
        if (u < Mq && v < Nq) {
          const long long g = 2ll * ((long long)u * Nq + v);
          const longlong2 tm = *reinterpret_cast<const longlong2*>(a.trimap + f * a.tm_fs + g);
          float* dst = a.out_mesh + f * a.out_fs;
          if (tm.x >= 0 && tm.x < a.n_out) {
            dst[3 * tm.x] = res[o][0];
            dst[3 * tm.x + 1] = res[o][1];
            dst[3 * tm.x + 2] = res[o][2];
          }
          if (tm.y >= 0 && tm.y < a.n_out) {
            dst[3 * tm.y] = res[o][3];
            dst[3 * tm.y + 1] = res[o][4];
            dst[3 * tm.y + 2] = res[o][5];
          }
        }
      }
    }
  } else {
    if (MODE != kFromPoints) __syncthreads();  // out tile aliases the FC tile read above
    if (out_lane) {
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        float* dst = out_s + ((2 * ty + o) * kSymOut + lane - 1) * 6;
#pragma unroll
        for (int j = 0; j < 6; ++j) dst[j] = res[o][j];
      }
    }
    fence_proxy_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      tma_store_3d(&tout, out_s, q0 * 6, u0, f);
      tma_store_commit();
    }
  }
  }  // persistent tile loop (the barrier at the loop top protects pack / exchange reuse)
  if (threadIdx.x == 0) tma_store_wait_read();
}

template <int MODE, bool SCATTER>
int launch_sym(const CUtensorMap& tp, const CUtensorMap& tn, const CUtensorMap& tc,
               const CUtensorMap& to, const BilArgs& a, int F, cudaStream_t st) {
  constexpr int smem = sym_smem_bytes<MODE>();
  static unsigned long long attr_mask = 0;
  ensure_smem_attr(bilateral_sym_kernel<MODE, SCATTER>, smem, attr_mask);
  static int resident = 0;  // CTAs per SM (same on every B200 of the box)
  static int sms = 0;
  if (resident == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, bilateral_sym_kernel<MODE, SCATTER>,
                                                  256, smem);
    if (resident < 1) resident = 1;
  }
  const int Mq = a.M - 1, Nq = a.N - 1;
  const long long tiles = (long long)((Nq + kSymOut - 1) / kSymOut) *
                          ((Mq + kSymRows - 1) / kSymRows) * F;
  const int grid = (int)std::min<long long>(tiles, (long long)sms * resident);  // persistent
  bilateral_sym_kernel<MODE, SCATTER><<<grid, 256, smem, st>>>(tp, tn, tc, to, a);
  return check_launch("bilateral_sym_kernel");
}

int launch_sym_any(int mode, bool scatter, const CUtensorMap& tp, const CUtensorMap& tn,
                   const CUtensorMap& tc, const CUtensorMap& to, const BilArgs& a, int F,
                   cudaStream_t st) {
  switch (mode) {
    case kFromPoints:
      return scatter ? launch_sym<kFromPoints, true>(tp, tn, tc, to, a, F, st)
                     : launch_sym<kFromPoints, false>(tp, tn, tc, to, a, F, st);
    case kNormalsBuf:
      return scatter ? launch_sym<kNormalsBuf, true>(tp, tn, tc, to, a, F, st)
                     : launch_sym<kNormalsBuf, false>(tp, tn, tc, to, a, F, st);
    default:
      return scatter ? launch_sym<kNormalsCentBuf, true>(tp, tn, tc, to, a, F, st)
                     : launch_sym<kNormalsCentBuf, false>(tp, tn, tc, to, a, F, st);
  }
}

}  // namespace

int bilateral(const float* pts, int F, int M, int N, int pitch, const float* normals_in,
              const float* centroids_in, float sigma_length, float sigma_angle, int ksize,
              int iters, float* buf_a, float* buf_b, float* out_fc, const int64_t* trimap,
              float* out_mesh, long long out_rows, cudaStream_t st) {
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
  if (!from_arrays && (pts == nullptr || pitch < 3 * N || pitch % 4))
    return fail(ERR_INVALID, "bilateral: point grid (pitch multiple of 4 floats) required");
  const bool scatter = out_mesh != nullptr;
  if (scatter && trimap == nullptr) return fail(ERR_INVALID, "bilateral: scatter needs trimap");
  if (!scatter && out_fc == nullptr) return fail(ERR_INVALID, "bilateral: no output given");
  if ((iters > 1 && !buf_a) || (iters > 2 && !buf_b))
    return fail(ERR_INVALID, "bilateral: ping-pong buffers required");

  const int Mq = M - 1, Nq = N - 1;
  const int fcp = fc_pitch(N);
  const uint64_t fc_fs = (uint64_t)Mq * fcp;
  const bool sym = (h == 1) && !g_bil_direct;
  const int QW = sym ? kSymQW : box_q(h), QH = sym ? kSymQH : kBilTQH + 2 * h;
  const int PW = sym ? kSymPW : box_p(h), PH = QH + 1;
  const int SW = sym ? kSymOut : kBilTQW, SH = sym ? kSymRows : kBilTQH;  // store box
  // kernel parameters need a valid encoding even where a mode ignores the map
  CUtensorMap m_pts, m_nin, m_cin, ld_a, st_a, ld_b, st_b, st_fin;
  int rc;
  auto fc_load = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, QW * 6, QH);
  };
  auto fc_store = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, SW * 6, SH);
  };
  if (from_arrays) {
    if ((rc = fc_load(&m_nin, normals_in)) || (rc = fc_load(&m_cin, centroids_in))) return rc;
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
  a.out_fs = 3ll * out_rows;
  a.n_out = out_rows;
  a.raw_pitch = fcp;
  a.raw_fs = (long long)fc_fs;

  // it0 reads (points | arrays) and writes A; it_k reads A/B and writes B/A; the last
  // iteration scatters to mesh order (trimap) or stores to out_fc.
  const CUtensorMap* src_n = &m_nin;
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    const int mode = from_arrays ? kNormalsCentBuf
                                 : ((it == 0 && !resume) ? kFromPoints : kNormalsBuf);
    const CUtensorMap* dst = last ? &st_fin : ((it % 2 == 0) ? &st_a : &st_b);
    a.raw_n = (it == 0) ? normals_in : (((it - 1) % 2 == 0) ? buf_a : buf_b);
    rc = sym ? launch_sym_any(mode, last && scatter, m_pts, *src_n, m_cin, *dst, a, F, st)
             : launch_h(h, mode, last && scatter, m_pts, *src_n, m_cin, *dst, a, F, st);
    if (rc) return rc;
    src_n = (it % 2 == 0) ? &ld_a : &ld_b;
  }
  return OK;
}

}  // namespace opcfe
