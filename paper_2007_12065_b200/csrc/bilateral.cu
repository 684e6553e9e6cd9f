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
// B200 mapping: one CTA = 32x8 quads (both triangles of a quad per thread, so each
// neighbour quad is read once from shared memory for two outputs).  Tile+halo
// inputs arrive by TMA 3-D box loads with NaN out-of-bounds fill (== the
// reference's "off-grid neighbours are skipped"): the point tile (centroids are
// recomputed from points every iteration: 12 B/point instead of 24 B/quad of
// stored centroids) and, after iteration 1, the previous normal tile.  Iteration 1
// computes the FC normals with fp64 edges + cross product (no cancellation on
// slivers) and an fp32 normalisation.  Weights use ex2 with
// pre-scaled exponents; the |acc| > 1e-30 test is evaluated underflow-safely as
// |acc/wsum| * wsum > 1e-30.
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

namespace {

constexpr int kBilTQW = 32;  // interior quads per tile row (= one warp)
constexpr int kBilTQH = 8;   // interior quad rows per tile
constexpr int kBilNT = kBilTQW * kBilTQH;

enum BilMode : int {
  kFromPoints = 0,     // iteration 1: normals + centroids from the point grid
  kNormalsBuf = 1,     // normals from the previous iteration, centroids from points
  kNormalsCentBuf = 2  // normals and centroids from FC arrays (drop-in bilateral_iterate)
};

template <int H>
struct BilTile {
  // TMA rule: box starts along the innermost dimension must be 16-B aligned.  FC rows
  // are 24 B per quad -> start LQ = round_up(H, 2) quads left of the tile; point rows
  // are 12 B per point -> start LP = round_up(H, 4) points left.
  static constexpr int LQ = (H + 1) / 2 * 2;
  static constexpr int LP = (H + 3) / 4 * 4;
  static constexpr int QW = ((LQ + kBilTQW + H + 1) / 2) * 2;  // FC box width (quads)
  static constexpr int QH = kBilTQH + 2 * H;
  static constexpr int PW = ((LP + kBilTQW + H + 1 + 3) / 4) * 4;  // point box width
  static constexpr int PH = QH + 1;
  static constexpr int PSHIFT = LP - LQ;  // point column of pack column 0
  static constexpr int PTS_F = ((PW * 3 * PH) + 31) / 32 * 32;
  static constexpr int FC_F = ((QW * 6 * QH) + 31) / 32 * 32;
  static constexpr int PACK_F = QW * QH * 12;
  static constexpr int OUT_F = kBilTQW * 6 * kBilTQH;
  static_assert(QW * 6 <= 256 && PW * 3 <= 256, "TMA box inner extent must be <= 256");
  static_assert((QW * 6) % 4 == 0, "FC box rows must be 16-B multiples");
};

template <int H, int MODE>
constexpr int bil_smem_bytes() {
  using T = BilTile<H>;
  return (((MODE != kNormalsCentBuf) ? T::PTS_F : 0) + ((MODE != kFromPoints) ? T::FC_F : 0) +
          ((MODE == kNormalsCentBuf) ? T::FC_F : 0) + T::PACK_F + T::OUT_F) *
             4 +
         kSmemSlack;
}

struct BilArgs {
  int M, N;          // point grid (Mq = M-1, Nq = N-1 quads)
  float A, B;        // log2(e)/(2 sl^2), log2(e)/(2 sa^2)
  const int64_t* trimap;  // scatter mode: per frame [G]
  long long tm_fs;
  float* out_mesh;   // scatter destination: per frame [cap][3]
  long long out_fs;  // floats per frame
  long long n_out;   // rows per frame available in out_mesh (bounds check)
};

// FC normal for the bilateral input: edges and cross product in fp64 (exact edge
// differences of fp32 vertices; no cancellation on slivers), normalisation in fp32.
// |n - float32(reference)| ~ 1e-7, far inside the 1e-5 contract, at ~1/8 the cost of
// the correctly rounded fp64 divide/sqrt used where bit-exact normals are returned.
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
    const float gx = fx / sc, gy = fy / sc, gz = fz / sc;
    const float r = rsqrtf(gx * gx + gy * gy + gz * gz);
    n[0] = gx * r;
    n[1] = gy * r;
    n[2] = gz * r;
  } else {
    n[0] = n[1] = n[2] = __int_as_float(0x7fc00000);
  }
}

template <int H, int MODE, bool SCATTER>
__global__ void __launch_bounds__(kBilNT)
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
  float4* pack = reinterpret_cast<float4*>(p);
  p += T::PACK_F;
  float* out_s = p;
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

  // ---- build the packed per-quad record {n0, n1, c0, c1} for interior + halo
  for (int q = threadIdx.x; q < T::QW * T::QH; q += kBilNT) {
    const int r = q / T::QW, c = q % T::QW;
    float n[6], cc[6];
    if (MODE == kNormalsCentBuf) {
#pragma unroll
      for (int j = 0; j < 6; ++j) {
        n[j] = nrm_s[(r * T::QW + c) * 6 + j];
        cc[j] = cen_s[(r * T::QW + c) * 6 + j];
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
        for (int j = 0; j < 6; ++j) n[j] = nrm_s[(r * T::QW + c) * 6 + j];
      }
    }
    float4* rec = pack + (r * T::QW + c) * 3;
    rec[0] = make_float4(n[0], n[1], n[2], n[3]);
    rec[1] = make_float4(n[4], n[5], cc[0], cc[1]);
    rec[2] = make_float4(cc[2], cc[3], cc[4], cc[5]);
  }
  __syncthreads();

  // ---- one thread per interior quad: both triangles
  const int tx = threadIdx.x % kBilTQW, ty = threadIdx.x / kBilTQW;
  const int u = u0 + ty, v = q0 + tx;
  const float4* own = pack + ((ty + H) * T::QW + (tx + T::LQ)) * 3;
  const float4 o0 = own[0], o1 = own[1], o2 = own[2];
  const float n0x = o0.x, n0y = o0.y, n0z = o0.z, n1x = o0.w, n1y = o1.x, n1z = o1.y;
  const float c0x = o1.z, c0y = o1.w, c0z = o2.x, c1x = o2.y, c1y = o2.z, c1z = o2.w;
  const bool val0 = !(isnan(n0x) || isnan(n0y) || isnan(n0z));
  const bool val1 = !(isnan(n1x) || isnan(n1y) || isnan(n1z));
  float a0x = 0.f, a0y = 0.f, a0z = 0.f, w0s = 0.f;
  float a1x = 0.f, a1y = 0.f, a1z = 0.f, w1s = 0.f;
  const float A = a.A, B = a.B;
  if (val0 || val1) {
#pragma unroll
    for (int du = -H; du <= H; ++du) {
#pragma unroll
      for (int dv = -H; dv <= H; ++dv) {
        const float4* nb = own + (du * T::QW + dv) * 3;
        const float4 r0 = nb[0], r1 = nb[1], r2 = nb[2];
        const float m[2][3] = {{r0.x, r0.y, r0.z}, {r0.w, r1.x, r1.y}};
        const float d[2][3] = {{r1.z, r1.w, r2.x}, {r2.y, r2.z, r2.w}};
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          // neighbour triangle kk vs own triangle 0
          if (!(du == 0 && dv == 0 && kk == 0)) {
            const float ex = d[kk][0] - c0x, ey = d[kk][1] - c0y, ez = d[kk][2] - c0z;
            const float fx = m[kk][0] - n0x, fy = m[kk][1] - n0y, fz = m[kk][2] - n0z;
            const float dc2 = ex * ex + ey * ey + ez * ez;
            const float dn2 = fx * fx + fy * fy + fz * fz;
            const float w = ex2_approx(-(dc2 * A + dn2 * B));
            if (w == w) {  // NaN neighbour normal / centroid -> skipped
              a0x += m[kk][0] * w;
              a0y += m[kk][1] * w;
              a0z += m[kk][2] * w;
              w0s += w;
            }
          }
          if (!(du == 0 && dv == 0 && kk == 1)) {
            const float ex = d[kk][0] - c1x, ey = d[kk][1] - c1y, ez = d[kk][2] - c1z;
            const float fx = m[kk][0] - n1x, fy = m[kk][1] - n1y, fz = m[kk][2] - n1z;
            const float dc2 = ex * ex + ey * ey + ez * ez;
            const float dn2 = fx * fx + fy * fy + fz * fz;
            const float w = ex2_approx(-(dc2 * A + dn2 * B));
            if (w == w) {
              a1x += m[kk][0] * w;
              a1y += m[kk][1] * w;
              a1z += m[kk][2] * w;
              w1s += w;
            }
          }
        }
      }
    }
  }
  // underflow-safe normalisation: n = m/|m|, m = acc/wsum; |acc| > 1e-30 <=> |m|*wsum > 1e-30
  float r0x = n0x, r0y = n0y, r0z = n0z, r1x = n1x, r1y = n1y, r1z = n1z;
  if (val0 && w0s > 0.f) {
    const float iw = 1.f / w0s;
    const float mx = a0x * iw, my = a0y * iw, mz = a0z * iw;
    const float len = sqrtf(mx * mx + my * my + mz * mz);
    if (len * w0s > 1e-30f) {
      r0x = mx / len;
      r0y = my / len;
      r0z = mz / len;
    }
  }
  if (val1 && w1s > 0.f) {
    const float iw = 1.f / w1s;
    const float mx = a1x * iw, my = a1y * iw, mz = a1z * iw;
    const float len = sqrtf(mx * mx + my * my + mz * mz);
    if (len * w1s > 1e-30f) {
      r1x = mx / len;
      r1y = my / len;
      r1z = mz / len;
    }
  }

  if (SCATTER) {
    if (u < Mq && v < Nq) {
      const long long g = 2ll * ((long long)u * Nq + v);
      const longlong2 tm = *reinterpret_cast<const longlong2*>(a.trimap + f * a.tm_fs + g);
      float* o = a.out_mesh + f * a.out_fs;
      if (tm.x >= 0 && tm.x < a.n_out) {
        o[3 * tm.x] = r0x;
        o[3 * tm.x + 1] = r0y;
        o[3 * tm.x + 2] = r0z;
      }
      if (tm.y >= 0 && tm.y < a.n_out) {
        o[3 * tm.y] = r1x;
        o[3 * tm.y + 1] = r1y;
        o[3 * tm.y + 2] = r1z;
      }
    }
  } else {
    float* o = out_s + (ty * kBilTQW + tx) * 6;
    o[0] = r0x;
    o[1] = r0y;
    o[2] = r0z;
    o[3] = r1x;
    o[4] = r1y;
    o[5] = r1z;
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
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bilateral_kernel<H, MODE, SCATTER>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int Mq = a.M - 1, Nq = a.N - 1;
  dim3 grid((Nq + kBilTQW - 1) / kBilTQW, (Mq + kBilTQH - 1) / kBilTQH, F);
  bilateral_kernel<H, MODE, SCATTER><<<grid, kBilNT, smem, st>>>(tp, tn, tc, to, a);
  return check_launch("bilateral_kernel");
}

template <int H, int MODE>
int launch_mode(bool scatter, const CUtensorMap& tp, const CUtensorMap& tn, const CUtensorMap& tc,
                const CUtensorMap& to, const BilArgs& a, int F, cudaStream_t st) {
  return scatter ? launch_bil<H, MODE, true>(tp, tn, tc, to, a, F, st)
                 : launch_bil<H, MODE, false>(tp, tn, tc, to, a, F, st);
}

template <int H>
int launch_any(int mode, bool scatter, const CUtensorMap& tp, const CUtensorMap& tn,
               const CUtensorMap& tc, const CUtensorMap& to, const BilArgs& a, int F,
               cudaStream_t st) {
  switch (mode) {
    case kFromPoints: return launch_mode<H, kFromPoints>(scatter, tp, tn, tc, to, a, F, st);
    case kNormalsBuf: return launch_mode<H, kNormalsBuf>(scatter, tp, tn, tc, to, a, F, st);
    default: return launch_mode<H, kNormalsCentBuf>(scatter, tp, tn, tc, to, a, F, st);
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

struct Maps {
  CUtensorMap pts, nin, cin, ld_a, st_a, ld_b, st_b;
};

int box_q(int h) { return ((((h + 1) / 2 * 2) + kBilTQW + h + 1) / 2) * 2; }
int box_p(int h) { return ((((h + 3) / 4 * 4) + kBilTQW + h + 1 + 3) / 4) * 4; }

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
  const bool from_arrays = normals_in != nullptr;
  if (from_arrays && centroids_in == nullptr)
    return fail(ERR_INVALID, "bilateral: FC normals given without FC centroids");
  if (!from_arrays && (pts == nullptr || pitch < 3 * N || pitch % 4))
    return fail(ERR_INVALID, "bilateral: point grid (pitch multiple of 4 floats) required");
  const bool scatter = out_mesh != nullptr;
  if (scatter && trimap == nullptr) return fail(ERR_INVALID, "bilateral: scatter needs trimap");
  if (!scatter && out_fc == nullptr) return fail(ERR_INVALID, "bilateral: no output given");
  const int nbuf_needed = (iters > 1 ? 1 : 0) + (iters > 2 ? 1 : 0);
  if ((nbuf_needed >= 1 && !buf_a) || (nbuf_needed >= 2 && !buf_b))
    return fail(ERR_INVALID, "bilateral: ping-pong buffers required");

  const int Mq = M - 1, Nq = N - 1;
  const int fcp = fc_pitch(N);
  const uint64_t fc_fs = (uint64_t)Mq * fcp;
  const uint64_t pt_fs = (uint64_t)M * pitch;
  const int QW = box_q(h), QH = kBilTQH + 2 * h, PW = box_p(h), PH = QH + 1;
  Maps mp;
  int rc;
  const float* any = from_arrays ? normals_in : pts;
  // unused maps still need a valid encoding (kernel params); point them at `any`
  if (!from_arrays) {
    if ((rc = make_tmap_3d(&mp.pts, pts, false, 3ull * N, M, F, pitch, pt_fs, PW * 3, PH))) return rc;
  }
  auto fc_load = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, QW * 6, QH);
  };
  auto fc_store = [&](CUtensorMap* m, const float* b) {
    return make_tmap_3d(m, b, false, 6ull * Nq, Mq, F, fcp, fc_fs, kBilTQW * 6, kBilTQH);
  };
  if (from_arrays) {
    if ((rc = fc_load(&mp.nin, normals_in))) return rc;
    if ((rc = fc_load(&mp.cin, centroids_in))) return rc;
    mp.pts = mp.nin;
  } else {
    mp.nin = mp.pts;
    mp.cin = mp.pts;
  }
  float* fin_dst = scatter ? nullptr : out_fc;
  CUtensorMap st_fin;
  if (fin_dst) {
    if ((rc = fc_store(&st_fin, fin_dst))) return rc;
  } else {
    st_fin = mp.pts;
  }
  if (buf_a) {
    if ((rc = fc_load(&mp.ld_a, buf_a)) || (rc = fc_store(&mp.st_a, buf_a))) return rc;
  }
  if (buf_b) {
    if ((rc = fc_load(&mp.ld_b, buf_b)) || (rc = fc_store(&mp.st_b, buf_b))) return rc;
  }
  (void)any;

  BilArgs a;
  a.M = M;
  a.N = N;
  const float log2e = 1.4426950408889634f;
  a.A = (float)(1.4426950408889634 / (2.0 * (double)sigma_length * (double)sigma_length));
  a.B = (float)(1.4426950408889634 / (2.0 * (double)sigma_angle * (double)sigma_angle));
  (void)log2e;
  a.trimap = trimap;
  a.tm_fs = 2ll * Mq * Nq;
  a.out_mesh = out_mesh;
  a.out_fs = 3ll * out_rows;
  a.n_out = out_rows;

  // iteration schedule: it0 reads (points | arrays), writes A; itk reads A/B, writes B/A;
  // last iteration scatters (mesh order) or stores to out_fc.
  const CUtensorMap* src_n = &mp.nin;
  for (int it = 0; it < iters; ++it) {
    const bool last = it == iters - 1;
    const int mode = it == 0 ? (from_arrays ? kNormalsCentBuf : kFromPoints)
                             : (from_arrays ? kNormalsCentBuf : kNormalsBuf);
    const CUtensorMap* dst = last ? &st_fin : ((it % 2 == 0) ? &mp.st_a : &mp.st_b);
    rc = launch_h(h, mode, last && scatter, mp.pts, *src_n, mp.cin, *dst, a, F, st);
    if (rc) return rc;
    src_n = (it % 2 == 0) ? &mp.ld_a : &mp.ld_b;
  }
  return OK;
}

}  // namespace opcfe
