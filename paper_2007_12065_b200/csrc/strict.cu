// Strict (fp64) front-end kernels: the reference's own arithmetic, in its own operation
// order, on the reference's own float64 layouts -- any odd kernel size.
//
//   laplacian_f64   _kernels.laplacian_filter (_native.pyx:225-284; _fallback.py:82-117)
//                   bit-identical to the reference: IEEE dmul / dadd / sqrt / div, no FMA
//                   contraction (the reference is built with -ffp-contract=off,
//                   setup.py:24-26), neighbours in the same du-outer / dv-inner order.
//   bilateral_f64   _kernels.bilateral_iterate (_native.pyx:287-364; _fallback.py:120-166)
//                   + the trimap gather of bilateral_filter_opc (smoothing.py:108-114):
//                   same arithmetic and accumulation order; only exp() differs (CUDA's
//                   vs libm's, both <= 1 ulp -- the reference's own two backends differ
//                   by as much).
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

namespace opcfe {

namespace {

constexpr int kSTW = 32;  // tile width (points / quads) = one warp
constexpr int kSTH = 8;   // tile height (rows) = warps per CTA
constexpr int kSNT = kSTW * kSTH;
constexpr int kSmemMax = 200 * 1024;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000LL); }

// ------------------------------------------------------------------ Laplacian
// in/out: [F][M][N][3].  HC > 0: compile-time half width; HC == 0: runtime h.
// SMEM: the tile + halo is staged in three planes of (kSTH+2h) x (kSTW+2h) doubles;
// out-of-grid cells hold NaN (the reference skips them; a NaN distance is skipped too).
template <int HC, bool SMEM>
__global__ void __launch_bounds__(kSNT) laplacian_f64_kernel(const double* __restrict__ in,
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
  if (SMEM) {
    const int u0 = blockIdx.y * kSTH - h, v0 = blockIdx.x * kSTW - h;
    const int tid = ty * kSTW + tx;
    const int rowlen = 3 * bw;
    for (int i = tid; i < rowlen * bh; i += kSNT) {
      const int r = i / rowlen, c3 = i - r * rowlen;
      const int c = c3 / 3, comp = c3 - 3 * c;
      const int uu = u0 + r, vv = v0 + c;
      const double x = (uu >= 0 && uu < M && vv >= 0 && vv < N)
                           ? src[((long long)uu * N + vv) * 3 + comp]
                           : qnan();
      sm[comp * plane + r * bw + c] = x;
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
      const double w = __ddiv_rn(1.0, dist);
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
};

template <int HC, bool SMEM, typename OUT>
__global__ void __launch_bounds__(kSNT) bilateral_f64_kernel(Bil64Args a) {
  const int h = HC > 0 ? HC : a.h;
  const int Mq = a.Mq, Nq = a.Nq;
  const int f = blockIdx.z;
  const long long fs = 6ll * Mq * Nq;
  const double* cen = a.cen + f * fs;
  const double* nrm = a.nin + f * fs;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int u = blockIdx.y * kSTH + ty, v = blockIdx.x * kSTW + tx;
  extern __shared__ double sm[];
  const int bw = kSTW + 2 * h, bh = kSTH + 2 * h, plane = bw * bh;
  // plane index: (k * 2 + {0 centroid, 1 normal}) * 3 + comp
  if (SMEM) {
    const int u0 = blockIdx.y * kSTH - h, v0 = blockIdx.x * kSTW - h;
    const int tid = ty * kSTW + tx;
    const int rowlen = 6 * bw;  // doubles of one array per box row
    for (int i = tid; i < 2 * rowlen * bh; i += kSNT) {
      const int arr = i >= rowlen * bh;  // 0 centroids, 1 normals
      const int j = i - arr * rowlen * bh;
      const int r = j / rowlen, c6 = j - r * rowlen;
      const int c = c6 / 6, kc = c6 - 6 * c, k = kc / 3, comp = kc - 3 * k;
      const int uu = u0 + r, vv = v0 + c;
      const double* base = arr ? nrm : cen;
      const double x = (uu >= 0 && uu < Mq && vv >= 0 && vv < Nq)
                           ? base[((long long)uu * Nq + vv) * 6 + kc]
                           : qnan();
      sm[((k * 2 + arr) * 3 + comp) * plane + r * bw + c] = x;
    }
    __syncthreads();
  }
  if (u >= Mq || v >= Nq) return;
  const long long qo = ((long long)u * Nq + v) * 6;
#pragma unroll 1
  for (int k = 0; k < 2; ++k) {
    double cx, cy, cz, nx, ny, nz;
    if (SMEM) {
      const int c = (ty + h) * bw + tx + h;
      cx = sm[((k * 2) * 3 + 0) * plane + c];
      cy = sm[((k * 2) * 3 + 1) * plane + c];
      cz = sm[((k * 2) * 3 + 2) * plane + c];
      nx = sm[((k * 2 + 1) * 3 + 0) * plane + c];
      ny = sm[((k * 2 + 1) * 3 + 1) * plane + c];
      nz = sm[((k * 2 + 1) * 3 + 2) * plane + c];
    } else {
      cx = cen[qo + 3 * k];
      cy = cen[qo + 3 * k + 1];
      cz = cen[qo + 3 * k + 2];
      nx = nrm[qo + 3 * k];
      ny = nrm[qo + 3 * k + 1];
      nz = nrm[qo + 3 * k + 2];
    }
    double rx = nx, ry = ny, rz = nz;  // NaN centre: kept (:313-318)
    if (!(nx != nx || ny != ny || nz != nz)) {
      double wsum = 0.0, ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
      for (int du = -h; du <= h; ++du) {
        const int uu = u + du;
        if (!SMEM && (uu < 0 || uu >= Mq)) continue;
#pragma unroll
        for (int dv = -h; dv <= h; ++dv) {
          const int vv = v + dv;
          if (!SMEM && (vv < 0 || vv >= Nq)) continue;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            if (du == 0 && dv == 0 && kk == k) continue;
            double mx, my, mz, qx, qy, qz;
            if (SMEM) {
              const int c = (ty + h + du) * bw + tx + h + dv;
              mx = sm[((kk * 2 + 1) * 3 + 0) * plane + c];
              my = sm[((kk * 2 + 1) * 3 + 1) * plane + c];
              mz = sm[((kk * 2 + 1) * 3 + 2) * plane + c];
              qx = sm[((kk * 2) * 3 + 0) * plane + c];
              qy = sm[((kk * 2) * 3 + 1) * plane + c];
              qz = sm[((kk * 2) * 3 + 2) * plane + c];
            } else {
              const long long o = ((long long)uu * Nq + vv) * 6 + 3 * kk;
              mx = __ldg(nrm + o);
              my = __ldg(nrm + o + 1);
              mz = __ldg(nrm + o + 2);
              qx = __ldg(cen + o);
              qy = __ldg(cen + o + 1);
              qz = __ldg(cen + o + 2);
            }
            if (mx != mx || my != my || mz != mz) continue;  // (:337-338)
            double dx = dsub(qx, cx), dy = dsub(qy, cy), dz = dsub(qz, cz);
            const double dc2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
            dx = dsub(mx, nx);
            dy = dsub(my, ny);
            dz = dsub(mz, nz);
            const double dn2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
            const double w = exp(dsub(dmul(-dc2, a.inv2sc), dmul(dn2, a.inv2ss)));
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

template <int HC, bool SMEM, typename OUT>
int bil_launch(const Bil64Args& a, int F, cudaStream_t st) {
  const int smem = SMEM ? bil_smem(a.h) : 0;
  int rc;
  if ((rc = set_smem(bilateral_f64_kernel<HC, SMEM, OUT>, smem))) return rc;
  dim3 grid((a.Nq + kSTW - 1) / kSTW, (a.Mq + kSTH - 1) / kSTH, F);
  bilateral_f64_kernel<HC, SMEM, OUT><<<grid, dim3(kSTW, kSTH), smem, st>>>(a);
  return check_launch("bilateral_f64_kernel");
}

template <typename OUT>
int bil_dispatch(const Bil64Args& a, int F, cudaStream_t st) {
  if (a.h == 1) return bil_launch<1, true, OUT>(a, F, st);
  if (a.h == 2) return bil_launch<2, true, OUT>(a, F, st);
  if (bil_smem(a.h) <= kSmemMax) return bil_launch<0, true, OUT>(a, F, st);
  return bil_launch<0, false, OUT>(a, F, st);
}

}  // namespace

int laplacian_f64(const double* in, double* out, double* tmp, int F, int M, int N, double lam,
                  int ksize, int iters, cudaStream_t st) {
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
    if (h == 1) rc = lap_launch<1, true>(src, dst, F, M, N, h, lam, st);
    else if (h == 2) rc = lap_launch<2, true>(src, dst, F, M, N, h, lam, st);
    else if (lap_smem(h) <= kSmemMax) rc = lap_launch<0, true>(src, dst, F, M, N, h, lam, st);
    else rc = lap_launch<0, false>(src, dst, F, M, N, h, lam, st);
    if (rc) return rc;
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

int fc_data_f64(const double* opc, int F, int M, int N, double* cen, double* nrm,
                cudaStream_t st) {
  if (F < 1 || M < 2 || N < 2) return fail(ERR_INVALID, "organized cloud must be at least 2 x 2");
  const long long Q = (long long)(M - 1) * (N - 1);
  fc_data_f64_kernel<<<dim3(nblk(Q, 256), F), 256, 0, st>>>(opc, M, N, cen, nrm);
  return check_launch("fc_data_f64_kernel");
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
