// Per-vertex / per-quad / per-triangle kernels of the front-end:
//   stage_in          (F,M,N,3) f32|f64 contiguous -> pitched fp32 grid + 1-bit validity mask
//   fc_data           compute_fc_triangle_data (smoothing.py:61-88), bit-exact in fp64
//   triangle_normals  geometry.triangle_normals (geometry.py:134-147), bit-exact in fp64
//   max_edge_mask     segmentation.group_assignment's l_max part (segmentation.py:59-67,73)
// All fp64 arithmetic uses the no-contraction helpers of common.cuh so results
// reproduce numpy bit for bit.  These are HBM-bound streaming kernels: one thread
// per element, warp-contiguous addresses.
#include "common.cuh"
#include "opcfe_internal.h"

#include <algorithm>

namespace opcfe {

namespace {

template <typename S>
__global__ void stage_in_kernel(const S* __restrict__ src, long long rs, long long fs,
                                float* __restrict__ dst, int pitch, uint32_t* __restrict__ vmask,
                                int wpr, int M, int N) {
  const int v = blockIdx.x * 32 + threadIdx.x;
  const int u = blockIdx.y * blockDim.y + threadIdx.y;
  const int f = blockIdx.z;
  if (u >= M) return;  // warp-uniform: a warp is one row segment
  bool ok = false;
  if (v < N) {
    const S* s = src + f * fs + u * rs + 3ll * v;
    const S x = s[0], y = s[1], z = s[2];
    ok = isfinite(x) && isfinite(y) && isfinite(z);  // validity from the SOURCE precision
    if (dst != nullptr) {
      float* d = dst + ((long long)f * M + u) * pitch + 3 * v;
      d[0] = (float)x;
      d[1] = (float)y;
      d[2] = (float)z;
    }
  }
  const uint32_t bits = __ballot_sync(0xffffffffu, ok);
  if (threadIdx.x == 0 && vmask != nullptr) vmask[((long long)f * M + u) * wpr + blockIdx.x] = bits;
}

template <typename S>
__device__ __forceinline__ double ld(const S* p) {
  return (double)*p;
}

template <typename S>
__global__ void fc_data_kernel(const S* __restrict__ opc, int M, int N, S* __restrict__ cen,
                               S* __restrict__ nrm) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int Nq = N - 1;
  if (q >= (long long)(M - 1) * Nq) return;
  const int u = (int)(q / Nq), v = (int)(q % Nq);
  const S* p1 = opc + ((long long)u * N + v) * 3;
  const S* p2 = p1 + 3;
  const S* p4 = p1 + (long long)N * 3;
  const S* p3 = p4 + 3;
  const S* tri[2][3] = {{p3, p2, p1}, {p1, p4, p3}};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const S *a = tri[k][0], *b = tri[k][1], *c = tri[k][2];
    S* co = cen + (q * 2 + k) * 3;
    S* no = nrm + (q * 2 + k) * 3;
#pragma unroll
    for (int j = 0; j < 3; ++j) co[j] = (S)centroid_f64(ld(a + j), ld(b + j), ld(c + j));
    double nx, ny, nz;
    unit_normal_f64(ld(a), ld(a + 1), ld(a + 2), ld(b), ld(b + 1), ld(b + 2), ld(c), ld(c + 1),
                    ld(c + 2), nx, ny, nz);
    no[0] = (S)nx;
    no[1] = (S)ny;
    no[2] = (S)nz;
  }
}

template <typename S>
__global__ void tri_normals_kernel(const S* __restrict__ pts, const int64_t* __restrict__ tris,
                                   long long T, S* __restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const S* a = pts + tris[3 * t] * 3;
  const S* b = pts + tris[3 * t + 1] * 3;
  const S* c = pts + tris[3 * t + 2] * 3;
  double nx, ny, nz;
  unit_normal_f64(ld(a), ld(a + 1), ld(a + 2), ld(b), ld(b + 1), ld(b + 2), ld(c), ld(c + 1),
                  ld(c + 2), nx, ny, nz);
  out[3 * t] = (S)nx;
  out[3 * t + 1] = (S)ny;
  out[3 * t + 2] = (S)nz;
}

template <typename S>
__global__ void max_edge_kernel(const S* __restrict__ pts, const int64_t* __restrict__ tris,
                                long long T, double l2_thr, uint8_t* __restrict__ flag) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const S* a = pts + tris[3 * t] * 3;
  const S* b = pts + tris[3 * t + 1] * 3;
  const S* c = pts + tris[3 * t + 2] * 3;
  flag[t] = (uint8_t)longest_edge_exceeds(
      edge_len2_f64(ld(a), ld(a + 1), ld(a + 2), ld(b), ld(b + 1), ld(b + 2)),
      edge_len2_f64(ld(b), ld(b + 1), ld(b + 2), ld(c), ld(c + 1), ld(c + 2)),
      edge_len2_f64(ld(c), ld(c + 1), ld(c + 2), ld(a), ld(a + 1), ld(a + 2)), l2_thr);
}


// padded fp32 grid -> contiguous f32|f64 (F,M,N,3).  With `orig` (the caller's input,
// same dtype as dst): components whose fp32 value equals float(orig) return orig
// bit-exactly -- every vertex/normal the filter leaves unchanged (outer ring, NaN and
// isolated vertices, unchanged normals) is returned exactly as given (smoothing.py:57,
// _fallback.py:111-115).
template <typename D>
__global__ void unstage_kernel(const float* __restrict__ src, int pitch, int M, int N,
                               D* __restrict__ dst, const D* __restrict__ orig) {
  const long long n = (long long)M * N * 3;
  const int f = blockIdx.y;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long row = i / (3ll * N), col = i % (3ll * N);
    const float x = src[((long long)f * M + row) * pitch + col];
    D y = (D)x;
    if (orig != nullptr) {
      const D o = orig[f * n + i];
      if ((float)o == x) y = o;
    }
    dst[f * n + i] = y;
  }
}

// group_assignment (segmentation.py:52-74): per triangle, argmax over the dominant normals
// of n . d (first maximum wins; NaN counts as maximal, numpy argmax), UNASSIGNED (255)
// unless best >= ang_min, and 255 where the l_max flag is set.  The dot products use the
// FMA chain fma(n2,d2, fma(n1,d1, n0*d0)) in fp64 -- the k-loop of the OpenBLAS dgemm
// kernel numpy's `normals @ dn.T` dispatches to (checked bit-for-bit in this image), so
// labels match the reference except at exact-rounding ties between two scores.
// Frames: `T` rows per frame with the live count in n_tri[f] (nullable = all rows).
template <typename S>
__global__ void group_assign_kernel(const S* __restrict__ normals, long long T, int F,
                                    const int64_t* __restrict__ n_tri,
                                    const double* __restrict__ dn, int G, double ang_min,
                                    const uint8_t* __restrict__ lflag, uint8_t* __restrict__ labels) {
  __shared__ double sd[254 * 3];
  for (int i = threadIdx.x; i < 3 * G; i += blockDim.x) sd[i] = dn[i];
  __syncthreads();
  const int f = blockIdx.y;
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long live = n_tri ? n_tri[f] : T;
  if (t >= live || t >= T) return;
  const long long row = f * T + t;
  const double n0 = (double)normals[3 * row], n1 = (double)normals[3 * row + 1],
               n2 = (double)normals[3 * row + 2];
  double best = fma(n2, sd[2], fma(n1, sd[1], n0 * sd[0]));
  int arg = 0;
  for (int g = 1; g < G; ++g) {
    if (isnan(best)) break;  // the first NaN is the argmax
    const double s = fma(n2, sd[3 * g + 2], fma(n1, sd[3 * g + 1], n0 * sd[3 * g]));
    if (isnan(s) || s > best) {
      best = s;
      arg = g;
    }
  }
  uint8_t lab = (uint8_t)arg;
  if (!(best >= ang_min)) lab = 255;  // catches NaN normals too (segmentation.py:72)
  if (lflag != nullptr && lflag[row]) lab = 255;
  labels[row] = lab;
}

// int64 index arrays -> int32 (the compact, non-reference output mode): frame f's first
// n_rows[f] rows (all `rows` when n_rows is NULL) of `width` indices each.  Values are
// < 2^31 by the caller's check; -1 stays -1.  Streaming: 8 B in, 4 B out per index.
__global__ void narrow_indices_kernel(const int64_t* __restrict__ src, int32_t* __restrict__ dst,
                                      long long rows, int width, const int64_t* __restrict__ n_rows,
                                      long long src_fs, long long dst_fs) {
  const int f = blockIdx.y;
  const long long n = (n_rows ? n_rows[f] : rows) * width;
  const int64_t* s = src + f * src_fs;
  int32_t* d = dst + f * dst_fs;
  for (long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x); i < n;
       i += 2ll * gridDim.x * blockDim.x) {
    const bool vec = reinterpret_cast<uintptr_t>(s + i) % 16 == 0 &&
                     reinterpret_cast<uintptr_t>(d + i) % 8 == 0;
    if (i + 1 < n && vec) {
      const longlong2 x = *reinterpret_cast<const longlong2*>(s + i);
      *reinterpret_cast<int2*>(d + i) = make_int2((int)x.x, (int)x.y);
    } else {
      d[i] = (int32_t)s[i];
      if (i + 1 < n) d[i + 1] = (int32_t)s[i + 1];
    }
  }
}

// Count of the valid (>= 0) entries of a GID map and its largest entry: the row count of
// bilateral_filter_opc's output (smoothing.py:110-112: `valid.sum()`) and the bound its
// `out[trimap[valid]]` scatter checks.  stats[0] += count, stats[1] = max(stats[1], max);
// the caller pre-sets stats to {0, -1}.
__global__ void trimap_stats_kernel(const int64_t* __restrict__ tm, long long n,
                                    long long* __restrict__ stats) {
  long long cnt = 0, mx = -1;
  const long long stride = 2ll * gridDim.x * blockDim.x;
  long long i = 2 * ((long long)blockIdx.x * blockDim.x + threadIdx.x);
  if (reinterpret_cast<uintptr_t>(tm) % 16 == 0) {
    for (; i + 1 < n; i += stride) {
      const longlong2 x = __ldcs(reinterpret_cast<const longlong2*>(tm + i));
      cnt += (x.x >= 0) + (x.y >= 0);
      mx = max(mx, max(x.x, x.y));
    }
  } else {
    for (; i + 1 < n; i += stride) {
      const long long a = tm[i], b = tm[i + 1];
      cnt += (a >= 0) + (b >= 0);
      mx = max(mx, max(a, b));
    }
  }
  if (i < n) {  // the odd tail element
    cnt += tm[i] >= 0;
    mx = max(mx, (long long)tm[i]);
  }
  for (int o = 16; o; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0 && (cnt || mx >= 0)) {
    atomicAdd(reinterpret_cast<unsigned long long*>(stats), (unsigned long long)cnt);
    atomicMax(stats + 1, mx);
  }
}

inline unsigned blocks_for(long long n, int nt) { return (unsigned)((n + nt - 1) / nt); }

}  // namespace

int narrow_indices(const int64_t* src, int32_t* dst, int F, long long rows, int width,
                   const int64_t* n_rows, long long src_fs, long long dst_fs, cudaStream_t st) {
  if (F < 1 || rows < 0 || width < 1 || !src || !dst)
    return fail(ERR_INVALID, "narrow_indices: bad arguments");
  if (rows == 0) return OK;
  const long long n = rows * width;
  dim3 grid((unsigned)std::min<long long>(blocks_for((n + 1) / 2, 256), 148 * 8), F);
  narrow_indices_kernel<<<grid, 256, 0, st>>>(src, dst, rows, width, n_rows, src_fs, dst_fs);
  return check_launch("narrow_indices_kernel");
}

int trimap_stats(const int64_t* trimap, long long n, long long* stats, cudaStream_t st) {
  if (n < 0 || !stats || (n > 0 && !trimap)) return fail(ERR_INVALID, "trimap_stats: bad arguments");
  if (cudaMemsetAsync(stats, 0, sizeof(long long), st) != cudaSuccess ||
      cudaMemsetAsync(stats + 1, 0xFF, sizeof(long long), st) != cudaSuccess)  // {0, -1}
    return check_launch("trimap_stats (init)");
  if (n == 0) return OK;
  const unsigned blocks = (unsigned)std::min<long long>(blocks_for((n + 1) / 2, 256), 148 * 4);
  trimap_stats_kernel<<<blocks, 256, 0, st>>>(trimap, n, stats);
  return check_launch("trimap_stats_kernel");
}

int stage_in(const void* src, bool f64, long long rs, long long fs, int F, int M, int N,
             float* dst, int pitch, uint32_t* vmask, cudaStream_t st) {
  if (F < 1 || M < 1 || N < 1 || !src) return fail(ERR_INVALID, "stage_in: bad shape");
  if (dst && (pitch < 3 * N || pitch % 4)) return fail(ERR_INVALID, "stage_in: bad pitch");
  const int wpr = (N + 31) / 32;
  dim3 block(32, 8);
  dim3 grid(wpr, (M + 7) / 8, F);
  if (f64)
    stage_in_kernel<double><<<grid, block, 0, st>>>(static_cast<const double*>(src), rs, fs, dst,
                                                    pitch, vmask, wpr, M, N);
  else
    stage_in_kernel<float><<<grid, block, 0, st>>>(static_cast<const float*>(src), rs, fs, dst,
                                                   pitch, vmask, wpr, M, N);
  return check_launch("stage_in_kernel");
}

int fc_data(const void* opc, bool f64, int M, int N, void* cen, void* nrm, cudaStream_t st) {
  if (M < 2 || N < 2) return fail(ERR_INVALID, "organized cloud must be at least 2 x 2");
  const long long Q = (long long)(M - 1) * (N - 1);
  if (f64 && reinterpret_cast<uintptr_t>(cen) % 16 == 0 && reinterpret_cast<uintptr_t>(nrm) % 16 == 0)
    return fc_data_f64(static_cast<const double*>(opc), 1, M, N, static_cast<double*>(cen),
                       static_cast<double*>(nrm), st);  // the row-segment kernel, same bits
  if (f64)
    fc_data_kernel<double><<<blocks_for(Q, 256), 256, 0, st>>>(
        static_cast<const double*>(opc), M, N, static_cast<double*>(cen), static_cast<double*>(nrm));
  else
    fc_data_kernel<float><<<blocks_for(Q, 256), 256, 0, st>>>(
        static_cast<const float*>(opc), M, N, static_cast<float*>(cen), static_cast<float*>(nrm));
  return check_launch("fc_data_kernel");
}

int triangle_normals(const void* pts, bool f64, const int64_t* tris, long long T, void* out,
                     cudaStream_t st) {
  if (T <= 0) return OK;
  if (f64)
    tri_normals_kernel<double><<<blocks_for(T, 256), 256, 0, st>>>(
        static_cast<const double*>(pts), tris, T, static_cast<double*>(out));
  else
    tri_normals_kernel<float><<<blocks_for(T, 256), 256, 0, st>>>(
        static_cast<const float*>(pts), tris, T, static_cast<float*>(out));
  return check_launch("tri_normals_kernel");
}

int group_assignment(const void* normals, bool f64, long long T, int F, const int64_t* n_tri,
                     const double* dominant, int G, double ang_min, const uint8_t* lflag,
                     uint8_t* labels, cudaStream_t st) {
  if (G < 1 || G > 254) return fail(ERR_INVALID, "need 1..254 dominant normals");
  if (T <= 0 || F < 1) return OK;
  dim3 grid(blocks_for(T, 256), F);
  if (f64)
    group_assign_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(normals), T, F,
                                                       n_tri, dominant, G, ang_min, lflag, labels);
  else
    group_assign_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(normals), T, F,
                                                      n_tri, dominant, G, ang_min, lflag, labels);
  return check_launch("group_assign_kernel");
}

int max_edge_mask(const void* pts, bool f64, const int64_t* tris, long long T, double l_max,
                  uint8_t* flag, cudaStream_t st) {
  if (T <= 0) return OK;
  const double thr = sq_threshold(l_max);
  if (f64)
    max_edge_kernel<double><<<blocks_for(T, 256), 256, 0, st>>>(static_cast<const double*>(pts),
                                                                tris, T, thr, flag);
  else
    max_edge_kernel<float><<<blocks_for(T, 256), 256, 0, st>>>(static_cast<const float*>(pts),
                                                               tris, T, thr, flag);
  return check_launch("max_edge_kernel");
}

int unstage(const float* src, int pitch, int F, int M, int N, void* dst, bool f64,
            const void* orig, cudaStream_t st) {
  if (F < 1 || M < 1 || N < 1 || pitch < 3 * N) return fail(ERR_INVALID, "unstage: bad shape");
  const long long n = (long long)M * N * 3;
  dim3 grid((unsigned)std::min<long long>((n + 255) / 256, 148 * 16), F);
  if (f64)
    unstage_kernel<double><<<grid, 256, 0, st>>>(src, pitch, M, N, static_cast<double*>(dst),
                                                 static_cast<const double*>(orig));
  else
    unstage_kernel<float><<<grid, 256, 0, st>>>(src, pitch, M, N, static_cast<float*>(dst),
                                                static_cast<const float*>(orig));
  return check_launch("unstage_kernel");
}

}  // namespace opcfe
