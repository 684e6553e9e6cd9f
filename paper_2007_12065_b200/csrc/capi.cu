// C ABI of libopcfe (include/opcfe.h): argument checking, error plumbing, TMA
// descriptor encoding and the fused front-end chain.  No allocation, no host sync.
#include <cudaTypedefs.h>

#include <cstdio>
#include <mutex>
#include <string>

#include "../../include/opcfe.h"
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return fail(ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int make_tmap_3d(CUtensorMap* map, const void* base, bool f64, uint64_t cols, uint64_t rows,
                 uint64_t frames, uint64_t row_pitch_elems, uint64_t frame_stride_elems,
                 uint32_t box_cols, uint32_t box_rows, bool zero_fill) {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) return fail(ERR_DRIVER, "cuTensorMapEncodeTiled not available from the driver");
  const uint64_t esz = f64 ? 8 : 4;
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return fail(ERR_INVALID, "TMA: base address must be 16-byte aligned");
  if ((row_pitch_elems * esz) % 16 != 0 || (frame_stride_elems * esz) % 16 != 0)
    return fail(ERR_INVALID, "TMA: row/frame strides must be multiples of 16 bytes");
  cuuint64_t dims[3] = {cols, rows, frames};
  cuuint64_t strides[2] = {row_pitch_elems * esz, frame_stride_elems * esz};
  cuuint32_t box[3] = {box_cols, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = g_encode(
      map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
      const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      zero_fill ? CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE : CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA);
  if (r != CUDA_SUCCESS) {
    char buf[160];
    snprintf(buf, sizeof buf, "cuTensorMapEncodeTiled failed (%d): dims %llu x %llu x %llu box %u x %u",
             (int)r, (unsigned long long)cols, (unsigned long long)rows,
             (unsigned long long)frames, box_cols, box_rows);
    return fail(ERR_DRIVER, buf);
  }
  return OK;
}

namespace {

inline cudaStream_t S(opcfe_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct FeLayout {
  size_t vmask = 0, status = 0, staged = 0, lap_tmp = 0, bil_a = 0, bil_b = 0, bil_c = 0,
         total = 0;
  size_t vmask_b = 0, status_b = 0, staged_b = 0, lap_b = 0, bil_b_bytes = 0;
  // fp64 stages (strict precision, or kernel sizes beyond the fp32 kernels); mixed: the
  // strict stages up to the FC data, then the fp32 bilateral on the FC arrays
  bool strict = false, mixed = false, lap64 = false, bil64 = false, bil_mixed = false;
  size_t g64_in = 0, g64_tmp = 0, g64_out = 0, fc_c = 0, fc_n = 0, fc_a = 0, fc_b = 0;
  size_t fc32 = 0;
};

FeLayout fe_layout(int F, int M, int N, const opcfe_front_end_params* p, int src_kind,
                   int src_pitch) {
  FeLayout L;
  const int pitch = points_pitch(N);
  const size_t grid_bytes = (size_t)F * M * pitch * sizeof(float);
  const size_t fc_bytes = (size_t)F * (M - 1) * fc_pitch(N) * sizeof(float);
  const size_t g64 = (size_t)F * M * N * 3 * sizeof(double);
  const size_t fc64 = (size_t)F * (M - 1) * (N - 1) * 6 * sizeof(double);
  const bool lap = p->laplacian_iterations > 0;
  const bool bil = p->bilateral_iterations > 0;
  L.strict = p->precision == OPCFE_PRECISION_STRICT;
  L.mixed = p->precision == OPCFE_PRECISION_MIXED;
  const bool f64_grid = L.strict || L.mixed;  // the smoothed grid (points output) is double
  L.lap64 = lap && (f64_grid || p->laplacian_kernel_size > kLapMaxK32);
  L.bil64 = bil && (L.strict || p->bilateral_kernel_size > kBilMaxK32);
  L.bil_mixed = bil && L.mixed && !L.bil64;
  L.vmask_b = (size_t)F * M * ((N + 31) / 32) * sizeof(uint32_t);
  L.status_b = triangulate_workspace_bytes(F, M);
  const bool need_stage = lap && !L.lap64 && !(src_kind == 0 && src_pitch == pitch);
  L.staged_b = need_stage ? grid_bytes : 0;
  L.lap_b = (lap && !L.lap64 && p->laplacian_iterations > 1) ? grid_bytes : 0;
  L.bil_b_bytes = fc_bytes;
  const bool bil32 = bil && !L.bil64;
  const bool packed_bil = bil32;  // the fused pipeline's packed windows (fast and mixed)
  size_t off = 0;
  auto take = [&](size_t& at, size_t bytes) {
    at = off;
    off += align256(bytes);
  };
  take(L.vmask, L.vmask_b);
  take(L.status, L.status_b);
  take(L.staged, L.staged_b);
  take(L.lap_tmp, L.lap_b);
  take(L.bil_a, (bil32 && p->bilateral_iterations > 1) ? fc_bytes : 0);
  take(L.bil_b, (bil32 && p->bilateral_iterations > 2) ? fc_bytes : 0);
  // packed centroid planes + tile origins of the fused bilateral (>= 2 it.)
  take(L.bil_c, (packed_bil && p->bilateral_iterations > 1)
                    ? bilateral_buf_c_bytes(F, M, N, p->bilateral_kernel_size)
                    : 0);
  // fp64 grids: the source as f64 (unless it is f64 already), the Laplacian ping-pong,
  // and (fast precision) the f64 smoothed grid the fp64 stages read
  take(L.g64_in, ((f64_grid || L.lap64) && src_kind != 2) ? g64 : 0);
  take(L.g64_tmp, (L.lap64 && p->laplacian_iterations > 1) ? g64 : 0);
  take(L.g64_out, (!f64_grid && (L.lap64 || L.bil64)) ? g64 : 0);
  // mixed FC arrays: only when iteration 1 cannot compute the FC data itself (odd N, B = 1)
  const bool fc_arrays = L.bil_mixed && !bilateral_fc_in_iteration1(N, p->bilateral_iterations);
  take(L.fc_c, (L.bil64 || fc_arrays) ? fc64 : 0);
  take(L.fc_n, L.bil64 ? fc64 : 0);
  take(L.fc32, fc_arrays ? fc_bytes : 0);

  take(L.fc_a, (L.bil64 && p->bilateral_iterations > 1) ? fc64 : 0);
  take(L.fc_b, (L.bil64 && p->bilateral_iterations > 2) ? fc64 : 0);
  L.total = off + 256;
  return L;
}

}  // namespace
}  // namespace opcfe

using namespace opcfe;

extern "C" {

int opcfe_version(void) { return 1; }

const char* opcfe_last_error(void) { return g_last_error.c_str(); }

int opcfe_points_pitch(int N) { return points_pitch(N); }

int opcfe_fc_pitch(int N) { return fc_pitch(N); }

size_t opcfe_vmask_words(int F, int M, int N) { return (size_t)F * M * ((N + 31) / 32); }

size_t opcfe_triangulate_workspace(int F, int M, int N) {
  (void)N;
  return triangulate_workspace_bytes(F, M);
}

int opcfe_stage_in(const void* src, int src_is_f64, long long src_row_stride,
                   long long src_frame_stride, int F, int M, int N, float* dst, int pitch,
                   uint32_t* vmask, opcfe_stream_t stream) {
  return stage_in(src, src_is_f64 != 0, src_row_stride, src_frame_stride, F, M, N, dst, pitch,
                  vmask, S(stream));
}

int opcfe_unstage(const float* src, int pitch, int F, int M, int N, void* dst, int dst_is_f64,
                  const void* orig, opcfe_stream_t stream) {
  return unstage(src, pitch, F, M, N, dst, dst_is_f64 != 0, orig, S(stream));
}

int opcfe_laplacian(const float* in, float* out, float* tmp, uint32_t* vmask, int F, int M,
                    int N, int pitch, float lam, int kernel_size, int iterations,
                    opcfe_stream_t stream) {
  if (!in || !out) return fail(ERR_INVALID, "laplacian: null buffer");
  return laplacian(in, out, tmp, vmask, F, M, N, pitch, lam, kernel_size, iterations, S(stream));
}

int opcfe_triangulate(const uint32_t* vmask, int F, int M, int N, int64_t* trimap,
                      int64_t* triangles, int64_t* halfedges, int64_t* n_tri, const float* pts,
                      int pitch, float* normals, double l_max, uint8_t* lmax_flag, void* ws,
                      size_t ws_bytes, opcfe_stream_t stream) {
  return triangulate(vmask, F, M, N, trimap, triangles, halfedges, n_tri, pts, pitch, normals,
                     l_max, lmax_flag, ws, ws_bytes, S(stream));
}

int opcfe_halfedges_from_trimap(const int64_t* trimap, int M, int N, int64_t n_tri,
                                int64_t* halfedges, opcfe_stream_t stream) {
  return halfedges_from_trimap(trimap, M, N, n_tri, halfedges, S(stream));
}

int opcfe_fc_data(const void* opc, int is_f64, int M, int N, void* centroids, void* normals,
                  opcfe_stream_t stream) {
  return fc_data(opc, is_f64 != 0, M, N, centroids, normals, S(stream));
}

int opcfe_bilateral(const float* pts, int F, int M, int N, int pitch, const float* normals_in,
                    const double* centroids_in, float sigma_length, float sigma_angle,
                    int kernel_size, int iterations, float* buf_a, float* buf_b, float* out_fc,
                    const int64_t* trimap, float* out_mesh, long long out_rows,
                    opcfe_stream_t stream) {
  return bilateral(pts, F, M, N, pitch, normals_in, centroids_in, sigma_length, sigma_angle,
                   kernel_size, iterations, buf_a, buf_b, out_fc, trimap, out_mesh, out_rows,
                   S(stream));
}

int opcfe_triangle_normals(const void* points, int is_f64, const int64_t* triangles,
                           long long n_tri, void* normals, opcfe_stream_t stream) {
  return triangle_normals(points, is_f64 != 0, triangles, n_tri, normals, S(stream));
}

int opcfe_find_cells(const double* queries, long long n, long long stride, const uint64_t* ids,
                     const double* cell_normals, const int64_t* neighbors, long long n_cells,
                     double slope, double intercept, long long window_lo, long long window_hi,
                     int64_t* cells, int64_t* counts, opcfe_stream_t stream) {
  if (!queries) return fail(ERR_INVALID, "find_cells: null queries");
  return find_cells(queries, n, stride, ids, cell_normals, neighbors, n_cells, slope, intercept,
                    window_lo, window_hi, cells, counts, S(stream));
}

int opcfe_group_assignment(const void* normals, int is_f64, long long T, int F,
                           const int64_t* n_tri, const double* dominant, int n_dominant,
                           double ang_min, const uint8_t* lmax_flag, uint8_t* labels,
                           opcfe_stream_t stream) {
  if (!normals || !dominant || !labels) return fail(ERR_INVALID, "group_assignment: null buffer");
  return group_assignment(normals, is_f64 != 0, T, F, n_tri, dominant, n_dominant, ang_min,
                          lmax_flag, labels, S(stream));
}

int opcfe_max_edge_mask(const void* points, int is_f64, const int64_t* triangles,
                        long long n_tri, double l_max, uint8_t* flag, opcfe_stream_t stream) {
  return max_edge_mask(points, is_f64 != 0, triangles, n_tri, l_max, flag, S(stream));
}

size_t opcfe_segments_workspace(long long n_tri) {
  return n_tri < 1 ? 0 : segments_workspace_bytes(n_tri);
}

int opcfe_grow_segment(const int64_t* triangles, const int64_t* halfedges, const double* points,
                       const uint8_t* groups, uint8_t* visited, long long n_tri, long long seed,
                       int label, const double* anchor, const double* normal, double ptp_max,
                       int64_t* members, int64_t* n_members, void* ws, size_t ws_bytes,
                       opcfe_stream_t stream) {
  return grow_segment(triangles, halfedges, points, groups, visited, n_tri, seed, label, anchor,
                      normal, ptp_max, members, n_members, ws, ws_bytes, S(stream));
}

int opcfe_segment_components(const int64_t* halfedges, const uint8_t* groups, long long n_tri,
                             int64_t* component, int64_t* size, void* ws, size_t ws_bytes,
                             opcfe_stream_t stream) {
  return segment_components(halfedges, groups, n_tri, component, size, ws, ws_bytes, S(stream));
}

int opcfe_narrow_indices(const int64_t* src, int32_t* dst, int F, long long rows, int width,
                         const int64_t* n_rows, long long src_frame_stride,
                         long long dst_frame_stride, opcfe_stream_t stream) {
  return narrow_indices(src, dst, F, rows, width, n_rows, src_frame_stride, dst_frame_stride,
                        S(stream));
}

int opcfe_trimap_stats(const int64_t* trimap, long long n, long long* stats,
                       opcfe_stream_t stream) {
  return trimap_stats(trimap, n, stats, S(stream));
}

int opcfe_laplacian_mixed(const double* in, double* out, double* tmp, int F, int M, int N,
                          double lam, int kernel_size, int iterations, opcfe_stream_t stream) {
  return laplacian_mixed(in, out, tmp, F, M, N, lam, kernel_size, iterations, S(stream));
}

int opcfe_laplacian_f64(const double* in, double* out, double* tmp, int F, int M, int N,
                        double lam, int kernel_size, int iterations, opcfe_stream_t stream) {
  return laplacian_f64(in, out, tmp, F, M, N, lam, kernel_size, iterations, S(stream));
}

int opcfe_fc_data_f64(const double* opc, int F, int M, int N, double* centroids, double* normals,
                      opcfe_stream_t stream) {
  if (!opc || !centroids || !normals) return fail(ERR_INVALID, "fc_data_f64: null buffer");
  return fc_data_f64(opc, F, M, N, centroids, normals, S(stream));
}

int opcfe_bilateral_f64(const double* centroids, const double* normals, int F, int M, int N,
                        double sigma_length, double sigma_angle, int kernel_size, int iterations,
                        double* buf_a, double* buf_b, double* out_fc, const int64_t* trimap,
                        double* out_mesh, long long out_rows, opcfe_stream_t stream) {
  if (M < 2 || N < 2) return fail(ERR_INVALID, "organized cloud must be at least 2 x 2");
  return bilateral_f64(centroids, normals, F, M - 1, N - 1, sigma_length, sigma_angle,
                       kernel_size, iterations, buf_a, buf_b, out_fc, trimap, out_mesh, false,
                       out_rows, S(stream));
}

size_t opcfe_front_end_workspace(int F, int M, int N, const opcfe_front_end_params* p,
                                 int src_kind, int src_pitch) {
  if (!p || F < 1 || M < 2 || N < 2) return 0;
  return fe_layout(F, M, N, p, src_kind, src_pitch).total;
}

}  // extern "C"

namespace {

inline void mark(void* const* ev, int i, cudaStream_t st) {
  if (ev && ev[i]) cudaEventRecord(reinterpret_cast<cudaEvent_t>(ev[i]), st);
}

// ev (optional): 5 cudaEvent_t recorded at stage boundaries
//   [0] start  [1] after stage-in  [2] after Laplacian  [3] after triangulation  [4] end
//
// Precision: OPCFE_PRECISION_FAST runs the fp32 kernels (fp64 where the contract needs it);
// OPCFE_PRECISION_STRICT runs the reference's own fp64 arithmetic end to end (points and
// normals outputs are then double).  A fast-precision stage whose kernel size is beyond the
// fp32 kernels' compiled set runs on the fp64 generic-window kernels (results converted).
int front_end_impl(int F, int M, int N, const opcfe_front_end_params* p,
                   const opcfe_front_end_io* io, void* ws, size_t ws_bytes,
                   opcfe_stream_t stream, void* const* ev) {
  if (!p || !io || F < 1 || M < 2 || N < 2)
    return fail(ERR_INVALID, "front_end: organized cloud must be at least 2 x 2");
  if (!io->src || !io->points || !io->trimap || !io->triangles || !io->n_tri)
    return fail(ERR_INVALID, "front_end: null input/output");
  if (io->src_kind < 0 || io->src_kind > 2) return fail(ERR_INVALID, "front_end: bad src_kind");
  if (io->src_kind == 0 && (io->src_pitch < 3 * N || io->src_pitch % 4))
    return fail(ERR_INVALID, "front_end: src_pitch must be >= 3N and a multiple of 4");
  if (io->lmax_flag && p->l_max < 0) return fail(ERR_INVALID, "front_end: lmax_flag needs l_max");
  if (p->precision != OPCFE_PRECISION_FAST && p->precision != OPCFE_PRECISION_STRICT &&
      p->precision != OPCFE_PRECISION_MIXED)
    return fail(ERR_INVALID, "front_end: bad precision");
  const int pitch = points_pitch(N);
  const FeLayout L = fe_layout(F, M, N, p, io->src_kind, io->src_pitch);
  if (!ws || ws_bytes < L.total) return fail(ERR_WORKSPACE, "front_end: workspace too small");
  char* base = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
  uint32_t* vmask = reinterpret_cast<uint32_t*>(base + L.vmask);
  void* status = base + L.status;
  float* staged = reinterpret_cast<float*>(base + L.staged);
  float* lap_tmp = reinterpret_cast<float*>(base + L.lap_tmp);
  float* bil_a = reinterpret_cast<float*>(base + L.bil_a);
  float* bil_b = reinterpret_cast<float*>(base + L.bil_b);
  float* bil_c = reinterpret_cast<float*>(base + L.bil_c);
  double* g64_in = reinterpret_cast<double*>(base + L.g64_in);
  double* g64_tmp = reinterpret_cast<double*>(base + L.g64_tmp);
  double* g64_out = reinterpret_cast<double*>(base + L.g64_out);
  const cudaStream_t st = S(stream);
  const bool f64 = io->src_kind == 2;
  const long long rs = io->src_kind == 0 ? io->src_pitch : 3ll * N;
  const long long fs = (long long)M * rs;
  const long long G = 2ll * (M - 1) * (N - 1);
  const bool lap = p->laplacian_iterations > 0;
  int rc;
  mark(ev, 0, st);
  const bool f64_grid = L.strict || L.mixed;  // points output (and the stages on it) double
  // the source as contiguous f64 (fp64 Laplacian input / strict points)
  const double* src64 = f64 ? static_cast<const double*>(io->src) : nullptr;
  // strict / mixed smoothing of an fp32 source: pass 1 reads the fp32 boxes itself
  const bool from32 = !f64 && f64_grid && lap &&
                      laplacian64_from32_ok(static_cast<const float*>(io->src), N, rs,
                                            p->laplacian_kernel_size);
  if (!f64 && (f64_grid || L.lap64) && !from32) {
    if ((rc = unstage(static_cast<const float*>(io->src), (int)rs, F, M, N, g64_in, true, nullptr,
                      st)))
      return rc;
    src64 = g64_in;
  }
  // 1. Laplacian (smoothing.laplacian_filter_opc, pipeline.py:127-129)
  // points64: the smoothed grid as f64 for the fp64 stages (strict: the output itself)
  double* points64 = f64_grid ? static_cast<double*>(io->points) : nullptr;
  if (f64_grid) {
    mark(ev, 1, st);
    // the first (TMA) pass also writes the validity bits (k = 3, even N)
    const bool mask_fused = lap && laplacian64_mask_fused(N, p->laplacian_kernel_size);
    uint32_t* lap_mask = mask_fused ? vmask : nullptr;
    if (from32) {
      if ((rc = laplacian64_from32(static_cast<const float*>(io->src), rs, fs, points64, g64_tmp,
                                   F, M, N, p->laplacian_lambda, p->laplacian_kernel_size,
                                   p->laplacian_iterations, L.mixed, st, lap_mask)))
        return rc;
    } else if (lap) {
      if ((rc = (L.mixed ? laplacian_mixed : laplacian_f64)(
               src64, points64, g64_tmp, F, M, N, p->laplacian_lambda, p->laplacian_kernel_size,
               p->laplacian_iterations, st, lap_mask)))
        return rc;
    } else if (src64 != points64) {
      const cudaError_t e = cudaMemcpyAsync(points64, src64, (size_t)F * M * N * 3 * sizeof(double),
                                            cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess)
        return fail(ERR_CUDA, std::string("front_end: copy: ") + cudaGetErrorString(e));
    }
    // validity bits of the smoothed grid (the NaN mask is iteration-invariant), unless the
    // first Laplacian pass wrote them
    if (!mask_fused &&
        (rc = stage_in(points64, true, 3ll * N, 3ll * N * M, F, M, N, nullptr, pitch, vmask, st)))
      return rc;
  } else if (L.lap64) {
    mark(ev, 1, st);
    if ((rc = laplacian_f64(src64, g64_out, g64_tmp, F, M, N, p->laplacian_lambda,
                            p->laplacian_kernel_size, p->laplacian_iterations, st)))
      return rc;
    points64 = g64_out;
    if ((rc = stage_in(g64_out, true, 3ll * N, 3ll * N * M, F, M, N,
                       static_cast<float*>(io->points), pitch, vmask, st)))
      return rc;
  } else if (lap) {
    const float* lin;
    uint32_t* lap_vmask;
    if (L.staged_b == 0) {
      lin = static_cast<const float*>(io->src);
      lap_vmask = vmask;
    } else {
      if ((rc = stage_in(io->src, f64, rs, fs, F, M, N, staged, pitch, vmask, st))) return rc;
      lin = staged;
      lap_vmask = nullptr;
    }
    mark(ev, 1, st);
    rc = laplacian(lin, static_cast<float*>(io->points), lap_tmp, lap_vmask, F, M, N, pitch,
                   (float)p->laplacian_lambda, p->laplacian_kernel_size, p->laplacian_iterations, st);
    if (rc) return rc;
  } else {
    if ((rc = stage_in(io->src, f64, rs, fs, F, M, N, static_cast<float*>(io->points), pitch,
                       vmask, st)))
      return rc;
    mark(ev, 1, st);
  }
  mark(ev, 2, st);
  // 2. mesh_from_opc (pipeline.py:130-131): triangles + trimap + twins [+ normals, flags]
  const bool bil = p->bilateral_iterations > 0 && io->normals != nullptr;
  const bool extras32 = !f64_grid;  // fp32 grid: normals / flags fused with the triangulation
  rc = triangulate(vmask, F, M, N, io->trimap, io->triangles, io->halfedges, io->n_tri,
                   extras32 ? static_cast<const float*>(io->points) : nullptr, pitch,
                   (extras32 && !bil) ? static_cast<float*>(io->normals) : nullptr, p->l_max,
                   extras32 ? io->lmax_flag : nullptr, status, L.status_b, st);
  if (rc) return rc;
  if (f64_grid && (io->lmax_flag || (!bil && io->normals))) {
    rc = tri_extras_f64(points64, F, M, N, io->triangles, io->n_tri, bil ? nullptr : io->normals,
                        false, p->l_max, io->lmax_flag, st);
    if (rc) return rc;
  }
  mark(ev, 3, st);
  // 3. bilateral_filter_opc (pipeline.py:132-134), scattered to mesh order via trimap
  if (bil && L.bil64) {
    if (!points64) {  // fast precision, fp32 grid: its exact f64 image
      if ((rc = unstage(static_cast<const float*>(io->points), pitch, F, M, N, g64_out, true,
                        nullptr, st)))
        return rc;
      points64 = g64_out;
    }
    double* fc_c = reinterpret_cast<double*>(base + L.fc_c);
    double* fc_n = reinterpret_cast<double*>(base + L.fc_n);
    if ((rc = fc_data_f64(points64, F, M, N, fc_c, fc_n, st))) return rc;
    rc = bilateral_f64(fc_c, fc_n, F, M - 1, N - 1, p->sigma_length,
                       p->sigma_angle, p->bilateral_kernel_size, p->bilateral_iterations,
                       reinterpret_cast<double*>(base + L.fc_a),
                       reinterpret_cast<double*>(base + L.fc_b), nullptr, io->trimap, io->normals,
                       !f64_grid, G, st);
    if (rc) return rc;
  } else if (bil && L.bil_mixed && bilateral_fc_in_iteration1(N, p->bilateral_iterations)) {
    // mixed, fused: the FC data computed inside iteration 1 from the f64 grid (the same
    // bits as fc_mixed + the FC-array iteration 1, without the FC arrays' round trip)
    rc = bilateral(nullptr, F, M, N, 0, nullptr, nullptr, (float)p->sigma_length,
                   (float)p->sigma_angle, p->bilateral_kernel_size, p->bilateral_iterations,
                   bil_a, p->bilateral_iterations > 2 ? bil_b : nullptr, nullptr, io->trimap,
                   nullptr, G, st, bil_c, static_cast<double*>(io->normals), points64);
    if (rc) return rc;
  } else if (bil && L.bil_mixed) {
    // mixed: the f64 centroids and fp32 FC normals of the smoothed grid, the fp32 filter on
    // them (FC-array form), the last iteration scattering float64 normals
    double* fc_c = reinterpret_cast<double*>(base + L.fc_c);
    float* fc32 = reinterpret_cast<float*>(base + L.fc32);
    if ((rc = fc_mixed(points64, F, M, N, fc_c, fc32, fc_pitch(N), st))) return rc;
    rc = bilateral(nullptr, F, M, N, 0, fc32, fc_c, (float)p->sigma_length,
                   (float)p->sigma_angle, p->bilateral_kernel_size, p->bilateral_iterations,
                   p->bilateral_iterations > 1 ? bil_a : nullptr,
                   p->bilateral_iterations > 2 ? bil_b : nullptr, nullptr, io->trimap, nullptr,
                   G, st, p->bilateral_iterations > 1 ? bil_c : nullptr,
                   static_cast<double*>(io->normals));
    if (rc) return rc;
  } else if (bil) {
    rc = bilateral(static_cast<const float*>(io->points), F, M, N, pitch, nullptr, nullptr,
                   (float)p->sigma_length, (float)p->sigma_angle, p->bilateral_kernel_size,
                   p->bilateral_iterations, p->bilateral_iterations > 1 ? bil_a : nullptr,
                   p->bilateral_iterations > 2 ? bil_b : nullptr, nullptr, io->trimap,
                   static_cast<float*>(io->normals), G, st,
                   p->bilateral_iterations > 1 ? bil_c : nullptr);
    if (rc) return rc;
  }
  // 4. group labels (segmentation.group_assignment) on the final normals
  if (p->dominant_normals && io->labels) {
    if (!io->normals) return fail(ERR_INVALID, "front_end: labels need normals");
    rc = group_assignment(io->normals, f64_grid, G, F, io->n_tri, p->dominant_normals,
                          p->n_dominant, p->ang_min, p->l_max >= 0 ? io->lmax_flag : nullptr,
                          io->labels, st);
    if (rc) return rc;
  }
  mark(ev, 4, st);
  return OK;
}

}  // namespace

extern "C" {

int opcfe_front_end(int F, int M, int N, const opcfe_front_end_params* p,
                    const opcfe_front_end_io* io, void* ws, size_t ws_bytes,
                    opcfe_stream_t stream) {
  return front_end_impl(F, M, N, p, io, ws, ws_bytes, stream, nullptr);
}

int opcfe_front_end_profiled(int F, int M, int N, const opcfe_front_end_params* p,
                             const opcfe_front_end_io* io, void* ws, size_t ws_bytes,
                             opcfe_stream_t stream, void* const* stage_events) {
  return front_end_impl(F, M, N, p, io, ws, ws_bytes, stream, stage_events);
}

}  // extern "C"
