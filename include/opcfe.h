/*
 * opcfe.h -- C ABI of libopcfe, the B200 (sm_100a) organized-point-cloud front-end.
 *
 * Drop-in boundary for the reference's hot path (flatpoly, arXiv 2007.12065 clean-room
 * reimplementation).  Every entry point names the reference interface it replaces;
 * paths are relative to /root/reference/pkg/src/flatpoly.  The reference's own plugin
 * point is the `_kernels` backend switch (_kernels/__init__.py:9-30); see
 * INTEGRATION.md for the ctypes binding a maintainer adds there.
 *
 * Conventions
 *   - All pointers are DEVICE pointers (cudaMalloc / torch CUDA tensors) unless noted.
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy stream),
 *     never allocates, never synchronises, and is safe to capture into a CUDA graph.
 *   - Return value: OPCFE_OK (0) or a negative OPCFE_ERR_*; the message is in
 *     opcfe_last_error() (thread-local).  No exception crosses the ABI.
 *   - Organized grids: F frames of M x N points, xyz interleaved, float32, each row
 *     padded to `pitch` floats (pitch >= 3N, pitch % 4 == 0: the TMA row-stride rule);
 *     frame stride = M * pitch.  opcfe_points_pitch(N) gives the minimal pitch.
 *   - FC (fully-connected triangle) grids: (M-1) x (N-1) quads x 2 triangles x xyz,
 *     rows padded to opcfe_fc_pitch(N) floats.
 *   - GID = 2*(u*(N-1)+v)+k (mesh.py:46-48).  Per-frame capacity G = 2(M-1)(N-1):
 *     frame f's triangles/twins/normals start at row f*G of their arrays.
 */
#ifndef OPCFE_H_
#define OPCFE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* opcfe_stream_t; /* cudaStream_t */

#define OPCFE_OK 0
#define OPCFE_ERR_INVALID (-1)     /* shape / parameter (reference: DegenerateInputError, ValueError) */
#define OPCFE_ERR_CUDA (-2)        /* CUDA runtime or launch failure */
#define OPCFE_ERR_UNSUPPORTED (-3) /* kernel_size beyond the compiled set */
#define OPCFE_ERR_WORKSPACE (-4)   /* workspace smaller than opcfe_*_workspace() */
#define OPCFE_ERR_DRIVER (-5)      /* cuTensorMapEncodeTiled unavailable */

int opcfe_version(void);
const char* opcfe_last_error(void);

/* layout helpers */
int opcfe_points_pitch(int N);
int opcfe_fc_pitch(int N);
size_t opcfe_vmask_words(int F, int M, int N); /* 1 validity bit per point, ceil(N/32) words/row */
size_t opcfe_triangulate_workspace(int F, int M, int N); /* row prefixes: F x M int64 */

/* Source grid (any f32/f64 layout with xyz contiguous) -> padded fp32 grid + validity bits.
 * Replaces the dtype coercion np.asarray(opc, dtype=float64) at smoothing.py:55 / mesh.py:65
 * and the finiteness mask at mesh.py:69.  dst may be NULL (mask only).  Strides in elements. */
int opcfe_stage_in(const void* src, int src_is_f64, long long src_row_stride,
                   long long src_frame_stride, int F, int M, int N, float* dst, int pitch,
                   uint32_t* vmask, opcfe_stream_t stream);

/* Inverse of opcfe_stage_in: padded fp32 grid -> contiguous (F,M,N,3) f32 or f64.  With
 * orig != NULL (the caller's original input, dst dtype), every component whose fp32
 * value equals float(orig) is returned as orig bit-exactly, so vertices/normals the
 * filters leave unchanged come back exactly as given (smoothing.py:57; border ring
 * and NaN vertices, _fallback.py:111-115). */
int opcfe_unstage(const float* src, int pitch, int F, int M, int N, void* dst, int dst_is_f64,
                  const void* orig, opcfe_stream_t stream);

/* Replaces _kernels.laplacian_filter(points, lam, kernel_size, iterations)
 * (_kernels/__init__.py:29 -> _native.pyx:225 / _fallback.py:82) as called by
 * smoothing.laplacian_filter_opc (smoothing.py:53-58).  Result in `out`; `tmp` is the
 * ping-pong buffer (same size, needed when iterations > 1).  If vmask != NULL the
 * first pass also writes the point-validity bits of `in`.  `in` must not alias `out` or
 * `tmp`: with kernel_size 3 and iterations > 1 the last pass re-reads it to return
 * partial-NaN vertices exactly as given. */
int opcfe_laplacian(const float* in, float* out, float* tmp, uint32_t* vmask, int F, int M,
                    int N, int pitch, float lam, int kernel_size, int iterations,
                    opcfe_stream_t stream);

/* Replaces mesh.extract_triangles_opc (mesh.py:58-96) + mesh.extract_halfedges_opc
 * (mesh.py:99-135), and optionally compute_normals (mesh.py:162 -> geometry.py:134, fp64
 * math on the fp32 grid) and the l_max longest-edge flag of group_assignment
 * (segmentation.py:59-67,73).  trimap [F][G], triangles [F][G][3], halfedges [F][G][3]
 * (nullable), n_tri [F]; normals [F][G][3] and lmax_flag [F][G] are optional (NULL);
 * pts/pitch are needed only for them.  ws: opcfe_triangulate_workspace() bytes. */
int opcfe_triangulate(const uint32_t* vmask, int F, int M, int N, int64_t* trimap,
                      int64_t* triangles, int64_t* halfedges, int64_t* n_tri, const float* pts,
                      int pitch, float* normals, double l_max, uint8_t* lmax_flag, void* ws,
                      size_t ws_bytes, opcfe_stream_t stream);

/* Replaces mesh.extract_halfedges_opc(trimap, M, N) for an arbitrary caller trimap
 * (mesh.py:99-135).  halfedges must be pre-filled with -1 (3*n_tri entries). */
int opcfe_halfedges_from_trimap(const int64_t* trimap, int M, int N, int64_t n_tri,
                                int64_t* halfedges, opcfe_stream_t stream);

/* Replaces smoothing.compute_fc_triangle_data (smoothing.py:61-88); contiguous (M,N,3) in,
 * (M-1,N-1,2,3) out, f64 (bit-exact) or f32. */
int opcfe_fc_data(const void* opc, int is_f64, int M, int N, void* centroids, void* normals,
                  opcfe_stream_t stream);

/* Replaces smoothing.bilateral_filter_opc (smoothing.py:91-114) -- FC data, the
 * _kernels.bilateral_iterate loop (_native.pyx:287 / _fallback.py:120) and the trimap
 * gather -- in `iterations` launches.  Three input forms:
 *   pts != NULL, normals_in == NULL: normals/centroids computed from the point grid
 *     (fused into iteration 1);
 *   pts != NULL, normals_in != NULL, centroids_in == NULL: continue filtering from the
 *     given FC normals (centroids from the grid): bilateral_iterate(.., k) followed by
 *     bilateral_iterate(.., m) equals bilateral_iterate(.., k + m) (_native.pyx:305);
 *   normals_in, centroids_in != NULL: FC arrays as given to _kernels.bilateral_iterate
 *     (_kernels/__init__.py:30): normals fp32 padded rows, centroids float64 contiguous
 *     [F][M-1][N-1][2][3] (differences to a per-tile origin are taken in fp64, so the
 *     centroid term keeps its precision far from the coordinate origin).
 * Output: out_mesh != NULL -> mesh order through trimap ([F][out_rows][3]);
 *         otherwise out_fc (FC layout, padded rows).
 * buf_a / buf_b: FC-sized ping-pong buffers (needed for iterations > 1 / > 2). */
int opcfe_bilateral(const float* pts, int F, int M, int N, int pitch, const float* normals_in,
                    const double* centroids_in, float sigma_length, float sigma_angle,
                    int kernel_size, int iterations, float* buf_a, float* buf_b, float* out_fc,
                    const int64_t* trimap, float* out_mesh, long long out_rows,
                    opcfe_stream_t stream);

/* Replaces geometry.triangle_normals (geometry.py:134-147) == mesh.compute_normals
 * (mesh.py:162-164) for any indexed set; contiguous (n,3) points, (T,3) int64 triangles.
 * f64 results are bit-identical to numpy. */
int opcfe_triangle_normals(const void* points, int is_f64, const int64_t* triangles,
                           long long n_tri, void* normals, opcfe_stream_t stream);

/* Replaces _kernels.find_cells (_kernels/__init__.py:27 -> _native.pyx:120 /
 * _fallback.py:14-44) and, with counts != NULL, the bincount of
 * accumulator.integrate_normals (accumulator.py:157-173).  queries: n rows taken every
 * `stride` rows of a contiguous (., 3) f64 array; the accumulator arrays are those of
 * GaussianAccumulator (s2ids uint64 [n_cells], normals [n_cells][3], neighbors int64
 * [n_cells][12]).  cells (nullable) [n] receives the cell index (-1 for skipped non-finite
 * rows in counting mode); counts (nullable) [n_cells] is incremented. */
int opcfe_find_cells(const double* queries, long long n, long long stride, const uint64_t* ids,
                     const double* cell_normals, const int64_t* neighbors, long long n_cells,
                     double slope, double intercept, long long window_lo, long long window_hi,
                     int64_t* cells, int64_t* counts, opcfe_stream_t stream);

/* Replaces segmentation.group_assignment (segmentation.py:52-74) on a mesh's normals:
 * labels[t] = argmax_g n_t . d_g (first max; fp64 FMA chain as numpy's BLAS matmul),
 * 255 unless the best score >= ang_min, 255 where lmax_flag[t] (nullable) is set.
 * F frames of T rows each; n_tri (device [F], nullable) bounds the live rows. */
int opcfe_group_assignment(const void* normals, int is_f64, long long T, int F,
                           const int64_t* n_tri, const double* dominant, int n_dominant,
                           double ang_min, const uint8_t* lmax_flag, uint8_t* labels,
                           opcfe_stream_t stream);

/* Replaces the l_max half of segmentation.group_assignment (segmentation.py:59-67,73):
 * flag[t] = longest edge of triangle t > l_max (fp64 edge lengths). */
int opcfe_max_edge_mask(const void* points, int is_f64, const int64_t* triangles,
                        long long n_tri, double l_max, uint8_t* flag, opcfe_stream_t stream);

/* Compact (NON-reference) index output: int64 index rows -> int32.  Frame f's first
 * n_rows[f] rows (all `rows` if n_rows == NULL) of `width` indices; strides in elements.
 * The caller guarantees every value fits (grids with M*N and 6(M-1)(N-1) below 2^31). */
int opcfe_narrow_indices(const int64_t* src, int32_t* dst, int F, long long rows, int width,
                         const int64_t* n_rows, long long src_frame_stride,
                         long long dst_frame_stride, opcfe_stream_t stream);

/* Row count and bound of a GID map, on the device: stats (device, 2 x int64) = {number of
 * entries >= 0, max(-1, largest entry)} of trimap[0..n).  Replaces the host pass
 * `valid = trimap >= 0; out = np.empty((int(valid.sum()), 3))` of bilateral_filter_opc
 * (smoothing.py:110-112); stats[1] >= stats[0] is the reference's IndexError
 * (`out[trimap[valid]] = ...` out of bounds).  Asynchronous on `stream`. */
int opcfe_trimap_stats(const int64_t* trimap, long long n, long long* stats,
                       opcfe_stream_t stream);

/* ---- strict precision: the reference's own fp64 arithmetic on its own layouts ----
 * Grids (F, M, N, 3) and FC arrays (F, M-1, N-1, 2, 3) are contiguous float64; any odd
 * kernel_size >= 3 (generic-window kernels).
 *
 * opcfe_laplacian_f64 replaces _kernels.laplacian_filter (_native.pyx:225-284,
 * _fallback.py:82-117) BIT-EXACTLY: IEEE mul / add / sqrt / div in the reference's
 * operation order (it is compiled with -ffp-contract=off, setup.py:24-26).  tmp: ping-pong
 * buffer (iterations > 1); `in` must alias neither. */
int opcfe_laplacian_f64(const double* in, double* out, double* tmp, int F, int M, int N,
                        double lam, int kernel_size, int iterations, opcfe_stream_t stream);

/* Precision "mixed" Laplacian (same contract as opcfe_laplacian_f64 -- replaces
 * _kernels.laplacian_filter, _native.pyx:225-284 -- but NOT bit-exact): float64 points in
 * and out, the reference's skip rules and update, the pair weight 1/dist as rsqrt(|d|^2)
 * (~1 ulp) instead of an IEEE sqrt and division, FMA-contracted sums.  Vertices within a
 * few ulp of the reference's (C4, 10 passes: 3.1e-16 relative, 67 % bit-identical).
 * k = 3 with an even N; other shapes run the strict kernels (exact). */
int opcfe_laplacian_mixed(const double* in, double* out, double* tmp, int F, int M, int N,
                          double lam, int kernel_size, int iterations, opcfe_stream_t stream);

/* compute_fc_triangle_data (smoothing.py:61-88) of F frames, bit-exact. */
int opcfe_fc_data_f64(const double* opc, int F, int M, int N, double* centroids, double* normals,
                      opcfe_stream_t stream);

/* Replaces _kernels.bilateral_iterate (_native.pyx:287-364, _fallback.py:120-166) on an
 * (M-1) x (N-1) FC grid, and with trimap != NULL also bilateral_filter_opc's gather
 * (smoothing.py:108-114: out_mesh[f][trimap[gid]] for trimap >= 0, out_rows rows per
 * frame); otherwise out_fc.  fp64 throughout; each iteration within a few ulp of the
 * reference's (FMA-contracted products, a pair-symmetric sum at kernel size 3, an own exp2;
 * the reference's two backends differ by ~1 ulp already).  buf_a / buf_b: FC-sized
 * ping-pong buffers (iterations > 1 / > 2). */
int opcfe_bilateral_f64(const double* centroids, const double* normals, int F, int M, int N,
                        double sigma_length, double sigma_angle, int kernel_size, int iterations,
                        double* buf_a, double* buf_b, double* out_fc, const int64_t* trimap,
                        double* out_mesh, long long out_rows, opcfe_stream_t stream);

/* Region growing over twin edges.  n_tri < 2^31.
 * opcfe_grow_segment replaces _kernels.grow_segment (_native.pyx:170-222): the connected
 * component of `seed` among triangles with groups == label, visited == 0 and (ptp_max > 0)
 * all vertices within ptp_max of the plane (anchor, normal) -- host double[3] each --
 * written SORTED to members (device [n_tri]); *n_members (device) = its size; members are
 * marked in visited.  opcfe_segment_components: for every triangle the minimum index of
 * its same-label twin-connected component (-1 where groups == 255) and, optionally, the
 * component size at its root: with ptp_max == 0 the segments of
 * segmentation.region_growing_task (segmentation.py:117-170) are exactly these
 * components (seed = root).  ws: opcfe_segments_workspace(n_tri) bytes. */
size_t opcfe_segments_workspace(long long n_tri);
int opcfe_grow_segment(const int64_t* triangles, const int64_t* halfedges, const double* points,
                       const uint8_t* groups, uint8_t* visited, long long n_tri, long long seed,
                       int label, const double* anchor, const double* normal, double ptp_max,
                       int64_t* members, int64_t* n_members, void* ws, size_t ws_bytes,
                       opcfe_stream_t stream);
int opcfe_segment_components(const int64_t* halfedges, const uint8_t* groups, long long n_tri,
                             int64_t* component, int64_t* size, void* ws, size_t ws_bytes,
                             opcfe_stream_t stream);

/* The organized branch of pipeline.run_scene (pipeline.py:125-134), all frames in one
 * call: [stage-in] -> Laplacian -> triangulation + twins -> bilateral (normals in mesh
 * order) [-> l_max flag]. */
typedef struct {
  int laplacian_iterations; /* 0 = no Laplacian */
  int laplacian_kernel_size;
  double laplacian_lambda;  /* double: the strict chain uses the caller's value as given */
  int bilateral_iterations; /* 0 = no bilateral: normals = triangle normals of the smoothed grid */
  int bilateral_kernel_size;
  double sigma_length;
  double sigma_angle;
  double l_max; /* < 0: no l_max flag */
  /* group_assignment (segmentation.py:52-74) fused after the normals: device f64
   * [n_dominant][3] dominant normals, or NULL for no labels */
  const double* dominant_normals;
  int n_dominant;
  double ang_min;
  /* OPCFE_PRECISION_FAST: fp32 kernels (+ the fp64 steps the 1e-5 contract needs);
   * OPCFE_PRECISION_STRICT: the reference's fp64 chain (points / normals outputs are
   * double: bit-exact Laplacian, FC data, topology; bilateral to <= a few ulp);
   * OPCFE_PRECISION_MIXED: the opcfe_laplacian_mixed Laplacian (double points within a
   * few ulp of the reference's), exact topology and FC data of those points, then
   * the fp32 bilateral on the FC arrays (normals double, within 1e-5
   * of the reference's chain end to end on well-conditioned frames -- the fast chain's
   * drift is fp32 vertex storage; at small sigma_angle fp32 normals alone can move the
   * reference's answer past 1e-5).
   * Fast-precision stages whose kernel size exceeds the fp32 kernels (Laplacian > 17,
   * bilateral > 9) run on the fp64 generic-window kernels, results rounded to fp32. */
  int precision;
} opcfe_front_end_params;

#define OPCFE_PRECISION_FAST 0
#define OPCFE_PRECISION_STRICT 1
#define OPCFE_PRECISION_MIXED 2

typedef struct {
  /* input: src_kind 0 = padded fp32 grid (src_pitch floats/row, frame stride M*src_pitch),
   *        1 = contiguous f32 (F,M,N,3), 2 = contiguous f64 (F,M,N,3) */
  const void* src;
  int src_kind;
  int src_pitch;
  /* outputs (device) */
  void* points;       /* fast: float [F][M][pitch], pitch = opcfe_points_pitch(N);
                         strict: double [F][M][N][3] */
  int64_t* trimap;    /* [F][G] */
  int64_t* triangles; /* [F][G][3] */
  int64_t* halfedges; /* [F][G][3] or NULL */
  void* normals;      /* [F][G][3] float (fast) / double (strict), or NULL */
  uint8_t* lmax_flag; /* [F][G] or NULL (needs l_max >= 0) */
  int64_t* n_tri;     /* [F] */
  uint8_t* labels;    /* [F][G] group labels (255 = unassigned) or NULL */
} opcfe_front_end_io;

size_t opcfe_front_end_workspace(int F, int M, int N, const opcfe_front_end_params* p,
                                 int src_kind, int src_pitch);
int opcfe_front_end(int F, int M, int N, const opcfe_front_end_params* p,
                    const opcfe_front_end_io* io, void* ws, size_t ws_bytes,
                    opcfe_stream_t stream);

/* opcfe_front_end with 5 optional cudaEvent_t (NULL entries skipped) recorded on `stream`
 * at the stage boundaries: [0] start, [1] after stage-in, [2] after the Laplacian,
 * [3] after triangulation, [4] after the bilateral filter (end) -- the analogue of the
 * reference's per-stage _Timer (pipeline.py:55-68, stages laplacian/front_end/bilateral). */
int opcfe_front_end_profiled(int F, int M, int N, const opcfe_front_end_params* p,
                             const opcfe_front_end_io* io, void* ws, size_t ws_bytes,
                             opcfe_stream_t stream, void* const* stage_events);

#ifdef __cplusplus
}
#endif

#endif /* OPCFE_H_ */
