// Internal launcher declarations (C++ linkage); the C ABI in capi.cu forwards here.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace opcfe {

int stage_in(const void* src, bool f64, long long src_row_stride, long long src_frame_stride,
             int F, int M, int N, float* dst, int pitch, uint32_t* vmask, cudaStream_t st);

int unstage(const float* src, int pitch, int F, int M, int N, void* dst, bool f64,
            const void* orig, cudaStream_t st);

int laplacian(const float* in, float* out, float* tmp, uint32_t* vmask, int F, int M, int N,
              int pitch, float lam, int ksize, int iters, cudaStream_t st);

size_t triangulate_workspace_bytes(int F, int M);
int triangulate(const uint32_t* vmask, int F, int M, int N, int64_t* trimap, int64_t* tris,
                int64_t* he, int64_t* ntri, const float* pts, int pitch, float* normals,
                double l_max, uint8_t* lflag, void* ws, size_t ws_bytes, cudaStream_t st);
int halfedges_from_trimap(const int64_t* trimap, int M, int N, int64_t n_tri, int64_t* he,
                          cudaStream_t st);

// fused-pipeline bilateral scratch `buf_c`: one packed centroid window (tile + halo, relative
// to the tile's origin) per 32 x 8-quad tile
size_t centroid_window_bytes(int h);
size_t bilateral_buf_c_bytes(int F, int M, int N, int ksize);
int bilateral(const float* pts, int F, int M, int N, int pitch, const float* normals_in,
              const double* centroids_in, float sigma_length, float sigma_angle, int ksize,
              int iters, float* buf_a, float* buf_b, float* out_fc, const int64_t* trimap,
              float* out_mesh, long long out_rows, cudaStream_t st,
              float* buf_c = nullptr,  // fused pipeline: centroid windows (bilateral_buf_c_bytes)
              double* out_mesh64 = nullptr,  // float64 scatter destination instead
              const double* pts64 = nullptr);  // mixed: FC data from the f64 grid in iteration 1

// the mixed front end computes its FC data inside the fused iteration 1 (bilateral(...,
// pts64)): even N (16-B f64 rows) and >= 2 iterations
bool bilateral_fc_in_iteration1(int N, int iters);

int fc_data(const void* opc, bool f64, int M, int N, void* cen, void* nrm, cudaStream_t st);

int trimap_stats(const int64_t* trimap, long long n, long long* stats, cudaStream_t st);

int narrow_indices(const int64_t* src, int32_t* dst, int F, long long rows, int width,
                   const int64_t* n_rows, long long src_fs, long long dst_fs, cudaStream_t st);

// strict (fp64, reference operation order) kernels: strict.cu
// vmask (nullable): the first pass also writes the grid's validity bits when
// laplacian64_mask_fused(N, ksize) (k = 3, even N: the TMA kernels)
int laplacian_f64(const double* in, double* out, double* tmp, int F, int M, int N, double lam,
                  int ksize, int iters, cudaStream_t st, uint32_t* vmask = nullptr);
bool laplacian64_mask_fused(int N, int ksize);
// the strict / mixed Laplacian of an fp32 source (row stride rs, frame stride fs floats):
// pass 1 reads the fp32 boxes directly (exact widening), no conversion pass; k = 3, even N,
// 16-B source rows (laplacian64_from32_ok)
bool laplacian64_from32_ok(const float* in, int N, long long rs, int ksize);
int laplacian64_from32(const float* in, long long rs, long long fs, double* out, double* tmp,
                       int F, int M, int N, double lam, int ksize, int iters, bool mixed,
                       cudaStream_t st, uint32_t* vmask = nullptr);
// precision "mixed": rsqrt pair weights, FMA sums, f64 points (k = 3, even N;
// otherwise laplacian_f64)
int laplacian_mixed(const double* in, double* out, double* tmp, int F, int M, int N, double lam,
                    int ksize, int iters, cudaStream_t st, uint32_t* vmask = nullptr);
int bilateral_f64(const double* centroids, const double* normals_in, int F, int Mq, int Nq,
                  double sigma_length, double sigma_angle, int ksize, int iters, double* buf_a,
                  double* buf_b, double* out_fc, const int64_t* trimap, void* out_mesh,
                  bool out_f32, long long out_rows, cudaStream_t st);
int fc_data_f64(const double* opc, int F, int M, int N, double* cen, double* nrm, cudaStream_t st);
int fc_mixed(const double* opc, int F, int M, int N, double* cen, float* nrm32, int fcp,
             cudaStream_t st);
int tri_extras_f64(const double* pts, int F, int M, int N, const int64_t* tris,
                   const int64_t* n_tri, void* normals, bool normals_f32, double l_max,
                   uint8_t* flag, cudaStream_t st);
// largest kernel sizes of the fp32 kernels (beyond: the fp64 generic-window kernels)
constexpr int kLapMaxK32 = 17;
constexpr int kBilMaxK32 = 9;
int triangle_normals(const void* pts, bool f64, const int64_t* tris, long long T, void* out,
                     cudaStream_t st);
int find_cells(const double* queries, long long n, long long stride, const uint64_t* ids,
               const double* cell_normals, const int64_t* neighbors, long long n_cells,
               double slope, double intercept, long long window_lo, long long window_hi,
               int64_t* cells, int64_t* counts, cudaStream_t st);
int group_assignment(const void* normals, bool f64, long long T, int F, const int64_t* n_tri,
                     const double* dominant, int G, double ang_min, const uint8_t* lflag,
                     uint8_t* labels, cudaStream_t st);
int max_edge_mask(const void* pts, bool f64, const int64_t* tris, long long T, double l_max,
                  uint8_t* flag, cudaStream_t st);

size_t segments_workspace_bytes(long long n_tri);
int grow_segment(const int64_t* tris, const int64_t* he, const double* pts,
                 const uint8_t* groups, uint8_t* visited, long long n_tri, long long seed,
                 int label, const double* anchor, const double* normal, double ptp_max,
                 int64_t* members, int64_t* n_members, void* ws, size_t ws_bytes,
                 cudaStream_t st);
int segment_components(const int64_t* he, const uint8_t* groups, long long n_tri, int64_t* comp,
                       int64_t* size, void* ws, size_t ws_bytes, cudaStream_t st);

}  // namespace opcfe
