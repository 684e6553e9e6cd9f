// FastGA cell search and histogram integration (the stage after the
// front-end's normals, pipeline.py:150-157).
//
// Reference semantics:
//   * s2_id (sfc.py:46-104): normalise, dominant axis -> cube face (face chain -y,+x,+z,
//     -x,-z,+y), face coordinates u, v = n_u/|n_dom|, n_v/|n_dom|, tangent warp
//     atan(t)*4/pi, 30-bit quantisation, per-face swap / flip, Hilbert curve position;
//     id = face << 60 | d;
//   * find_cells (_kernels/_fallback.py:14-44 == _native.pyx:120-167): predicted index
//     rint(slope*id + intercept), window [k+lo, k+hi] clamped, nearest id inside the window
//     (searchsorted + clamp, ties to the lower), then argmin |cell_normal - q|^2 over that
//     cell and its <= 12 neighbours (first minimum);
//   * integrate_normals (accumulator.py:157-173): every round(1/sample_pct)-th normal,
//     non-finite rows skipped, counts += bincount(cells).
// One thread per query; fp64 throughout with numpy's operation order (no FMA).  The
// accumulator arrays (level 4: 5120 cells, ~650 KB) stay L2-resident.  CUDA's atan
// differs from glibc's in the last ulp on rare inputs, which can move a query across a
// 2^-30 quantisation boundary -- the same class of difference the reference's own two
// backends show (tests/test_kernels.py:19-33: >= 0.9999 agreement, flips within the 1-ring).
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

namespace {

constexpr int kHbOrder = 30;
constexpr long long kHbGrid = 1ll << kHbOrder;

__constant__ int c_face_u[6] = {0, 1, 0, 1, 0, 0};
__constant__ int c_face_v[6] = {2, 2, 1, 2, 1, 2};
__constant__ int c_face_swap[6] = {0, 1, 0, 1, 1, 0};
__constant__ int c_face_negu[6] = {0, 0, 1, 1, 0, 0};
__constant__ int c_face_of[6] = {1, 3, 5, 0, 2, 4};  // axis*2 + (sign < 0) -> face

__device__ __forceinline__ long long hb_quantize(double t) {
  const double a = dmul(atan(t), 4.0 / 3.141592653589793);
  const double f = floor(dmul(dmul(dadd(a, 1.0), 0.5), (double)kHbGrid));
  long long i = (long long)f;
  return i < 0 ? 0 : (i > kHbGrid - 1 ? kHbGrid - 1 : i);
}

__device__ __forceinline__ long long hb_d(long long x, long long y) {
  long long d = 0;
  for (long long s = kHbGrid >> 1; s > 0; s >>= 1) {
    const long long rx = (x & s) > 0, ry = (y & s) > 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = s - 1 - x;
        y = s - 1 - y;
      }
      const long long t = x;
      x = y;
      y = t;
    }
  }
  return d;
}

__device__ __forceinline__ unsigned long long s2_id(double x, double y, double z) {
  const double nrm = __dsqrt_rn(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z)));
  const double n[3] = {__ddiv_rn(x, nrm), __ddiv_rn(y, nrm), __ddiv_rn(z, nrm)};
  int ax = 0;
  if (fabs(n[1]) > fabs(n[ax])) ax = 1;
  if (fabs(n[2]) > fabs(n[ax])) ax = 2;
  const double dom = n[ax];
  const int face = c_face_of[ax * 2 + (dom < 0.0)];
  const double ad = fabs(dom);
  long long iu = hb_quantize(__ddiv_rn(n[c_face_u[face]], ad));
  long long iv = hb_quantize(__ddiv_rn(n[c_face_v[face]], ad));
  if (c_face_swap[face]) {
    const long long t = iu;
    iu = iv;
    iv = t;
  }
  if (c_face_negu[face]) iu = kHbGrid - 1 - iu;
  return ((unsigned long long)face << (2 * kHbOrder)) | (unsigned long long)hb_d(iu, iv);
}

struct GaArgs {
  const double* q;
  long long n;        // queries (after striding)
  long long stride;   // row stride between sampled queries
  const unsigned long long* ids;
  const double* cn;
  const long long* nbrs;
  long long ncell;
  double slope, icpt;
  long long wlo, whi;
  long long* cells;   // nullable
  unsigned long long* counts;  // nullable: histogram (skip non-finite rows)
};

__global__ void find_cells_kernel(GaArgs a) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const double* qi = a.q + 3 * i * a.stride;
  const double qx = qi[0], qy = qi[1], qz = qi[2];
  if (a.counts != nullptr && !(isfinite(qx) && isfinite(qy) && isfinite(qz))) {
    if (a.cells) a.cells[i] = -1;
    return;
  }
  const unsigned long long id = s2_id(qx, qy, qz);
  const long long kp = (long long)rint(dadd(dmul(a.slope, __ull2double_rn(id)), a.icpt));
  long long lo = kp + a.wlo, hi = kp + a.whi;
  lo = lo < 0 ? 0 : (lo > a.ncell - 1 ? a.ncell - 1 : lo);
  hi = hi < 0 ? 0 : (hi > a.ncell - 1 ? a.ncell - 1 : hi);
  // lower bound restricted to [lo, hi+1): equivalent after the clamps below
  long long b0 = lo, b1 = hi + 1;
  while (b0 < b1) {
    const long long m = (b0 + b1) >> 1;
    if (__ldg(a.ids + m) < id) b0 = m + 1;
    else b1 = m;
  }
  const long long ch = b0 < lo ? lo : (b0 > hi ? hi : b0);
  const long long cl = b0 - 1 < lo ? lo : (b0 - 1 > hi ? hi : b0 - 1);
  const unsigned long long ih = __ldg(a.ids + ch), il = __ldg(a.ids + cl);
  const unsigned long long dh = ih > id ? ih - id : id - ih;
  const unsigned long long dl = il > id ? il - id : id - il;
  const long long j = dl <= dh ? cl : ch;
  long long best = j;
  double bd = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  for (int k = -1; k < 12; ++k) {
    const long long c = k < 0 ? j : __ldg(a.nbrs + 12 * j + k);
    if (c < 0) continue;
    const double dx = dsub(__ldg(a.cn + 3 * c), qx), dy = dsub(__ldg(a.cn + 3 * c + 1), qy),
                 dz = dsub(__ldg(a.cn + 3 * c + 2), qz);
    const double d2 = dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
    if (d2 < bd) {
      bd = d2;
      best = c;
    }
  }
  if (a.cells) a.cells[i] = best;
  if (a.counts) atomicAdd(a.counts + best, 1ull);
}

}  // namespace

int find_cells(const double* queries, long long n, long long stride, const uint64_t* ids,
               const double* cell_normals, const int64_t* neighbors, long long n_cells,
               double slope, double intercept, long long window_lo, long long window_hi,
               int64_t* cells, int64_t* counts, cudaStream_t st) {
  if (n < 0 || stride < 1 || n_cells < 1 || !ids || !cell_normals || !neighbors)
    return fail(ERR_INVALID, "find_cells: bad accumulator or query arrays");
  if (n == 0) return OK;
  GaArgs a;
  a.q = queries;
  a.n = n;
  a.stride = stride;
  a.ids = reinterpret_cast<const unsigned long long*>(ids);
  a.cn = cell_normals;
  a.nbrs = reinterpret_cast<const long long*>(neighbors);
  a.ncell = n_cells;
  a.slope = slope;
  a.icpt = intercept;
  a.wlo = window_lo;
  a.whi = window_hi;
  a.cells = reinterpret_cast<long long*>(cells);
  a.counts = reinterpret_cast<unsigned long long*>(counts);
  find_cells_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(a);
  return check_launch("find_cells_kernel");
}

}  // namespace opcfe
