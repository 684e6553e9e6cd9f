// Shared device/host helpers for libopcfe (sm_100a only).
//  * TMA (cp.async.bulk.tensor) tile loads/stores + mbarrier completion
//  * fp64 arithmetic without FMA contraction (numpy operation order)
//  * error plumbing for the C ABI
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cmath>
#include <string>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libopcfe is built for sm_100a (B200) only"
#endif

namespace opcfe {

// ----------------------------------------------------------------- errors (host)
enum Status : int {
  OK = 0,
  ERR_INVALID = -1,      // bad shape / parameter
  ERR_CUDA = -2,         // CUDA runtime / launch failure
  ERR_UNSUPPORTED = -3,  // kernel size beyond the compiled set
  ERR_WORKSPACE = -4,    // workspace too small
  ERR_DRIVER = -5,       // driver entry point (cuTensorMapEncodeTiled) unavailable
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);

// ------------------------------------------------------------ small host utils
inline int round_up(int x, int m) { return (x + m - 1) / m * m; }
inline int points_pitch(int N) { return round_up(3 * N, 4); }      // floats per grid row
inline int fc_pitch(int N) { return round_up(6 * (N - 1), 4); }    // floats per FC quad row

// The l_max test without square roots, bit-exact: IEEE sqrt is correctly rounded, hence
// monotone, so {s : fl(sqrt(s)) <= l} is an interval (-inf, t] and
//   fl(sqrt(s)) > l  <=>  s > t   for every s >= 0 (NaN s: false on both sides).
// t is found next to fl(l*l) by stepping one ulp at a time (at most a few steps).
inline double sq_threshold(double l) {
  if (std::isnan(l)) return l;                 // every comparison false
  if (l < 0.0) return -1.0;                    // every s >= 0 passes
  if (std::isinf(l)) return l;                 // nothing passes
  double t = l * l;
  while (std::sqrt(t) > l) t = std::nextafter(t, -INFINITY);
  for (double n = std::nextafter(t, INFINITY); std::sqrt(n) <= l; n = std::nextafter(t, INFINITY))
    t = n;
  return t;
}

// TMA descriptor for a 3-D fp32/fp64 tensor [F][rows][cols] with a row pitch
// (elements) and a frame stride (elements).  Out-of-bounds reads fill with NaN,
// which is exactly the reference's "off-grid neighbour is skipped" rule
// (_kernels/_fallback.py:94 pads with NaN).
// zero_fill: out-of-bounds reads return 0 instead of NaN (packed bilateral planes).
int make_tmap_3d(CUtensorMap* map, const void* base, bool f64, uint64_t cols, uint64_t rows,
                 uint64_t frames, uint64_t row_pitch_elems, uint64_t frame_stride_elems,
                 uint32_t box_cols, uint32_t box_rows, bool zero_fill = false);

// Opt a kernel into `smem` bytes of dynamic shared memory on the CURRENT device.  The
// attribute is per device context; `mask` (one per kernel) remembers the devices already
// done (ids >= 64 set it on every call).  Returns OK or the CUDA error via fail().
template <typename Kernel>
inline int ensure_smem_attr(Kernel kernel, int smem, std::atomic<unsigned long long>& mask) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(ERR_CUDA, std::string("cudaGetDevice: ") + cudaGetErrorString(e));
  const unsigned long long bit = dev < 64 ? (1ull << dev) : 0ull;
  if (bit && (mask.load(std::memory_order_acquire) & bit)) return OK;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess)
    return fail(ERR_CUDA, std::string("cudaFuncSetAttribute(MaxDynamicSharedMemorySize): ") +
                              cudaGetErrorString(e));
  if (bit) mask.fetch_or(bit, std::memory_order_acq_rel);
  return OK;
}

// ------------------------------------------------------------- device helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Dynamic shared memory carve-up for TMA kernels.  TMA tile destinations must be
// 128-B aligned in the shared window; the dynamic-smem base is only guaranteed 16-B
// aligned, so kernels request kSmemSlack extra bytes and align here.  The mbarrier
// lives in the slack, in front of the tiles (no static __shared__ in TMA kernels).
constexpr int kSmemSlack = 256;

__device__ __forceinline__ char* smem_aligned_base(char* raw, uint64_t** bar) {
  const uint32_t off = static_cast<uint32_t>(__cvta_generic_to_shared(raw));
  const uint32_t pad = (128u - (off + 16u) % 128u) % 128u + 16u;  // >= 16 B for the barrier
  char* base = raw + pad;
  *bar = reinterpret_cast<uint64_t*>(base - 8);
  return base;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  const uint32_t a = smem_u32(bar);
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(a), "r"(phase)
        : "memory");
  } while (!done);
}

// global -> shared tile (3-D box), completion counted on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global tile (3-D box); out-of-bounds elements are not written
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0,
                                             int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
      : "memory");
}

__device__ __forceinline__ void tma_store_commit_and_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void tma_store_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// all committed bulk stores of this thread have finished READING shared memory
__device__ __forceinline__ void tma_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

// plain arrive (release.cta): producer -> consumer hand-off of smem written by this thread
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// named barrier over `count` threads (ids 1..15; 0 is __syncthreads)
__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// make generic-proxy smem writes visible to the async (TMA) proxy
// 1-D bulk copies (16-B aligned addresses, sizes multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(dst)),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// 2^x as ONE MUFU.EX2 (.ftz: the non-ftz form adds range fix-ups around the MUFU).
// Flushing results below 2^-126 is harmless for the bilateral weights: a triangle
// whose weights are all that small has |acc| < 17 * 2^-126 < 1e-30 and is left
// unchanged by the reference too (_native.pyx:352-360).
// ---- packed fp32x2 (one b64 register pair = lanes (lo, hi)); .rn, denormals kept
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2(float lo, float hi) {
  f2_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float f2lo(f2_t r) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
  return lo;
}
__device__ __forceinline__ float f2hi(f2_t r) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(r));
  return hi;
}
__device__ __forceinline__ f2_t add2(f2_t a, f2_t b) {
  f2_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t sub2(f2_t a, f2_t b) {
  f2_t r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t mul2(f2_t a, f2_t b) {
  f2_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ f2_t fma2(f2_t a, f2_t b, f2_t c) {
  f2_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// broadcast scalar operand (ptxas encodes it as a .F32 operand of FADD2 / FFMA2)
__device__ __forceinline__ f2_t bc2(float x) { return f2(x, x); }

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 1/sqrt(x) and 1/x as single MUFU ops (~1 ulp); inputs below 2^-126 are out of range
// for the callers (squared distances of distinct vertices / weight sums >= 2^-126).
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// acquire/release for the decoupled look-back status words
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ---- float64 math in numpy's operation order: no FMA contraction allowed.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// unit normal of triangle (a, b, c) = cross(b-a, c-a)/|.|, NaN unless |.| > 0
// (geometry.py:134-147; numpy np.cross component order, norm sqrt((x^2+y^2)+z^2))
__device__ __forceinline__ void unit_normal_f64(double ax, double ay, double az, double bx,
                                                double by, double bz, double cx, double cy,
                                                double cz, double& nx, double& ny, double& nz) {
  const double e1x = dsub(bx, ax), e1y = dsub(by, ay), e1z = dsub(bz, az);
  const double e2x = dsub(cx, ax), e2y = dsub(cy, ay), e2z = dsub(cz, az);
  const double x = dsub(dmul(e1y, e2z), dmul(e1z, e2y));
  const double y = dsub(dmul(e1z, e2x), dmul(e1x, e2z));
  const double z = dsub(dmul(e1x, e2y), dmul(e1y, e2x));
  const double n = __dsqrt_rn(dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z)));
  if (n > 0.0) {
    nx = __ddiv_rn(x, n);
    ny = __ddiv_rn(y, n);
    nz = __ddiv_rn(z, n);
  } else {
    nx = ny = nz = __longlong_as_double(0x7ff8000000000000LL);
  }
}

// cross(b - a, c - a) * rsqrt(|.|^2) (~1.5 ulp), NaN unless |.|^2 > 0.  The cross
// product and its squared norm keep the reference's uncontracted operations, so the
// degenerate (NaN) set is exactly the reference's; only sqrt + 3 divisions become rsqrt.
__device__ __forceinline__ void fast_unit_normal_f64(const double* a, const double* b,
                                                     const double* c, double& nx, double& ny,
                                                     double& nz) {
  const double e1x = dsub(b[0], a[0]), e1y = dsub(b[1], a[1]), e1z = dsub(b[2], a[2]);
  const double e2x = dsub(c[0], a[0]), e2y = dsub(c[1], a[1]), e2z = dsub(c[2], a[2]);
  const double x = dsub(dmul(e1y, e2z), dmul(e1z, e2y));
  const double y = dsub(dmul(e1z, e2x), dmul(e1x, e2z));
  const double z = dsub(dmul(e1x, e2y), dmul(e1y, e2x));
  const double r2 = dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z));
  if (r2 > 0.0) {
    const double r = rsqrt(r2);
    nx = x * r;
    ny = y * r;
    nz = z * r;
  } else {
    nx = ny = nz = __longlong_as_double(0x7ff8000000000000LL);
  }
}

// the mixed FC data's centroid: ((a + b) + c) * (1/3) with an uncontracted product (the
// fused bilateral's mode 3 recomputes it bit for bit)
__device__ __forceinline__ double mixed_centroid(double a, double b, double c) {
  return __dmul_rn(dadd(dadd(a, b), c), 1.0 / 3.0);
}

// ((a+b)+c)/3.0 (smoothing.py:79)
__device__ __forceinline__ double centroid_f64(double a, double b, double c) {
  return __ddiv_rn(dadd(dadd(a, b), c), 3.0);
}

// squared edge length (dx^2 + dy^2) + dz^2 in numpy's order (the operand of
// np.linalg.norm's sqrt); compared against sq_threshold(l_max) instead of taking the root
__device__ __forceinline__ double edge_len2_f64(double px, double py, double pz, double qx,
                                                double qy, double qz) {
  const double dx = dsub(qx, px), dy = dsub(qy, py), dz = dsub(qz, pz);
  return dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
}

// np.maximum(|ab|, np.maximum(|bc|, |ca|)) > l_max (segmentation.py:59-67,73) from the
// squared lengths and thr = sq_threshold(l_max); a NaN edge makes the maximum NaN -> false
__device__ __forceinline__ bool longest_edge_exceeds(double sab, double sbc, double sca,
                                                     double thr) {
  return !(isnan(sab) || isnan(sbc) || isnan(sca)) && fmax(sab, fmax(sbc, sca)) > thr;
}

// A unit normal from an fp64 cross product with an fp32 normalisation (the bilateral
// input): MUFU rcp / rsqrt + one Newton step instead of IEEE divide / sqrt,
// |n - float32(reference)| ~ 1e-7.
// Degenerate (zero cross product), non-finite or out-of-range crosses give NaN normals: the
// test runs on the fp32-rounded components (a NaN component makes the Newton step NaN).
__device__ __forceinline__ void normalise_fast(double x, double y, double z, float* n) {
  const float fx = (float)x, fy = (float)y, fz = (float)z;
  const float m = fmaxf(fabsf(fx), fmaxf(fabsf(fy), fabsf(fz)));
  if (m > 0.f && m <= 3.402823466e38f) {
    // rescale into [1, 3] before squaring (tiny triangles: |x| ~ 1e-20); the scale cancels
    const float is = rcp_approx(m);
    const float gx = fx * is, gy = fy * is, gz = fz * is;
    const float l2 = gx * gx + gy * gy + gz * gz;
    float r = rsqrt_approx(l2);
    r = r * fmaf(-0.5f * l2, r * r, 1.5f);
    n[0] = gx * r;
    n[1] = gy * r;
    n[2] = gz * r;
  } else {
    n[0] = n[1] = n[2] = __int_as_float(0x7fc00000);
  }
}

__device__ __forceinline__ bool finite3f(float x, float y, float z) {
  return isfinite(x) && isfinite(y) && isfinite(z);
}

}  // namespace opcfe
