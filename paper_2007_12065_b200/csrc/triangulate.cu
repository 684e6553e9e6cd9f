// Implicit right-cut triangulation of the organized grid, in ONE pass.
//
// Reference semantics (flatpoly/mesh.py):
//   * quad (u,v): p1=(u,v) p2=(u,v+1) p3=(u+1,v+1) p4=(u+1,v) (mesh.py:73-80);
//     first {p3,p2,p1} valid iff p1&p2&p3 finite, second {p1,p4,p3} iff p1&p3&p4
//     (mesh.py:81-82, :88-94);
//   * GID = 2*(u*(N-1)+v)+k; trimap = where(ok, cumsum(ok)-1, -1) (mesh.py:85-86);
//     triangles emitted in GID order (mesh.py:95);
//   * twins (mesh.py:129-134): edge k links edge k of the neighbour
//       first  e0 -> (u,v+1,1)  e1 -> (u-1,v,1)  e2 -> (u,v,1)
//       second e0 -> (u,v-1,0)  e1 -> (u+1,v,0)  e2 -> (u,v,0)
//   * optional fused extras: mesh-order normals (geometry.py:134-147, fp64 math)
//     and the l_max longest-edge flag (segmentation.py:59-67,73, fp64 math).
//
// B200 mapping: one CTA per quad row (grid = rows x frames).  The CTA
//   1. counts the valid GIDs of rows u-1 and u from the 1-bit point-validity mask,
//   2. gets the exclusive prefix of row u by a single-pass DECOUPLED LOOK-BACK over
//      per-row status words (one warp reads 32 predecessors per step),
//   3. re-scans rows u-1, u, u+1 chunk by chunk with a packed 3-field warp-shuffle
//      block scan, which yields trimap[] of every neighbour needed for the twins --
//      so twins are emitted in the same pass, without reading trimap back.
// Integer outputs are bit-exact by construction (deterministic GID-order ranks).
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

namespace {

constexpr int kTriNT = 256;
constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagInc = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 62) - 1;

struct TriArgs {
  const uint32_t* vmask;
  long long vm_fs;
  int wpr;
  int M, N;
  long long G;  // per-frame capacity (= 2(M-1)(N-1))
  int64_t* trimap;
  int64_t* tris;
  int64_t* he;
  int64_t* ntri;
  unsigned long long* status;
  const float* pts;
  int pitch;
  long long pts_fs;
  float* normals;
  uint8_t* lflag;
  double l_max;
};

struct RowBits {
  const uint32_t* vm;
  int wpr, Mq, Nq;
  __device__ __forceinline__ uint32_t bit(int u, int v) const {
    return (__ldg(vm + (long long)u * wpr + (v >> 5)) >> (v & 31)) & 1u;
  }
  // bit0 = first triangle valid, bit1 = second; 0 off-grid
  __device__ __forceinline__ uint32_t quad(int u, int v) const {
    if (u < 0 || u >= Mq || v < 0 || v >= Nq) return 0u;
    const uint32_t p1 = bit(u, v), p2 = bit(u, v + 1), p3 = bit(u + 1, v + 1), p4 = bit(u + 1, v);
    return (p1 & p2 & p3) | ((p1 & p3 & p4) << 1);
  }
};

// exclusive block scan of a packed 3 x 10-bit counter word; returns the exclusive
// prefix, writes the block total to *total (all threads)
__device__ __forceinline__ uint32_t block_exscan_packed(uint32_t x, uint32_t* warp_tot,
                                                        uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t inc = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < kTriNT / 32 ? warp_tot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < kTriNT / 32) warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t warp_base = warp > 0 ? warp_tot[warp - 1] : 0u;
  *total = warp_tot[kTriNT / 32 - 1];
  const uint32_t ex = warp_base + inc - x;
  __syncthreads();  // warp_tot reused by the next chunk
  return ex;
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void emit_extras(const TriArgs& a, int f, long long t, int64_t ia,
                                            int64_t ib, int64_t ic) {
  const int N = a.N;
  const float* P = a.pts + f * a.pts_fs;
  const float* pa = P + (ia / N) * a.pitch + (ia % N) * 3;
  const float* pb = P + (ib / N) * a.pitch + (ib % N) * 3;
  const float* pc = P + (ic / N) * a.pitch + (ic % N) * 3;
  const double ax = pa[0], ay = pa[1], az = pa[2];
  const double bx = pb[0], by = pb[1], bz = pb[2];
  const double cx = pc[0], cy = pc[1], cz = pc[2];
  if (a.normals != nullptr) {
    double nx, ny, nz;
    unit_normal_f64(ax, ay, az, bx, by, bz, cx, cy, cz, nx, ny, nz);
    float* o = a.normals + (f * a.G + t) * 3;
    o[0] = (float)nx;
    o[1] = (float)ny;
    o[2] = (float)nz;
  }
  if (a.lflag != nullptr) {
    const double lab = edge_len_f64(ax, ay, az, bx, by, bz);
    const double lbc = edge_len_f64(bx, by, bz, cx, cy, cz);
    const double lca = edge_len_f64(cx, cy, cz, ax, ay, az);
    // np.maximum(lab, np.maximum(lbc, lca)) > l_max ; NaN propagates -> False
    const double m = (isnan(lbc) || isnan(lca)) ? lbc + lca : fmax(lbc, lca);
    const double e = (isnan(lab) || isnan(m)) ? lab + m : fmax(lab, m);
    a.lflag[f * a.G + t] = (uint8_t)(e > a.l_max);
  }
}

__global__ void __launch_bounds__(kTriNT) triangulate_kernel(TriArgs a) {
  __shared__ uint32_t warp_tot[kTriNT / 32];
  __shared__ unsigned long long red[kTriNT / 32];
  __shared__ long long s_base;
  __shared__ unsigned long long s_tot;

  const int u = blockIdx.x;
  const int f = blockIdx.y;
  const int Mq = a.M - 1, Nq = a.N - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  RowBits rb{a.vmask + f * a.vm_fs, a.wpr, Mq, Nq};

  // ---- 1. valid-GID counts of rows u (low 32 bits) and u-1 (high 32 bits)
  unsigned long long cnt = 0;
  for (int v = threadIdx.x; v < Nq; v += kTriNT) {
    cnt += __popc(rb.quad(u, v));
    cnt += (unsigned long long)__popc(rb.quad(u - 1, v)) << 32;
  }
  cnt = warp_sum_u64(cnt);
  if (lane == 0) red[warp] = cnt;
  __syncthreads();
  if (warp == 0) {
    unsigned long long t = lane < kTriNT / 32 ? red[lane] : 0ull;
    t = warp_sum_u64(t);
    // ---- 2. decoupled look-back over the rows of this frame
    unsigned long long* st = a.status + (long long)f * Mq;
    const unsigned long long tot_cur = t & 0xffffffffull;
    long long excl = 0;
    if (u == 0) {
      if (lane == 0) st_release_u64(st, kFlagInc | tot_cur);
    } else {
      if (lane == 0) st_release_u64(st + u, kFlagAgg | tot_cur);
      int j = u - 1;
      while (true) {
        const int idx = j - lane;
        unsigned long long s = kFlagInc;  // before row 0: inclusive prefix 0
        if (idx >= 0) {
          do {
            s = ld_acquire_u64(st + idx);
          } while ((s >> 62) == 0);
        }
        const uint32_t inc_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
        const int stop = inc_mask ? (__ffs(inc_mask) - 1) : 31;
        const unsigned long long val = (lane <= stop) ? (s & kValMask) : 0ull;
        excl += (long long)warp_sum_u64(val);
        if (inc_mask) break;
        j -= 32;
      }
      if (lane == 0) st_release_u64(st + u, kFlagInc | ((unsigned long long)excl + tot_cur));
    }
    if (lane == 0) {
      s_base = excl;
      s_tot = t;
    }
  }
  __syncthreads();
  const long long base_cur = s_base;
  const long long tot_cur = (long long)(s_tot & 0xffffffffull);
  const long long base_prev = base_cur - (long long)(s_tot >> 32);
  const long long base_next = base_cur + tot_cur;

  // ---- 3. chunked re-scan of rows u-1 / u / u+1 and emission
  const long long fG = (long long)f * a.G;
  int64_t* trimap = a.trimap + fG;
  int64_t* tris = a.tris + fG * 3;
  int64_t* he = a.he ? a.he + fG * 3 : nullptr;
  const int N = a.N;
  long long carry_p = 0, carry_c = 0, carry_n = 0;
  for (int c0 = 0; c0 < Nq; c0 += kTriNT) {
    const int v = c0 + threadIdx.x;
    const uint32_t qc = rb.quad(u, v);
    const uint32_t qp = rb.quad(u - 1, v);
    const uint32_t qn = rb.quad(u + 1, v);
    const uint32_t packed = __popc(qp) | (__popc(qc) << 10) | (__popc(qn) << 20);
    uint32_t total;
    const uint32_t ex = block_exscan_packed(packed, warp_tot, &total);
    const long long pre_p = carry_p + (ex & 1023u);
    const long long pre_c = carry_c + ((ex >> 10) & 1023u);
    const long long pre_n = carry_n + ((ex >> 20) & 1023u);
    if (v < Nq) {
      const long long g = 2ll * ((long long)u * Nq + v);
      const long long t0 = base_cur + pre_c;
      const long long t1 = t0 + (qc & 1u);
      const longlong2 tm = make_longlong2((qc & 1u) ? t0 : -1ll, (qc & 2u) ? t1 : -1ll);
      *reinterpret_cast<longlong2*>(trimap + g) = tm;
      const int64_t i1 = (int64_t)u * N + v, i2 = i1 + 1, i4 = i1 + N, i3 = i4 + 1;
      if (qc & 1u) {
        int64_t* o = tris + 3 * t0;
        o[0] = i3;
        o[1] = i2;
        o[2] = i1;
        if (he) {
          const uint32_t qr = rb.quad(u, v + 1);
          int64_t* e = he + 3 * t0;
          e[0] = (qr & 2u) ? 3 * (base_cur + pre_c + __popc(qc) + (qr & 1u)) + 0 : -1;
          e[1] = (qp & 2u) ? 3 * (base_prev + pre_p + (qp & 1u)) + 1 : -1;
          e[2] = (qc & 2u) ? 3 * t1 + 2 : -1;
        }
        if (a.normals || a.lflag) emit_extras(a, f, t0, i3, i2, i1);
      }
      if (qc & 2u) {
        int64_t* o = tris + 3 * t1;
        o[0] = i1;
        o[1] = i4;
        o[2] = i3;
        if (he) {
          const uint32_t ql = rb.quad(u, v - 1);
          int64_t* e = he + 3 * t1;
          e[0] = (ql & 1u) ? 3 * (base_cur + pre_c - __popc(ql)) + 0 : -1;
          e[1] = (qn & 1u) ? 3 * (base_next + pre_n) + 1 : -1;
          e[2] = (qc & 1u) ? 3 * t0 + 2 : -1;
        }
        if (a.normals || a.lflag) emit_extras(a, f, t1, i1, i4, i3);
      }
    }
    carry_p += total & 1023u;
    carry_c += (total >> 10) & 1023u;
    carry_n += (total >> 20) & 1023u;
  }
  if (u == Mq - 1 && threadIdx.x == 0) a.ntri[f] = base_cur + tot_cur;
}

// Twins from an arbitrary trimap (drop-in extract_halfedges_opc(trimap, M, N),
// mesh.py:99-135): one thread per quad, he pre-filled with -1 by the caller.
__global__ void halfedges_from_trimap_kernel(const int64_t* __restrict__ tm, int Mq, int Nq,
                                             long long n_tri, int64_t* __restrict__ he) {
  const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= (long long)Mq * Nq) return;
  const int u = (int)(q / Nq), v = (int)(q % Nq);
  const long long g = 2 * q;
  const long long t0 = tm[g], t1 = tm[g + 1];
  auto put = [&](long long t, int e, long long nb) {
    if (t >= 0 && t < n_tri) he[3 * t + e] = nb >= 0 ? 3 * nb + e : -1;
  };
  if (t0 >= 0) {
    put(t0, 0, v + 1 < Nq ? tm[g + 3] : -1);
    put(t0, 1, u > 0 ? tm[g - 2ll * Nq + 1] : -1);
    put(t0, 2, t1);
  }
  if (t1 >= 0) {
    put(t1, 0, v > 0 ? tm[g - 2] : -1);
    put(t1, 1, u + 1 < Mq ? tm[g + 2ll * Nq] : -1);
    put(t1, 2, t0);
  }
}

}  // namespace

size_t triangulate_workspace_bytes(int F, int M) {
  return (size_t)F * (size_t)(M > 1 ? M - 1 : 1) * sizeof(unsigned long long);
}

int triangulate(const uint32_t* vmask, int F, int M, int N, int64_t* trimap, int64_t* tris,
                int64_t* he, int64_t* ntri, const float* pts, int pitch, float* normals,
                double l_max, uint8_t* lflag, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (F < 1 || M < 2 || N < 2) return fail(ERR_INVALID, "triangulate: grid must be at least 2 x 2");
  if (!vmask || !trimap || !tris || !ntri) return fail(ERR_INVALID, "triangulate: null output");
  if ((normals || lflag) && (!pts || pitch < 3 * N))
    return fail(ERR_INVALID, "triangulate: normals / l_max flag need the point grid");
  if (ws_bytes < triangulate_workspace_bytes(F, M) || !ws)
    return fail(ERR_WORKSPACE, "triangulate: workspace too small");
  if (N - 1 > (1 << 30)) return fail(ERR_INVALID, "triangulate: row too wide");
  TriArgs a;
  a.vmask = vmask;
  a.wpr = (N + 31) / 32;
  a.vm_fs = (long long)M * a.wpr;
  a.M = M;
  a.N = N;
  a.G = 2ll * (M - 1) * (N - 1);
  a.trimap = trimap;
  a.tris = tris;
  a.he = he;
  a.ntri = ntri;
  a.status = static_cast<unsigned long long*>(ws);
  a.pts = pts;
  a.pitch = pitch;
  a.pts_fs = (long long)M * pitch;
  a.normals = normals;
  a.lflag = lflag;
  a.l_max = l_max;
  if (cudaMemsetAsync(ws, 0, triangulate_workspace_bytes(F, M), st) != cudaSuccess)
    return check_launch("triangulate: status reset");
  dim3 grid(M - 1, F);
  triangulate_kernel<<<grid, kTriNT, 0, st>>>(a);
  return check_launch("triangulate_kernel");
}

int halfedges_from_trimap(const int64_t* trimap, int M, int N, int64_t n_tri, int64_t* he,
                          cudaStream_t st) {
  if (M < 2 || N < 2) return fail(ERR_INVALID, "halfedges: grid must be at least 2 x 2");
  const long long Q = (long long)(M - 1) * (N - 1);
  if (Q == 0 || n_tri <= 0) return OK;
  const int nt = 256;
  halfedges_from_trimap_kernel<<<(unsigned)((Q + nt - 1) / nt), nt, 0, st>>>(trimap, M - 1, N - 1,
                                                                           n_tri, he);
  return check_launch("halfedges_from_trimap_kernel");
}

}  // namespace opcfe
