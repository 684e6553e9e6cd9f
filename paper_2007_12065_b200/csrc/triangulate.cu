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
//   * optional extras: mesh-order normals (geometry.py:134-147, fp64 math) and the
//     l_max longest-edge flag (segmentation.py:59-67,73, fp64 math), by a 4th launch
//     per quad (quad_extras_kernel) once trimap exists.
//
// B200 mapping: three launches, none of which waits on another CTA.
//   1. tri_count_kernel: one warp per quad row counts its valid triangles (popc of the
//      row's first/second masks) -> row_base[f][u];
//   2. tri_scan_kernel: one CTA per frame turns the row counts into exclusive row
//      prefixes (row_base[f][Mq] = triangle count of the frame);
//   3. triangulate_kernel: one CTA per quad row, 4 warps (2 for rows <= 256 quads), a warp
//      = 32 consecutive quads.
//      Validity is pure bit algebra on the 1-bit point mask: from 3 mask words per point
//      row a warp gets the 32-quad first/second masks of rows u-1, u, u+1 and of the
//      left/right neighbour quads with a few shifts/ANDs (lane-uniform), so ranks inside
//      the warp are popc(mask & lanemask_lt) -- no shuffles, no per-quad loads.  Rows
//      u-1 / u / u+1 bases come from row_base, so every twin index (which needs trimap
//      of the rows above and below) is computed in the same pass -- trimap is never
//      read back.  Per row segment (up to 8192 quads) one block scan of the packed
//      per-group counts of rows u-1 | u | u+1 gives every 32-quad group its prefixes;
//      each warp then emits its groups with no further block barrier: triangles and
//      twins (int64, 24 B each) are staged per warp in shared memory and written out as
//      contiguous, fully coalesced 8-B streams; trimap pairs are 16-B stores.
//   (A single-pass decoupled look-back over row status words stalled 28 % of the warps
//   at the barrier behind the look-back: 0.39 ms.)
// Integer outputs are bit-exact by construction (deterministic GID-order ranks).
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

namespace {

// threads per row CTA: 128 (4 warps), 64 for rows of <= 8 groups (256 quads).  Measured
// per 16 x 1080p / 64 x 480x640 / 512 x 64x1024 / 256 x 250x250 frames: 256 threads 0.61 /
// 0.41 / 1.10 / 0.44 ms, 128: 0.61 / 0.34 / 1.04 / 0.32, 64: 0.64 / 0.36 / 1.07 / 0.29
// (narrow rows left most warps of a 256-thread CTA idle behind the block scan).

struct TriArgs {
  const uint32_t* vmask;
  long long vm_fs;
  int wpr;
  int M, N;
  long long G;  // per-frame capacity (= 2(M-1)(N-1))
  int64_t* trimap;
  int64_t* tris;
  int64_t* he;
  const long long* row_base;  // [F][M]: exclusive prefix of row u's triangles; [Mq] = total
};

// validity bits of point row r around the 32-point group starting at v0 = 32*word
struct PtBits {
  uint32_t a, a1, a2, am;  // bit i = point v0+i, v0+i+1, v0+i+2, v0+i-1
};

__device__ __forceinline__ PtBits pt_bits(const uint32_t* row, int word, int wpr) {
  const uint32_t w0 = __ldg(row + word);
  const uint32_t w1 = (word + 1 < wpr) ? __ldg(row + word + 1) : 0u;
  const uint32_t wm = (word > 0) ? __ldg(row + word - 1) : 0u;
  return PtBits{w0, (w0 >> 1) | (w1 << 31), (w0 >> 2) | (w1 << 30), (w0 << 1) | (wm >> 31)};
}

// first / second masks of a quad row from its two point rows (top t, bottom b)
struct QuadBits {
  uint32_t f, s;     // quads v0+i
  uint32_t fr, sr;   // quads v0+i+1 (right neighbour)
  uint32_t fl, sl;   // quads v0+i-1 (left neighbour)
};

__device__ __forceinline__ QuadBits quad_bits(const PtBits& t, const PtBits& b) {
  QuadBits q;
  q.f = t.a & t.a1 & b.a1;    // p1 & p2 & p3
  q.s = t.a & b.a1 & b.a;     // p1 & p3 & p4
  q.fr = t.a1 & t.a2 & b.a2;
  q.sr = t.a1 & b.a2 & b.a1;
  q.fl = t.am & t.a & b.a;
  q.sl = t.am & b.a & b.am;
  return q;
}

// Normals + l_max flags per QUAD, after the triangulation (which then runs its lean
// variant): one thread loads the quad's 4 points (coalesced) and converts them to fp64
// once; the two triangles (p3,p2,p1) and (p1,p4,p3) share the diagonal p1 - p3, so 5
// edge vectors serve 6 edges.  Results go to mesh order through trimap.  The arithmetic
// is numpy's (geometry.py:134-147; segmentation.py:59-67,73), so normals are
// float32(reference) exactly and the flags bit-exact (see sq_threshold).
// float32(fl64(c / fl64(sqrt(s)))) -- the reference's fp64 normal component rounded to
// fp32 -- without the correctly rounded divide and square root: q = c * rsqrt(s) is
// within a few ulp64 of fl64(c / n), so both round to the same fp32 value unless q lies
// within 16 ulp64 of an fp32 rounding midpoint (probability ~6e-8) or in the fp32
// subnormal range; those take the exact path.
__device__ __forceinline__ float div_norm_to_f32(double c, double r, double s) {
  const double q = c * r;
  const long long b = __double_as_longlong(q);
  const int low = (int)(b & 0x1fffffff) - 0x10000000;  // distance to the fp32 midpoint
  if (low > 16 || low < -16) {
    if (fabs(q) >= 2.4e-38) return (float)q;             // fp32 normal range
    if (q == 0.0) return (float)q;
  }
  return (float)__ddiv_rn(c, __dsqrt_rn(s));
}

__device__ __forceinline__ void normal_from_edges_f64(const double* e1, const double* e2,
                                                      float* o) {
  const double x = dsub(dmul(e1[1], e2[2]), dmul(e1[2], e2[1]));
  const double y = dsub(dmul(e1[2], e2[0]), dmul(e1[0], e2[2]));
  const double z = dsub(dmul(e1[0], e2[1]), dmul(e1[1], e2[0]));
  const double s = dadd(dadd(dmul(x, x), dmul(y, y)), dmul(z, z));
  if (s >= 2.3e-308 && s <= 1.7e308) {  // normal range: rsqrt <= 1 ulp
    const double r = rsqrt(s);
    o[0] = div_norm_to_f32(x, r, s);
    o[1] = div_norm_to_f32(y, r, s);
    o[2] = div_norm_to_f32(z, r, s);
  } else {
    const double n = __dsqrt_rn(s);
    if (n > 0.0) {
      o[0] = (float)__ddiv_rn(x, n);
      o[1] = (float)__ddiv_rn(y, n);
      o[2] = (float)__ddiv_rn(z, n);
    } else {
      o[0] = o[1] = o[2] = __int_as_float(0x7fc00000);
    }
  }
}
__device__ __forceinline__ double len2_f64(const double* d) {
  return dadd(dadd(dmul(d[0], d[0]), dmul(d[1], d[1])), dmul(d[2], d[2]));
}

__global__ void __launch_bounds__(128) quad_extras_kernel(const float* __restrict__ pts, int pitch,
                                                          long long pts_fs, int M, int N,
                                                          const int64_t* __restrict__ trimap,
                                                          long long G, float* __restrict__ normals,
                                                          uint8_t* __restrict__ lflag,
                                                          double l2_thr) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  const int u = blockIdx.y, f = blockIdx.z;
  const int Nq = N - 1;
  if (v >= Nq) return;
  const long long gid = 2ll * ((long long)u * Nq + v);
  // the quad's points (always in bounds) are loaded before, not after, its trimap pair:
  // both loads are in flight together instead of back to back (C3: ~1 % on the stage)
  const float* P1 = pts + f * pts_fs + (long long)u * pitch + 3 * v;
  const float* P4 = P1 + pitch;
  float q1[3], q2[3], q3[3], q4[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    q1[j] = __ldg(P1 + j);
    q2[j] = __ldg(P1 + 3 + j);
    q4[j] = __ldg(P4 + j);
    q3[j] = __ldg(P4 + 3 + j);
  }
  const longlong2 tm = __ldg(reinterpret_cast<const longlong2*>(trimap + f * G + gid));
  if (tm.x < 0 && tm.y < 0) return;
  double p1[3], p2[3], p3[3], p4[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    p1[j] = q1[j];
    p2[j] = q2[j];
    p4[j] = q4[j];
    p3[j] = q3[j];
  }
  double d31[3], d13[3], e23[3], e14[3];  // p3 - p1, p1 - p3, p2 - p3, p4 - p1
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    d13[j] = dsub(p1[j], p3[j]);
    d31[j] = -d13[j];  // exact: the same value numpy's p3 - p1 rounds to
    e23[j] = dsub(p2[j], p3[j]);
    e14[j] = dsub(p4[j], p1[j]);
  }
  if (tm.x >= 0) {  // (p3, p2, p1): e1 = p2 - p3, e2 = p1 - p3
    if (normals) normal_from_edges_f64(e23, d13, normals + (f * G + tm.x) * 3);
    if (lflag) {
      double e12[3];  // c - b = p1 - p2
#pragma unroll
      for (int j = 0; j < 3; ++j) e12[j] = dsub(p1[j], p2[j]);
      lflag[f * G + tm.x] =
          (uint8_t)longest_edge_exceeds(len2_f64(e23), len2_f64(e12), len2_f64(d31), l2_thr);
    }
  }
  if (tm.y >= 0) {  // (p1, p4, p3): e1 = p4 - p1, e2 = p3 - p1
    if (normals) normal_from_edges_f64(e14, d31, normals + (f * G + tm.y) * 3);
    if (lflag) {
      double e43[3];  // c - b = p3 - p4
#pragma unroll
      for (int j = 0; j < 3; ++j) e43[j] = dsub(p3[j], p4[j]);
      lflag[f * G + tm.y] =
          (uint8_t)longest_edge_exceeds(len2_f64(e14), len2_f64(e43), len2_f64(d13), l2_thr);
    }
  }
}

template <int kTriNT>
__global__ void __launch_bounds__(kTriNT, 1024 / kTriNT) triangulate_kernel(TriArgs a) {
  constexpr int kTriWarps = kTriNT / 32;
  constexpr int kSegGroups = kTriNT;  // 32-quad groups per scan segment (one per thread)
  __shared__ unsigned long long red[kTriWarps];
  __shared__ unsigned long long gpre[kSegGroups];     // packed per-group exclusive prefixes
  __shared__ int64_t stage[kTriWarps][2][3 * 64];     // per-warp tris / twins staging

  const int u = blockIdx.x;
  const int f = blockIdx.y;
  const int Mq = a.M - 1, Nq = a.N - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t* vm = a.vmask + f * a.vm_fs;
  const int groups = (Nq + 31) / 32;
  const long long* rb = a.row_base + (long long)f * a.M;
  const long long base_cur = rb[u];
  const long long base_prev = u > 0 ? rb[u - 1] : 0;
  const long long base_next = rb[u + 1];

  // ---- segments of up to kSegGroups 32-quad groups: packed group counts of rows
  // u-1 | u | u+1 (21 bits each), block exclusive scan, then every warp emits its groups
  // independently (ranks by popc, per-warp staging, no block barrier per group).
  const long long fG = (long long)f * a.G;
  int64_t* trimap = a.trimap + fG;
  int64_t* tris = a.tris + fG * 3;
  int64_t* he = a.he ? a.he + fG * 3 : nullptr;
  const int N = a.N;
  const uint32_t lt = (1u << lane) - 1u;
  constexpr unsigned long long F21 = (1ull << 21) - 1;
  auto group_bits = [&](int g, QuadBits& qp, QuadBits& qc, QuadBits& qn) {
    const PtBits pu = pt_bits(vm + (long long)u * a.wpr, g, a.wpr);
    const PtBits pd = pt_bits(vm + (long long)(u + 1) * a.wpr, g, a.wpr);
    qc = quad_bits(pu, pd);
    qp = QuadBits{};
    qn = QuadBits{};
    if (u > 0) qp = quad_bits(pt_bits(vm + (long long)(u - 1) * a.wpr, g, a.wpr), pu);
    if (u + 1 < Mq) qn = quad_bits(pd, pt_bits(vm + (long long)(u + 2) * a.wpr, g, a.wpr));
  };
  long long carry_p = 0, carry_c = 0, carry_n = 0;
  for (int s0 = 0; s0 < groups; s0 += kSegGroups) {
    const int ng = min(kSegGroups, groups - s0);
    unsigned long long x = 0;  // this thread's group (one per thread: kSegGroups == kTriNT)
    if (threadIdx.x < ng) {
      QuadBits qp, qc, qn;
      group_bits(s0 + threadIdx.x, qp, qc, qn);
      x = (unsigned long long)(__popc(qp.f) + __popc(qp.s)) |
          ((unsigned long long)(__popc(qc.f) + __popc(qc.s)) << 21) |
          ((unsigned long long)(__popc(qn.f) + __popc(qn.s)) << 42);
    }
    // block exclusive scan of the packed counts (fields never carry: <= 2 * 8192)
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    __syncthreads();  // previous segment's gpre / red reads are done
    if (lane == 31) red[warp] = inc;
    __syncthreads();
    unsigned long long woff = 0, stot = 0;
#pragma unroll
    for (int w = 0; w < kTriWarps; ++w) {
      const unsigned long long r = red[w];
      woff += (w < warp) ? r : 0ull;
      stot += r;
    }
    gpre[threadIdx.x] = woff + inc - x;
    __syncthreads();

    int64_t* st_t = stage[warp][0];
    int64_t* st_h = stage[warp][1];
    for (int gl = warp; gl < ng; gl += kTriWarps) {
      const int g = s0 + gl;
      const int v = 32 * g + lane;
      QuadBits qp, qc, qn;
      group_bits(g, qp, qc, qn);
      const unsigned long long pre = gpre[gl];
      const uint32_t bf = (qc.f >> lane) & 1u, bs = (qc.s >> lane) & 1u;
      const int l0 = __popc(qc.f & lt) + __popc(qc.s & lt), l1 = l0 + (int)bf;  // warp-local
      const long long t_first = base_cur + carry_c + (long long)((pre >> 21) & F21);
      const long long pre_p = carry_p + (long long)(pre & F21) + __popc(qp.f & lt) + __popc(qp.s & lt);
      const long long pre_n = carry_n + (long long)((pre >> 42) & F21) + __popc(qn.f & lt) +
                              __popc(qn.s & lt);
      if (v < Nq) {
        const long long gid = 2ll * ((long long)u * Nq + v);
        const long long t0 = t_first + l0;
        const long long t1 = t0 + bf;
        __stcs(reinterpret_cast<longlong2*>(trimap + gid), make_longlong2(bf ? t0 : -1ll, bs ? t1 : -1ll));
        const int64_t i1 = (int64_t)u * N + v, i2 = i1 + 1, i4 = i1 + N, i3 = i4 + 1;
        if (bf) {
          st_t[3 * l0] = i3;
          st_t[3 * l0 + 1] = i2;
          st_t[3 * l0 + 2] = i1;
          if (he) {
            st_h[3 * l0] = ((qc.sr >> lane) & 1u)
                               ? 3 * (t0 + bf + bs + ((qc.fr >> lane) & 1u)) + 0 : -1;
            st_h[3 * l0 + 1] = ((qp.s >> lane) & 1u)
                                   ? 3 * (base_prev + pre_p + ((qp.f >> lane) & 1u)) + 1 : -1;
            st_h[3 * l0 + 2] = bs ? 3 * t1 + 2 : -1;
          }
        }
        if (bs) {
          st_t[3 * l1] = i1;
          st_t[3 * l1 + 1] = i4;
          st_t[3 * l1 + 2] = i3;
          if (he) {
            const uint32_t lf = (qc.fl >> lane) & 1u, ls = (qc.sl >> lane) & 1u;
            st_h[3 * l1] = lf ? 3 * (t0 - lf - ls) + 0 : -1;
            st_h[3 * l1 + 1] = ((qn.f >> lane) & 1u) ? 3 * (base_next + pre_n) + 1 : -1;
            st_h[3 * l1 + 2] = bf ? 3 * t0 + 2 : -1;
          }
        }
      }
      __syncwarp();
      // contiguous, coalesced copy-out of this group's triangles [t_first, + n)
      const int n3 = 3 * (__popc(qc.f) + __popc(qc.s));
      int64_t* tdst = tris + 3 * t_first;
      for (int i = lane; i < n3; i += 32) __stcs(reinterpret_cast<long long*>(tdst) + i, st_t[i]);
      if (he) {
        int64_t* hdst = he + 3 * t_first;
        for (int i = lane; i < n3; i += 32) __stcs(reinterpret_cast<long long*>(hdst) + i, st_h[i]);
      }
      __syncwarp();  // staging reused by the warp's next group
    }
    carry_p += (long long)(stot & F21);
    carry_c += (long long)((stot >> 21) & F21);
    carry_n += (long long)((stot >> 42) & F21);
  }
}

// valid-triangle count of every quad row: one warp per row
__global__ void __launch_bounds__(256) tri_count_kernel(const uint32_t* __restrict__ vmask,
                                                        long long vm_fs, int wpr, int M, int N,
                                                        long long* __restrict__ row_base) {
  const int lane = threadIdx.x & 31;
  const int u = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int f = blockIdx.y;
  if (u >= M - 1) return;
  const uint32_t* vm = vmask + f * vm_fs;
  const int groups = (N - 1 + 31) / 32;
  unsigned cnt = 0;
  for (int g = lane; g < groups; g += 32) {
    const QuadBits q = quad_bits(pt_bits(vm + (long long)u * wpr, g, wpr),
                                 pt_bits(vm + (long long)(u + 1) * wpr, g, wpr));
    cnt += __popc(q.f) + __popc(q.s);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if (lane == 0) row_base[(long long)f * M + u] = cnt;
}

// exclusive prefix of the row counts, one CTA per frame; row_base[Mq] = ntri[f] = total
__global__ void __launch_bounds__(1024) tri_scan_kernel(long long* __restrict__ row_base, int M,
                                                         int64_t* __restrict__ ntri) {
  __shared__ long long wsum[32];
  const int f = blockIdx.x;
  const int Mq = M - 1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long* rb = row_base + (long long)f * M;
  long long carry = 0;
  for (int r0 = 0; r0 < Mq; r0 += 1024) {
    const int r = r0 + threadIdx.x;
    const long long x = r < Mq ? rb[r] : 0;
    long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    long long woff = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      const long long t = wsum[w];
      woff += (w < warp) ? t : 0;
      tot += t;
    }
    if (r < Mq) rb[r] = carry + woff + inc - x;
    carry += tot;
    __syncthreads();  // wsum reused
  }
  if (threadIdx.x == 0) {
    rb[Mq] = carry;
    ntri[f] = carry;
  }
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
  return (size_t)F * (size_t)(M > 1 ? M : 2) * sizeof(long long);  // row_base [F][M]
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
  long long* row_base = static_cast<long long*>(ws);
  a.row_base = row_base;
  tri_count_kernel<<<dim3((M - 1 + 7) / 8, F), 256, 0, st>>>(vmask, a.vm_fs, a.wpr, M, N, row_base);
  if (int rc = check_launch("tri_count_kernel")) return rc;
  tri_scan_kernel<<<F, 1024, 0, st>>>(row_base, M, ntri);
  if (int rc = check_launch("tri_scan_kernel")) return rc;
  dim3 grid(M - 1, F);
  if (N - 1 <= 256)
    triangulate_kernel<64><<<grid, 64, 0, st>>>(a);
  else
    triangulate_kernel<128><<<grid, 128, 0, st>>>(a);
  if (int rc = check_launch("triangulate_kernel")) return rc;
  if (normals || lflag) {
    dim3 xg((N - 1 + 127) / 128, M - 1, F);
    quad_extras_kernel<<<xg, 128, 0, st>>>(pts, pitch, (long long)M * pitch, M, N, trimap, a.G,
                                            normals, lflag, sq_threshold(l_max));
    return check_launch("quad_extras_kernel");
  }
  return OK;
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
