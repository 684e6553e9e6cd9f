// Region growing over twin edges.
//
// Reference semantics:
//   * _kernels.grow_segment (_native.pyx:170-222 == _fallback.py:47-80): from `seed`,
//     join every twin-adjacent triangle that carries `label`, is unvisited and -- for
//     ptp_max > 0 -- has all three vertices within ptp_max of the plane (anchor, normal),
//     d = (px-ax)*nx + (py-ay)*ny + (pz-az)*nz in that operation order, |d| > ptp_max
//     rejects; joined triangles are marked visited; the members are returned sorted.
//   * segmentation.region_growing_task (segmentation.py:117-170): seeds are the label's
//     unvisited triangles in ascending index, anchor = the seed triangle's centroid.
//
// The joinable set of one call does not depend on the visiting order (the predicate is
// per triangle), so a segment is exactly the connected component of the seed in the
// subgraph of eligible triangles -- computed here without any frontier loop:
//   1. eligible -> parent[t] = t (else -1);
//   2. every twin edge between two eligible triangles is a union: link the larger root
//      under the smaller with atomicCAS (roots stay component minima), finds use path
//      halving (benign races: parents only ever decrease toward the root);
//   3. compress (parent[t] = find(t), read-only walks so that no slot holding its final
//      root is overwritten by a concurrent halving step); members = parent == parent[seed];
//   4. ordered compaction (block counts -> one-CTA scan -> scatter) gives the sorted
//      member list and marks them visited.
// With ptp_max == 0 (the reference default) the components of ALL labels come out of
// one pass (segment_components): every segment of region_growing_task is a component
// whose minimum index is its seed.
#include "common.cuh"
#include "opcfe_internal.h"

namespace opcfe {

namespace {

constexpr int kSegNT = 256;
constexpr uint8_t kUnassigned = 255;

// link phase: path halving; loads bypass L1 (other SMs CAS the roots in L2)
__device__ __forceinline__ int find_root(int* parent, int x) {
  int p = __ldcg(parent + x);
  while (p != x) {
    const int g = __ldcg(parent + p);
    if (g != p) parent[x] = g;  // path halving (benign race: g is an ancestor of x)
    x = p;
    p = g;
  }
  return x;
}

// compress phase: read-only walk.  A halving write here could land AFTER another
// thread stored the final root into that slot and regress it to an inner ancestor.
__device__ __forceinline__ int find_root_ro(const int* parent, int x) {
  int p = __ldcg(parent + x);
  while (p != x) {
    x = p;
    p = __ldcg(parent + x);
  }
  return x;
}

__device__ __forceinline__ void unite(int* parent, int a, int b) {
  while (true) {
    a = find_root(parent, a);
    b = find_root(parent, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    // link root b under the smaller root a (only if b is still a root)
    if (atomicCAS(parent + b, b, a) == b) return;
  }
}

// ptp predicate of one triangle (the reference's operation order, fp64, no contraction)
__device__ __forceinline__ bool within_ptp(const int64_t* tris, const double* pts, long long t,
                                           double ax, double ay, double az, double nx,
                                           double ny, double nz, double ptp) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const long long v = tris[3 * t + k];
    const double* p = pts + 3 * v;
    const double d = dadd(dadd(dmul(dsub(p[0], ax), nx), dmul(dsub(p[1], ay), ny)),
                          dmul(dsub(p[2], az), nz));
    if (fabs(d) > ptp) return false;
  }
  return true;
}

struct GrowArgs {
  const int64_t* tris;
  const int64_t* he;
  const double* pts;
  const uint8_t* groups;
  uint8_t* visited;
  int n;
  int seed;
  int label;
  double ax, ay, az, nx, ny, nz, ptp;
  int* parent;
};

__global__ void grow_init_kernel(GrowArgs a) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= a.n) return;
  bool el = t == a.seed;
  if (!el && a.groups[t] == a.label && !a.visited[t])
    el = a.ptp <= 0.0 ||
         within_ptp(a.tris, a.pts, t, a.ax, a.ay, a.az, a.nx, a.ny, a.nz, a.ptp);
  a.parent[t] = el ? t : -1;
}

// every undirected twin edge once (from its larger triangle index)
__global__ void link_kernel(const int64_t* __restrict__ he, int n, int* parent) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || parent[t] < 0) return;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const long long tw = he[3ll * t + e];
    if (tw < 0) continue;
    const int u = (int)(tw / 3);
    if (u < t && parent[u] >= 0) unite(parent, t, u);
  }
}

__global__ void compress_kernel(int n, int* parent) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || parent[t] < 0) return;
  parent[t] = find_root_ro(parent, t);  // only ever a root: no regression of other slots
}

// all labels at once: same-label (non-unassigned) twin neighbours
__global__ void comp_init_kernel(const uint8_t* __restrict__ groups, int n, int* parent) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  parent[t] = groups[t] != kUnassigned ? t : -1;
}
__global__ void comp_link_kernel(const int64_t* __restrict__ he, const uint8_t* __restrict__ groups,
                                 int n, int* parent) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n || parent[t] < 0) return;
  const uint8_t g = groups[t];
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const long long tw = he[3ll * t + e];
    if (tw < 0) continue;
    const int u = (int)(tw / 3);
    if (u < t && groups[u] == g) unite(parent, t, u);
  }
}
__global__ void comp_out_kernel(const int* __restrict__ parent, int n, int64_t* __restrict__ comp,
                                int64_t* __restrict__ size) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int r = parent[t];
  comp[t] = r;
  if (size != nullptr) {
    size[t] = 0;  // (re)initialised here; sizes accumulate at the roots below
  }
}
__global__ void comp_size_kernel(const int* __restrict__ parent, int n, int64_t* size) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int r = parent[t];
  if (r >= 0) atomicAdd(reinterpret_cast<unsigned long long*>(size + r), 1ull);
}

// ---- ordered compaction of {t : parent[t] == parent[seed]}: sorted members, visited = 1
__global__ void member_count_kernel(const int* __restrict__ parent, int n, int seed,
                                    int* __restrict__ block_cnt) {
  __shared__ int wsum[kSegNT / 32];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int root = parent[seed];
  const bool m = t < n && parent[t] == root;
  const unsigned b = __ballot_sync(0xffffffffu, m);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = __popc(b);
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kSegNT / 32; ++w) s += wsum[w];
    block_cnt[blockIdx.x] = s;
  }
}

// exclusive scan of the block counts (one CTA); total -> *n_out
__global__ void block_scan_kernel(int* cnt, int nb, int64_t* n_out) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int carry = 0;
  for (int b0 = 0; b0 < nb; b0 += 1024) {
    const int i = b0 + threadIdx.x;
    const int x = i < nb ? cnt[i] : 0;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    int woff = 0, tot = 0;
    for (int w = 0; w < 32; ++w) {
      const int v = wsum[w];
      woff += w < warp ? v : 0;
      tot += v;
    }
    if (i < nb) cnt[i] = carry + woff + inc - x;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) *n_out = carry;
}

__global__ void member_scatter_kernel(const int* __restrict__ parent, int n, int seed,
                                      const int* __restrict__ block_off, uint8_t* visited,
                                      int64_t* __restrict__ members) {
  __shared__ int wsum[kSegNT / 32];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int root = parent[seed];
  const bool m = t < n && parent[t] == root;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned b = __ballot_sync(0xffffffffu, m);
  if (lane == 0) wsum[warp] = __popc(b);
  __syncthreads();
  int woff = 0;
  for (int w = 0; w < warp; ++w) woff += wsum[w];
  if (m) {
    members[block_off[blockIdx.x] + woff + __popc(b & ((1u << lane) - 1u))] = t;
    visited[t] = 1;
  }
}

inline int blocks(long long n) { return (int)((n + kSegNT - 1) / kSegNT); }

}  // namespace

size_t segments_workspace_bytes(long long n_tri) {
  const long long nb = (n_tri + kSegNT - 1) / kSegNT;
  return (size_t)(n_tri * 4 + 256 + nb * 4 + 256);
}

int grow_segment(const int64_t* tris, const int64_t* he, const double* pts,
                 const uint8_t* groups, uint8_t* visited, long long n_tri, long long seed,
                 int label, const double* anchor, const double* normal, double ptp_max,
                 int64_t* members, int64_t* n_members, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  if (n_tri < 1 || n_tri > INT32_MAX - 1) return fail(ERR_INVALID, "grow_segment: bad n_tri");
  if (seed < 0 || seed >= n_tri) return fail(ERR_INVALID, "grow_segment: seed out of range");
  if (!he || !groups || !visited || !members || !n_members || !anchor || !normal)
    return fail(ERR_INVALID, "grow_segment: null buffer");
  if (ptp_max > 0.0 && (!tris || !pts))
    return fail(ERR_INVALID, "grow_segment: the ptp check needs triangles and points");
  if (!ws || ws_bytes < segments_workspace_bytes(n_tri))
    return fail(ERR_WORKSPACE, "grow_segment: workspace too small");
  const int n = (int)n_tri;
  int* parent = static_cast<int*>(ws);
  int* bcnt = reinterpret_cast<int*>(static_cast<char*>(ws) + ((size_t)n * 4 + 255) / 256 * 256);
  GrowArgs a{tris, he, pts, groups, visited, n, (int)seed, label, anchor[0], anchor[1],
             anchor[2], normal[0], normal[1], normal[2], ptp_max, parent};
  const int nb = blocks(n);
  grow_init_kernel<<<nb, kSegNT, 0, st>>>(a);
  link_kernel<<<nb, kSegNT, 0, st>>>(he, n, parent);
  compress_kernel<<<nb, kSegNT, 0, st>>>(n, parent);
  member_count_kernel<<<nb, kSegNT, 0, st>>>(parent, n, (int)seed, bcnt);
  block_scan_kernel<<<1, 1024, 0, st>>>(bcnt, nb, n_members);
  member_scatter_kernel<<<nb, kSegNT, 0, st>>>(parent, n, (int)seed, bcnt, visited, members);
  return check_launch("grow_segment");
}

int segment_components(const int64_t* he, const uint8_t* groups, long long n_tri, int64_t* comp,
                       int64_t* size, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n_tri < 1 || n_tri > INT32_MAX - 1) return fail(ERR_INVALID, "segment_components: bad n_tri");
  if (!he || !groups || !comp) return fail(ERR_INVALID, "segment_components: null buffer");
  if (!ws || ws_bytes < segments_workspace_bytes(n_tri))
    return fail(ERR_WORKSPACE, "segment_components: workspace too small");
  const int n = (int)n_tri;
  int* parent = static_cast<int*>(ws);
  const int nb = blocks(n);
  comp_init_kernel<<<nb, kSegNT, 0, st>>>(groups, n, parent);
  comp_link_kernel<<<nb, kSegNT, 0, st>>>(he, groups, n, parent);
  compress_kernel<<<nb, kSegNT, 0, st>>>(n, parent);
  comp_out_kernel<<<nb, kSegNT, 0, st>>>(parent, n, comp, size);
  if (size) comp_size_kernel<<<nb, kSegNT, 0, st>>>(parent, n, size);
  return check_launch("segment_components");
}

}  // namespace opcfe
