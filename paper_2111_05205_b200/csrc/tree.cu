// tree.cu -- the space-time octree and its lists, built on the device.
//
// Restates the reference's build_tree (pkg/src/tdwavebem/fmm_tree.py:73-231) bit
// for bit, as the host builder paper_2111_05205_b200/fmm_tree.py does (both are
// pinned to tests/golden/tree_cfg{1,2,3,4}.npz):
//   * leaf depth: the first level whose fullest cell holds <= Z centroids
//     (:86-97); cell coordinates clip(floor((p - lo) / side), 0, n - 1);
//   * cells per level in lexicographic (x, y, z) order = ascending packed key
//     (np.unique, :99-114); elem_cell = rank of an element's cell; parents by
//     binary search of coords >> 1 (:116-123);
//   * interaction lists (:134-160): per observer cell (ascending), the 27 parent
//     neighbours (dx, dy, dz) x 8 children (cx, cy, cz) in that order, kept when
//     the candidate exists and is not adjacent;
//   * near pairs (:163-177): per leaf cell (ascending), its existing neighbours in
//     (dx, dy, dz) order, all (element of a) x (element of b) in row-major order,
//     elements of a cell ascending;
//   * the mu-interval causality check and the marginal ("extra") element pairs
//     (:188-231), with the reference's or SURVEY 8(c)'s corrected margin/reach.
// Floating-point expressions are evaluated in the host builder's (numpy's)
// operation order with explicit round-to-nearest intrinsics (no contraction),
// so every comparison sees the same doubles.  Counting passes + scans give each
// list's output offsets; the fills then write in the reference's order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "tdw_impl.cuh"

struct tdw_tree {
  tdw_ctx* ctx = nullptr;
  int ns = 0, leaf = 0;
  double centre[3] = {0, 0, 0}, root_half = 0.0;
  std::vector<std::vector<int>> coords;       // [level][n*3]
  std::vector<std::vector<long long>> parent;  // [level][n] (level 0: empty)
  std::vector<std::vector<long long>> elem_cell;  // [level][ns]
  std::vector<std::vector<long long>> il_obs, il_src;
  std::vector<std::vector<int>> il_off;       // [level][nil*3]
  std::vector<long long> near_i, near_j;
  std::vector<int> extra_levels;
  std::vector<std::vector<long long>> extra_i, extra_j;
  std::string err;
};

namespace {

constexpr int KSH = 21;
__host__ __device__ __forceinline__ long long pack_key(long long x, long long y, long long z) {
  return (x << (2 * KSH)) | (y << KSH) | z;
}

// leaf-level cell coordinates of every centroid: clip(floor((p - lo) / side), 0, n - 1)
__global__ void cell_coords_kernel(const double* __restrict__ cen, int ns, double lo0, double lo1, double lo2,
                                   double side, long long n, long long* keys, int* vals) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ns; e += gridDim.x * blockDim.x) {
    const double lo[3] = {lo0, lo1, lo2};
    long long c[3];
    for (int k = 0; k < 3; ++k) {
      const double q = __ddiv_rn(__dsub_rn(cen[3 * e + k], lo[k]), side);
      long long v = (long long)floor(q);
      c[k] = v < 0 ? 0 : (v > n - 1 ? n - 1 : v);
    }
    keys[e] = pack_key(c[0], c[1], c[2]);
    vals[e] = e;
  }
}

__global__ void shift_keys_kernel(const long long* __restrict__ leaf_keys, int ns, int sh, long long* keys,
                                  int* vals) {
  const long long m = (1LL << KSH) - 1;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < ns; e += gridDim.x * blockDim.x) {
    const long long k = leaf_keys[e];
    keys[e] = pack_key(((k >> (2 * KSH)) & m) >> sh, ((k >> KSH) & m) >> sh, (k & m) >> sh);
    vals[e] = e;
  }
}

// run heads of a sorted key array: head[i] = 1 where a new key starts
__global__ void heads_kernel(const long long* __restrict__ k, int n, int* head) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    head[i] = (i == 0 || k[i] != k[i - 1]) ? 1 : 0;
}

__device__ __forceinline__ long long find_key(const long long* __restrict__ keys, long long n, long long q) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (keys[mid] < q) lo = mid + 1; else hi = mid;
  }
  return (lo < n && keys[lo] == q) ? lo : -1;
}

__device__ __forceinline__ void unpack(long long k, long long& x, long long& y, long long& z) {
  const long long m = (1LL << KSH) - 1;
  x = (k >> (2 * KSH)) & m;
  y = (k >> KSH) & m;
  z = k & m;
}

// interaction-list candidates of cell c: parent neighbour q = 0..26, child h = 0..7
__device__ __forceinline__ bool il_candidate(const long long* __restrict__ keys, long long n, long long cx,
                                             long long cy, long long cz, int q, int h, long long& src,
                                             int* off) {
  const long long px = (cx >> 1) + (q / 9 - 1), py = (cy >> 1) + ((q / 3) % 3 - 1), pz = (cz >> 1) + (q % 3 - 1);
  const long long x = (px << 1) + (h >> 2), y = (py << 1) + ((h >> 1) & 1), z = (pz << 1) + (h & 1);
  if (x < 0 || y < 0 || z < 0) return false;
  const long long dx = x - cx, dy = y - cy, dz = z - cz;
  if (llabs(dx) <= 1 && llabs(dy) <= 1 && llabs(dz) <= 1) return false;
  src = find_key(keys, n, pack_key(x, y, z));
  if (src < 0) return false;
  off[0] = (int)dx;
  off[1] = (int)dy;
  off[2] = (int)dz;
  return true;
}

__global__ void il_count_kernel(const long long* __restrict__ keys, long long n, int* cnt) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    long long cx, cy, cz;
    unpack(keys[c], cx, cy, cz);
    int k = 0;
    for (int q = 0; q < 27; ++q)
      for (int h = 0; h < 8; ++h) {
        long long s;
        int off[3];
        k += il_candidate(keys, n, cx, cy, cz, q, h, s, off);
      }
    cnt[c] = k;
  }
}

__global__ void il_fill_kernel(const long long* __restrict__ keys, long long n, const long long* __restrict__ start,
                               long long* obs, long long* src, int* off3) {
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < n; c += (long long)gridDim.x * blockDim.x) {
    long long cx, cy, cz;
    unpack(keys[c], cx, cy, cz);
    long long p = start[c];
    for (int q = 0; q < 27; ++q)
      for (int h = 0; h < 8; ++h) {
        long long s;
        int off[3];
        if (il_candidate(keys, n, cx, cy, cz, q, h, s, off)) {
          obs[p] = c;
          src[p] = s;
          off3[3 * p] = off[0];
          off3[3 * p + 1] = off[1];
          off3[3 * p + 2] = off[2];
          ++p;
        }
      }
  }
}

// near pairs: per leaf cell, the existing neighbours in (dx, dy, dz) order
__global__ void near_count_kernel(const long long* __restrict__ keys, long long n,
                                  const long long* __restrict__ cptr, long long* cnt) {
  for (long long a = blockIdx.x * (long long)blockDim.x + threadIdx.x; a < n; a += (long long)gridDim.x * blockDim.x) {
    long long cx, cy, cz;
    unpack(keys[a], cx, cy, cz);
    const long long na = cptr[a + 1] - cptr[a];
    long long k = 0;
    for (int q = 0; q < 27; ++q) {
      const long long x = cx + q / 9 - 1, y = cy + (q / 3) % 3 - 1, z = cz + q % 3 - 1;
      if (x < 0 || y < 0 || z < 0) continue;
      const long long b = find_key(keys, n, pack_key(x, y, z));
      if (b >= 0) k += na * (cptr[b + 1] - cptr[b]);
    }
    cnt[a] = k;
  }
}

// one block per leaf cell: its element pairs in row-major order per neighbour
__global__ void near_fill_kernel(const long long* __restrict__ keys, long long n, const long long* __restrict__ cptr,
                                 const int* __restrict__ celems, const long long* __restrict__ start,
                                 long long* ii, long long* jj) {
  const long long a = blockIdx.x;
  long long cx, cy, cz;
  unpack(keys[a], cx, cy, cz);
  const long long a0 = cptr[a], na = cptr[a + 1] - a0;
  long long p = start[a];
  for (int q = 0; q < 27; ++q) {
    const long long x = cx + q / 9 - 1, y = cy + (q / 3) % 3 - 1, z = cz + q % 3 - 1;
    if (x < 0 || y < 0 || z < 0) continue;
    const long long b = find_key(keys, n, pack_key(x, y, z));
    if (b < 0) continue;
    const long long b0 = cptr[b], nb = cptr[b + 1] - b0;
    for (long long t = threadIdx.x; t < na * nb; t += blockDim.x) {
      ii[p + t] = celems[a0 + t / nb];
      jj[p + t] = celems[b0 + t % nb];
    }
    p += na * nb;
  }
}

// numpy's np.linalg.norm of a 3-vector: sqrt((x*x + y*y) + z*z), no contraction
__device__ __forceinline__ double norm3(double x, double y, double z) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// marginal element pairs: per marginal interaction pair m, the (a in obs cell,
// b in src cell) with |c_a - c_b| <= reach, row-major; count pass then fill pass
__global__ void marginal_kernel(const long long* __restrict__ mobs, const long long* __restrict__ msrc, long long nm,
                                const long long* __restrict__ cptr, const int* __restrict__ celems,
                                const double* __restrict__ cen, double reach, const long long* __restrict__ start,
                                long long* cnt, long long* ii, long long* jj) {
  const long long m = blockIdx.x;
  if (m >= nm) return;
  const long long a0 = cptr[mobs[m]], na = cptr[mobs[m] + 1] - a0;
  const long long b0 = cptr[msrc[m]], nb = cptr[msrc[m] + 1] - b0;
  __shared__ long long base;
  __shared__ int warp_tot[32];
  if (threadIdx.x == 0) base = start ? start[m] : 0;
  __syncthreads();
  long long total = 0;
  for (long long t0 = 0; t0 < na * nb; t0 += blockDim.x) {
    const long long t = t0 + threadIdx.x;
    bool keep = false;
    long long ea = 0, eb = 0;
    if (t < na * nb) {
      ea = celems[a0 + t / nb];
      eb = celems[b0 + t % nb];
      const double d = norm3(__dsub_rn(cen[3 * ea], cen[3 * eb]), __dsub_rn(cen[3 * ea + 1], cen[3 * eb + 1]),
                             __dsub_rn(cen[3 * ea + 2], cen[3 * eb + 2]));
      keep = d <= reach;
    }
    // block-wide exclusive scan of keep, in thread order (= row-major order)
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      if (k < w) before += warp_tot[k];
      tot += warp_tot[k];
    }
    before += __popc(bal & ((1u << lane) - 1u));
    if (keep && ii) {
      ii[base + total + before] = ea;
      jj[base + total + before] = eb;
    }
    total += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0 && cnt) cnt[m] = total;
}

// copies on the library stream, waited for (the stream is non-blocking: a plain
// cudaMemcpy on the legacy stream would not wait for its kernels)
cudaError_t scopy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind, cudaStream_t st) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

template <class T>
int dalloc(tdw_ctx* ctx, T** p, size_t n) {
  TDW_CUDA(ctx, cudaMalloc(p, sizeof(T) * std::max<size_t>(1, n)));
  return TDW_OK;
}

template <class T>
int exclusive_scan(tdw_ctx* ctx, const T* in, T* out, int n, cudaStream_t st) {
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, st);
  void* t = nullptr;
  TDW_CUDA(ctx, cudaMalloc(&t, std::max<size_t>(1, tmp)));
  cub::DeviceScan::ExclusiveSum(t, tmp, in, out, n, st);
  TDW_CUDA(ctx, cudaGetLastError());
  TDW_CUDA(ctx, cudaStreamSynchronize(st));
  cudaFree(t);
  return TDW_OK;
}

}  // namespace

extern "C" {

int tdw_tree_build(tdw_ctx* ctx, int ns, const double* centroids, double rho, double c, double dt,
                   int leaf_capacity, int mu, int max_depth, int corrected, tdw_tree** out) {
  if (!ctx || !out || ns < 1 || !centroids || !(c > 0.0) || !(dt > 0.0) || leaf_capacity < 1 || max_depth < 0 ||
      max_depth > 20)
    return TDW_ERR_INVALID_ARG;
  *out = nullptr;
  cudaSetDevice(ctx->device);
  cudaStream_t st = ctx->stream;
  tdw_tree* T = new tdw_tree();
  T->ctx = ctx;
  T->ns = ns;
  std::vector<void*> dfree;
  auto cleanup = [&]() {
    for (void* p : dfree) cudaFree(p);
  };
  auto fail = [&](int code, const std::string& msg) {
    cleanup();
    delete T;
    return tdw_fail(ctx, code, msg);
  };
  // bounding box and root cell (host, the reference's expression order)
  double lo[3], hi[3];
  for (int k = 0; k < 3; ++k) { lo[k] = centroids[k]; hi[k] = centroids[k]; }
  for (int e = 1; e < ns; ++e)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], centroids[3 * e + k]);
      hi[k] = std::max(hi[k], centroids[3 * e + k]);
    }
  double ext = 0.0;
  for (int k = 0; k < 3; ++k) {
    T->centre[k] = 0.5 * (lo[k] + hi[k]);
    ext = std::max(ext, hi[k] - lo[k]);
  }
  T->root_half = 0.5 * ext * (1 + 1e-9) + 1e-12;
  const double blo[3] = {T->centre[0] - T->root_half, T->centre[1] - T->root_half, T->centre[2] - T->root_half};

  double* d_cen = nullptr;
  long long *d_keys = nullptr, *d_keys2 = nullptr;
  int *d_vals = nullptr, *d_vals2 = nullptr, *d_head = nullptr;
  int rc;
#define TREE_TRY(x) do { if ((rc = (x)) != TDW_OK) return fail(rc, ctx->err); } while (0)
  TREE_TRY(dalloc(ctx, &d_cen, 3 * (size_t)ns)); dfree.push_back(d_cen);
  TREE_TRY(dalloc(ctx, &d_keys, ns)); dfree.push_back(d_keys);
  TREE_TRY(dalloc(ctx, &d_keys2, ns)); dfree.push_back(d_keys2);
  TREE_TRY(dalloc(ctx, &d_vals, ns)); dfree.push_back(d_vals);
  TREE_TRY(dalloc(ctx, &d_vals2, ns)); dfree.push_back(d_vals2);
  TREE_TRY(dalloc(ctx, &d_head, ns)); dfree.push_back(d_head);
  if (scopy(d_cen, centroids, sizeof(double) * 3 * ns, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(TDW_ERR_CUDA, "tree: centroid upload");
  void* sort_tmp = nullptr;
  size_t sort_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, d_keys, d_keys2, d_vals, d_vals2, ns, 0, 3 * KSH, st);
  if (cudaMalloc(&sort_tmp, sort_bytes) != cudaSuccess) return fail(TDW_ERR_CUDA, "tree: sort scratch");
  dfree.push_back(sort_tmp);
  const int blocks = std::max(1, std::min(4096, (ns + 255) / 256));
  // stable key sort (radix sort is stable: equal keys keep ascending element order)
  auto sort_level = [&](std::vector<long long>& ukeys, std::vector<long long>& ecell) -> int {
    cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, d_keys, d_keys2, d_vals, d_vals2, ns, 0, 3 * KSH, st);
    heads_kernel<<<blocks, 256, 0, st>>>(d_keys2, ns, d_head);
    TDW_CUDA(ctx, cudaGetLastError());
    std::vector<long long> k(ns);
    std::vector<int> v(ns), h(ns);
    TDW_CUDA(ctx, cudaMemcpyAsync(k.data(), d_keys2, sizeof(long long) * ns, cudaMemcpyDeviceToHost, st));
    TDW_CUDA(ctx, cudaMemcpyAsync(v.data(), d_vals2, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    TDW_CUDA(ctx, cudaMemcpyAsync(h.data(), d_head, sizeof(int) * ns, cudaMemcpyDeviceToHost, st));
    TDW_CUDA(ctx, cudaStreamSynchronize(st));
    ukeys.clear();
    ecell.assign(ns, 0);
    for (int i = 0; i < ns; ++i) {
      if (h[i]) ukeys.push_back(k[i]);
      ecell[v[i]] = (long long)ukeys.size() - 1;
    }
    return TDW_OK;
  };
  // leaf depth: the first level whose fullest cell holds <= Z centroids
  int leaf = -1;
  std::vector<long long> ukeys, ecell;
  for (int L = 0; L <= max_depth && leaf < 0; ++L) {
    const long long n = 1LL << L;
    cell_coords_kernel<<<blocks, 256, 0, st>>>(d_cen, ns, blo[0], blo[1], blo[2], 2 * T->root_half / (double)n, n,
                                                d_keys, d_vals);
    if (cudaGetLastError() != cudaSuccess) return fail(TDW_ERR_CUDA, "tree: cell coordinates");
    TREE_TRY(sort_level(ukeys, ecell));
    std::vector<long long> cnt(ukeys.size(), 0);
    for (long long e : ecell) cnt[e]++;
    if (*std::max_element(cnt.begin(), cnt.end()) <= leaf_capacity) leaf = L;
  }
  if (leaf < 0) return fail(TDW_ERR_INVALID_ARG, "octree did not reach the leaf capacity");
  T->leaf = leaf;
  // leaf keys (the last pass ran at the leaf level), kept per element
  long long* d_leaf_keys = nullptr;
  TREE_TRY(dalloc(ctx, &d_leaf_keys, ns)); dfree.push_back(d_leaf_keys);
  {
    const long long n = 1LL << leaf;
    cell_coords_kernel<<<blocks, 256, 0, st>>>(d_cen, ns, blo[0], blo[1], blo[2], 2 * T->root_half / (double)n, n,
                                                d_leaf_keys, d_vals);
    if (cudaGetLastError() != cudaSuccess) return fail(TDW_ERR_CUDA, "tree: leaf coordinates");
  }
  T->coords.resize(leaf + 1);
  T->parent.resize(leaf + 1);
  T->elem_cell.resize(leaf + 1);
  T->il_obs.resize(leaf + 1);
  T->il_src.resize(leaf + 1);
  T->il_off.resize(leaf + 1);
  std::vector<std::vector<long long>> lkeys(leaf + 1);
  for (int L = 0; L <= leaf; ++L) {
    shift_keys_kernel<<<blocks, 256, 0, st>>>(d_leaf_keys, ns, leaf - L, d_keys, d_vals);
    if (cudaGetLastError() != cudaSuccess) return fail(TDW_ERR_CUDA, "tree: level keys");
    TREE_TRY(sort_level(lkeys[L], T->elem_cell[L]));
    const size_t n = lkeys[L].size();
    T->coords[L].resize(3 * n);
    const long long m = (1LL << KSH) - 1;
    for (size_t q = 0; q < n; ++q) {
      T->coords[L][3 * q] = (int)((lkeys[L][q] >> (2 * KSH)) & m);
      T->coords[L][3 * q + 1] = (int)((lkeys[L][q] >> KSH) & m);
      T->coords[L][3 * q + 2] = (int)(lkeys[L][q] & m);
    }
    if (L >= 1) {  // parents: coords >> 1 located in the coarser level (sorted keys)
      T->parent[L].resize(n);
      for (size_t q = 0; q < n; ++q) {
        const long long pk = pack_key(T->coords[L][3 * q] >> 1, T->coords[L][3 * q + 1] >> 1, T->coords[L][3 * q + 2] >> 1);
        T->parent[L][q] = std::lower_bound(lkeys[L - 1].begin(), lkeys[L - 1].end(), pk) - lkeys[L - 1].begin();
      }
    }
  }
  // interaction lists per level (L >= 2)
  for (int L = 2; L <= leaf; ++L) {
    const long long n = (long long)lkeys[L].size();
    long long* dk = nullptr;
    int* dcnt = nullptr;
    long long *dstart = nullptr, *dcnt64 = nullptr;
    TREE_TRY(dalloc(ctx, &dk, n)); dfree.push_back(dk);
    TREE_TRY(dalloc(ctx, &dcnt, n + 1)); dfree.push_back(dcnt);
    TREE_TRY(dalloc(ctx, &dcnt64, n + 1)); dfree.push_back(dcnt64);
    TREE_TRY(dalloc(ctx, &dstart, n + 1)); dfree.push_back(dstart);
    if (scopy(dk, lkeys[L].data(), sizeof(long long) * n, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: level keys upload");
    const int cb = (int)std::min<long long>(4096, (n + 127) / 128);
    il_count_kernel<<<cb, 128, 0, st>>>(dk, n, dcnt);
    std::vector<int> hc(n);
    if (scopy(hc.data(), dcnt, sizeof(int) * n, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: IL counts");
    std::vector<long long> hs(n + 1, 0);
    for (long long q = 0; q < n; ++q) hs[q + 1] = hs[q] + hc[q];
    const long long nil = hs[n];
    if (scopy(dstart, hs.data(), sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: IL offsets");
    long long *dobs = nullptr, *dsrc = nullptr;
    int* doff = nullptr;
    TREE_TRY(dalloc(ctx, &dobs, nil)); dfree.push_back(dobs);
    TREE_TRY(dalloc(ctx, &dsrc, nil)); dfree.push_back(dsrc);
    TREE_TRY(dalloc(ctx, &doff, 3 * nil)); dfree.push_back(doff);
    il_fill_kernel<<<cb, 128, 0, st>>>(dk, n, dstart, dobs, dsrc, doff);
    T->il_obs[L].resize(nil);
    T->il_src[L].resize(nil);
    T->il_off[L].resize(3 * nil);
    if (scopy(T->il_obs[L].data(), dobs, sizeof(long long) * nil, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        scopy(T->il_src[L].data(), dsrc, sizeof(long long) * nil, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        scopy(T->il_off[L].data(), doff, sizeof(int) * 3 * nil, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: IL download");
  }
  // leaf cell -> elements (ascending), on the device
  const long long nleaf = (long long)lkeys[leaf].size();
  std::vector<long long> cptr(nleaf + 1, 0);
  std::vector<int> celems(ns);
  for (long long e : T->elem_cell[leaf]) cptr[e + 1]++;
  for (long long q = 0; q < nleaf; ++q) cptr[q + 1] += cptr[q];
  {
    std::vector<long long> fill(cptr.begin(), cptr.end() - 1);
    for (int e = 0; e < ns; ++e) celems[fill[T->elem_cell[leaf][e]]++] = e;
  }
  long long *d_lk = nullptr, *d_cptr = nullptr;
  int* d_celems = nullptr;
  TREE_TRY(dalloc(ctx, &d_lk, nleaf)); dfree.push_back(d_lk);
  TREE_TRY(dalloc(ctx, &d_cptr, nleaf + 1)); dfree.push_back(d_cptr);
  TREE_TRY(dalloc(ctx, &d_celems, ns)); dfree.push_back(d_celems);
  if (scopy(d_lk, lkeys[leaf].data(), sizeof(long long) * nleaf, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      scopy(d_cptr, cptr.data(), sizeof(long long) * (nleaf + 1), cudaMemcpyHostToDevice, st) != cudaSuccess ||
      scopy(d_celems, celems.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return fail(TDW_ERR_CUDA, "tree: leaf cells upload");
  // near pairs of adjacent leaf cells
  {
    long long *dcnt = nullptr, *dstart = nullptr;
    TREE_TRY(dalloc(ctx, &dcnt, nleaf + 1)); dfree.push_back(dcnt);
    TREE_TRY(dalloc(ctx, &dstart, nleaf + 1)); dfree.push_back(dstart);
    const int cb = (int)std::min<long long>(4096, (nleaf + 127) / 128);
    near_count_kernel<<<cb, 128, 0, st>>>(d_lk, nleaf, d_cptr, dcnt);
    TDW_CUDA(ctx, cudaMemsetAsync(dcnt + nleaf, 0, sizeof(long long), st));
    TREE_TRY(exclusive_scan(ctx, dcnt, dstart, (int)(nleaf + 1), st));
    long long nnear = 0;
    if (scopy(&nnear, dstart + nleaf, sizeof(long long), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: near count");
    long long *dii = nullptr, *djj = nullptr;
    TREE_TRY(dalloc(ctx, &dii, nnear)); dfree.push_back(dii);
    TREE_TRY(dalloc(ctx, &djj, nnear)); dfree.push_back(djj);
    near_fill_kernel<<<(unsigned)nleaf, 256, 0, st>>>(d_lk, nleaf, d_cptr, d_celems, dstart, dii, djj);
    T->near_i.resize(nnear);
    T->near_j.resize(nnear);
    if (scopy(T->near_i.data(), dii, sizeof(long long) * nnear, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        scopy(T->near_j.data(), djj, sizeof(long long) * nnear, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: near download");
  }
  // causality check and marginal (extra) pairs per level, host arithmetic on the
  // pair lists in numpy's operation order; element pairs on the device
  for (int L = 2; L <= leaf; ++L) {
    const long long nil = (long long)T->il_obs[L].size();
    if (nil == 0) continue;
    const double side = 2 * T->root_half / (double)(1LL << L);
    const double interval = side / c;
    auto centre_of = [&](long long cell, int k) {
      return (T->centre[k] - T->root_half) + ((double)T->coords[L][3 * cell + k] + 0.5) * side;
    };
    double pmax = 0.0;
    for (long long p = 0; p < nil; ++p) {
      double s2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double dlt = centre_of(T->il_obs[L][p], k) - centre_of(T->il_src[L][p], k);
        s2 = s2 + dlt * dlt;
      }
      pmax = std::max(pmax, std::sqrt(s2));
    }
    const double dmax = pmax + std::sqrt(3.0) * side + 2 * rho;
    if (c * mu * interval <= dmax) {
      char buf[256];
      snprintf(buf, sizeof(buf), "level %d: interval gap mu=%d does not clear the farthest interaction pair "
               "(%.3f vs %.3f)", L, mu, dmax, c * mu * interval);
      return fail(TDW_ERR_INVALID_ARG, buf);
    }
    const double margin = corrected ? c * interval : c * (interval - dt);
    const double reach = corrected ? c * (interval + dt) + 2 * rho : c * interval + 2 * rho;
    std::vector<long long> mo, ms;
    for (long long p = 0; p < nil; ++p) {
      double s2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double g = std::max(std::abs((double)T->il_off[L][3 * p + k]) - 1.0, 0.0) * side;
        s2 = s2 + g * g;
      }
      if (std::sqrt(s2) - 2 * rho < margin) {
        mo.push_back(T->il_obs[L][p]);
        ms.push_back(T->il_src[L][p]);
      }
    }
    if (mo.empty()) continue;
    const long long nm = (long long)mo.size();
    const long long ncl = (long long)lkeys[L].size();
    std::vector<long long> lp(ncl + 1, 0);
    std::vector<int> le(ns);
    for (long long e : T->elem_cell[L]) lp[e + 1]++;
    for (long long q = 0; q < ncl; ++q) lp[q + 1] += lp[q];
    {
      std::vector<long long> fill(lp.begin(), lp.end() - 1);
      for (int e = 0; e < ns; ++e) le[fill[T->elem_cell[L][e]]++] = e;
    }
    long long *dmo = nullptr, *dms = nullptr, *dlp = nullptr, *dcnt = nullptr, *dstart = nullptr;
    int* dle = nullptr;
    TREE_TRY(dalloc(ctx, &dmo, nm)); dfree.push_back(dmo);
    TREE_TRY(dalloc(ctx, &dms, nm)); dfree.push_back(dms);
    TREE_TRY(dalloc(ctx, &dlp, ncl + 1)); dfree.push_back(dlp);
    TREE_TRY(dalloc(ctx, &dle, ns)); dfree.push_back(dle);
    TREE_TRY(dalloc(ctx, &dcnt, nm + 1)); dfree.push_back(dcnt);
    TREE_TRY(dalloc(ctx, &dstart, nm + 1)); dfree.push_back(dstart);
    if (scopy(dmo, mo.data(), sizeof(long long) * nm, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        scopy(dms, ms.data(), sizeof(long long) * nm, cudaMemcpyHostToDevice, st) != cudaSuccess ||
        scopy(dlp, lp.data(), sizeof(long long) * (ncl + 1), cudaMemcpyHostToDevice, st) != cudaSuccess ||
        scopy(dle, le.data(), sizeof(int) * ns, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: marginal upload");
    marginal_kernel<<<(unsigned)nm, 256, 0, st>>>(dmo, dms, nm, dlp, dle, d_cen, reach, nullptr, dcnt, nullptr,
                                                   nullptr);
    TDW_CUDA(ctx, cudaMemsetAsync(dcnt + nm, 0, sizeof(long long), st));
    TREE_TRY(exclusive_scan(ctx, dcnt, dstart, (int)(nm + 1), st));
    long long nx = 0;
    if (scopy(&nx, dstart + nm, sizeof(long long), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: marginal count");
    if (nx == 0) continue;
    long long *dii = nullptr, *djj = nullptr;
    TREE_TRY(dalloc(ctx, &dii, nx)); dfree.push_back(dii);
    TREE_TRY(dalloc(ctx, &djj, nx)); dfree.push_back(djj);
    marginal_kernel<<<(unsigned)nm, 256, 0, st>>>(dmo, dms, nm, dlp, dle, d_cen, reach, dstart, nullptr, dii, djj);
    T->extra_levels.push_back(L);
    T->extra_i.emplace_back(nx);
    T->extra_j.emplace_back(nx);
    if (scopy(T->extra_i.back().data(), dii, sizeof(long long) * nx, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        scopy(T->extra_j.back().data(), djj, sizeof(long long) * nx, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return fail(TDW_ERR_CUDA, "tree: marginal download");
  }
#undef TREE_TRY
  cleanup();
  *out = T;
  return TDW_OK;
}

// sizes: n_levels = leaf + 1; per level cells, IL length; near pairs; extra levels
int tdw_tree_info(const tdw_tree* T, int* leaf, double* centre3, double* root_half, int64_t* cells,
                  int64_t* nil, int64_t* n_near, int* n_extra) {
  if (!T) return TDW_ERR_INVALID_ARG;
  if (leaf) *leaf = T->leaf;
  if (centre3) memcpy(centre3, T->centre, sizeof(T->centre));
  if (root_half) *root_half = T->root_half;
  for (int L = 0; L <= T->leaf; ++L) {
    if (cells) cells[L] = (int64_t)(T->coords[L].size() / 3);
    if (nil) nil[L] = (int64_t)T->il_obs[L].size();
  }
  if (n_near) *n_near = (int64_t)T->near_i.size();
  if (n_extra) *n_extra = (int)T->extra_levels.size();
  return TDW_OK;
}

// level L: coords (n, 3), parent (n; L >= 1), elem_cell (ns), IL obs/src (nil), offsets (nil, 3)
int tdw_tree_level(const tdw_tree* T, int L, int64_t* coords, int64_t* parent, int64_t* elem_cell, int64_t* il_obs,
                   int64_t* il_src, int64_t* il_off) {
  if (!T || L < 0 || L > T->leaf) return TDW_ERR_INVALID_ARG;
  for (size_t q = 0; q < T->coords[L].size(); ++q) if (coords) coords[q] = T->coords[L][q];
  if (parent) for (size_t q = 0; q < T->parent[L].size(); ++q) parent[q] = T->parent[L][q];
  if (elem_cell) for (int e = 0; e < T->ns; ++e) elem_cell[e] = T->elem_cell[L][e];
  if (il_obs) for (size_t q = 0; q < T->il_obs[L].size(); ++q) il_obs[q] = T->il_obs[L][q];
  if (il_src) for (size_t q = 0; q < T->il_src[L].size(); ++q) il_src[q] = T->il_src[L][q];
  if (il_off) for (size_t q = 0; q < T->il_off[L].size(); ++q) il_off[q] = T->il_off[L][q];
  return TDW_OK;
}

int tdw_tree_near(const tdw_tree* T, int64_t* ii, int64_t* jj) {
  if (!T || !ii || !jj) return TDW_ERR_INVALID_ARG;
  memcpy(ii, T->near_i.data(), sizeof(int64_t) * T->near_i.size());
  memcpy(jj, T->near_j.data(), sizeof(int64_t) * T->near_j.size());
  return TDW_OK;
}

// extra pairs of the k-th extra level: *level, *n; ii/jj (nullable) filled when given
int tdw_tree_extra(const tdw_tree* T, int k, int* level, int64_t* n, int64_t* ii, int64_t* jj) {
  if (!T || k < 0 || k >= (int)T->extra_levels.size()) return TDW_ERR_INVALID_ARG;
  if (level) *level = T->extra_levels[k];
  if (n) *n = (int64_t)T->extra_i[k].size();
  if (ii) memcpy(ii, T->extra_i[k].data(), sizeof(int64_t) * T->extra_i[k].size());
  if (jj) memcpy(jj, T->extra_j[k].data(), sizeof(int64_t) * T->extra_j[k].size());
  return TDW_OK;
}

int tdw_tree_destroy(tdw_tree* T) {
  delete T;
  return TDW_OK;
}

}  // extern "C"
