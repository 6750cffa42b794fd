// Domain decomposition on the device (host restatement paper_2605_16082_b200/
// partition.py decompose, independent checker oracle/partition.py): the O(nt) parts -- the
// prism-weight prefix sum and its split points, and the ghost-ring breadth-first search of each
// rank -- run here; the host only segments the (small) ghost lists by owner into send / recv maps.
// Every output is an integer map, bit-exact with the host restatement (tests/test_partition_gpu.py).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace pdg {

// first k with cum[k] * P >= t (numpy searchsorted(cum * P, t, side="left")), one thread per split
__global__ void k_split_search(const long long* __restrict__ cum, int n, int P, long long* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x + 1;   // split k = 1 .. P-1
  if (k >= P) return;
  const long long W = cum[n - 1];
  const long long t = (long long)k * W;
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (cum[mid] * (long long)P < t)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[k - 1] = lo;
}

__global__ void k_level_init(int nt, int lo, int hi, int* __restrict__ level) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < nt) level[c] = (c >= lo && c < hi) ? 0 : -1;
}

// ring k+1 = edge neighbours of ring k that are not local yet.  Every write in one launch stores
// the same value k + 1 and only into columns still at -1, so the concurrent writes are benign and
// the result does not depend on thread order.
__global__ void k_ring(int nt, const int* __restrict__ nbr, int k, int* __restrict__ level) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nt || level[c] != k) return;
#pragma unroll
  for (int e = 0; e < 3; ++e) {
    const int j = nbr[e * nt + c];
    if (j >= 0 && level[j] < 0) level[j] = k + 1;
  }
}

struct IsGhost {
  const int* level;
  __device__ bool operator()(int c) const { return level[c] >= 1; }
};

__global__ void k_iota(int n, int* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = i;
}
__global__ void k_gather_level(int n, const int* __restrict__ ids, const int* __restrict__ level,
                               int* __restrict__ ring) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ring[i] = level[ids[i]];
}

}  // namespace pdg

using namespace pdg;

extern "C" {

// split_ranges (partition.py): raw split points k = 1..P-1 of the prism-weight prefix sum; the
// host applies the non-empty / capacity clamps (a sequential dependency on the previous bound).
// w: DEVICE int64 weights [n]; raw: HOST [P-1]
int pdg_split_search(const long long* w, int n, int P, long long* raw, void* stream) {
  if (n <= 0 || P < 1) return PDG_ERR_SHAPE;
  if (P == 1) return PDG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  long long *cum = nullptr, *out = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  if (cudaMallocAsync(&cum, n * sizeof(long long), s) || cudaMallocAsync(&out, (P - 1) * sizeof(long long), s))
    return PDG_ERR_CUDA;
  cub::DeviceScan::InclusiveSum(nullptr, tb, w, cum, n, s);
  if (cudaMallocAsync(&tmp, tb, s)) return PDG_ERR_CUDA;
  cub::DeviceScan::InclusiveSum(tmp, tb, w, cum, n, s);
  k_split_search<<<nblocks(P - 1, 128), 128, 0, s>>>(cum, n, P, out);
  cudaMemcpyAsync(raw, out, (P - 1) * sizeof(long long), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(cum, s);
  cudaFreeAsync(out, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return PDG_ERR_CUDA;
  return check_launch_noctx();
}

// ghost rings of the owned range [lo, hi) of the context's mesh, `depth` rings: ghost global ids
// in ascending order and the ring (1..depth) of each.  ghosts / rings: DEVICE, capacity nt - (hi - lo);
// n_ghosts: HOST.
int pdg_partition_rings(pdg_ctx* ctx, int lo, int hi, int depth, int* ghosts, int* rings, int* n_ghosts,
                        void* stream) {
  const int nt = ctx->nt;
  if (lo < 0 || hi > nt || lo >= hi || depth < 0) return PDG_ERR_SHAPE;
  cudaStream_t s = (cudaStream_t)stream;
  int *level = nullptr, *ids = nullptr, *cnt = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  if (cudaMallocAsync(&level, nt * sizeof(int), s) || cudaMallocAsync(&ids, nt * sizeof(int), s) ||
      cudaMallocAsync(&cnt, sizeof(int), s))
    return PDG_ERR_CUDA;
  const int nb = nblocks(nt, 256);
  k_level_init<<<nb, 256, 0, s>>>(nt, lo, hi, level);
  for (int k = 0; k < depth; ++k) k_ring<<<nb, 256, 0, s>>>(nt, ctx->nbr, k, level);
  k_iota<<<nb, 256, 0, s>>>(nt, ids);
  IsGhost pred{level};
  cub::DeviceSelect::If(nullptr, tb, ids, ghosts, cnt, nt, pred, s);
  if (cudaMallocAsync(&tmp, tb, s)) return PDG_ERR_CUDA;
  cub::DeviceSelect::If(tmp, tb, ids, ghosts, cnt, nt, pred, s);   // stable: ascending global ids
  int n = 0;
  cudaMemcpyAsync(&n, cnt, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (cudaStreamSynchronize(s) != cudaSuccess) return PDG_ERR_CUDA;
  if (n > 0) k_gather_level<<<nblocks(n, 256), 256, 0, s>>>(n, ghosts, level, rings);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(level, s);
  cudaFreeAsync(ids, s);
  cudaFreeAsync(cnt, s);
  *n_ghosts = n;
  return check_launch(ctx);
}

}  // extern "C"
