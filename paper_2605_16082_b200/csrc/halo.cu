// Halo exchange support for partitioned runs: pack owned boundary columns / unpack ghost columns.
// Every device field is a stack of planes of `nt` doubles ([..][L][nt]); a halo message is
// [plane][i] for the listed columns, so pack/unpack are coalesced gathers/scatters per plane.
#include "ctx.cuh"

namespace pdg {
__global__ void k_pack(const double* __restrict__ src, long long nplanes, int nt, const int* __restrict__ idx, int n,
                       double* __restrict__ dst) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nplanes * n) return;
  const long long p = t / n;
  const int i = (int)(t - p * n);
  dst[t] = src[p * nt + idx[i]];
}
__global__ void k_unpack(const double* __restrict__ src, long long nplanes, int nt, const int* __restrict__ idx, int n,
                         double* __restrict__ dst) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nplanes * n) return;
  const long long p = t / n;
  const int i = (int)(t - p * n);
  dst[p * nt + idx[i]] = src[t];
}
}  // namespace pdg

using namespace pdg;
extern "C" {
int pdg_halo_pack(const double* field, long long nplanes, int nt, const int* idx, int n, double* buf, void* stream) {
  if (n == 0 || nplanes == 0) return PDG_OK;
  k_pack<<<nblocks(nplanes * n, 256), 256, 0, (cudaStream_t)stream>>>(field, nplanes, nt, idx, n, buf);
  return check_launch_noctx();
}
int pdg_halo_unpack(const double* buf, long long nplanes, int nt, const int* idx, int n, double* field, void* stream) {
  if (n == 0 || nplanes == 0) return PDG_OK;
  k_unpack<<<nblocks(nplanes * n, 256), 256, 0, (cudaStream_t)stream>>>(buf, nplanes, nt, idx, n, field);
  return check_launch_noctx();
}
}  // extern "C"
