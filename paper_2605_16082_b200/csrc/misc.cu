// Small elementwise entries of the drop-in API (EOS, mass pattern helpers).
#include "ctx.cuh"

namespace pdg {
// linear EOS, external2d.py:81-87: rho' = -alpha (T - t_ref) [+ beta (S - s_ref)]
__global__ void k_eos(const double* __restrict__ T, const double* __restrict__ S, long long n, double alpha,
                      double beta, double tref, double sref, double* __restrict__ out) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double r = -alpha * (T[i] - tref);
  if (beta != 0.0) r = r + beta * ((S ? S[i] : sref) - sref);
  out[i] = r;
}
}  // namespace pdg

using namespace pdg;
extern "C" int pdg_eos(const double* T, const double* S, long long n, double alpha, double beta, double tref,
                       double sref, double* out, void* stream) {
  k_eos<<<nblocks(n, 256), 256, 0, (cudaStream_t)stream>>>(T, S, n, alpha, beta, tref, sref, out);
  return check_launch_noctx();
}
