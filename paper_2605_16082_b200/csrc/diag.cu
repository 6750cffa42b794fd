// Device-resident diagnostics of the stepper state: diagnostics_2d (external2d.py:366-380) and
// budget_3d (internal3d.py:942-951) of the current fields in one fused pass over the columns,
// with a deterministic two-level reduction (block partials in a fixed tree order, then one block
// over the partials in index order), so a long run can be monitored with an 80-byte read-back.
//
// out[0] 2D volume        sum Mh (eta - b)            (integrate_nodal)
// out[1] 2D energy        sum_q J2D QW (g eta^2 / 2 + |Q|^2 / (2 h))
// out[2] eta min          out[3] eta max
// out[4] 3D volume        sum 1^T M 1                 (integrate_prism, M on the current grid)
// out[5] momentum x       sum 1^T M u_x               out[6] momentum y
// out[7] tracer mass      sum 1^T M T                 out[8] T min   out[9] T max
#include <cfloat>

#include "col3d.cuh"
#include "ctx.cuh"

namespace pdg {

constexpr int DG_N = 10;
constexpr int DG_BS = 256;

__global__ void __launch_bounds__(DG_BS) k_diag_partial(DMesh m, const double* __restrict__ S,
                                                        const double* __restrict__ u, const double* __restrict__ T,
                                                        double g, double* __restrict__ part) {
  const int nt = m.nt, L = m.L, t = threadIdx.x;
  const size_t P6 = (size_t)6 * L * nt;
  double acc[DG_N] = {0, 0, DBL_MAX, -DBL_MAX, 0, 0, 0, 0, DBL_MAX, -DBL_MAX};
  for (int c = blockIdx.x * DG_BS + t; c < m.nown; c += gridDim.x * DG_BS) {
    const double j2d = __ldg(m.j2d + c);
    double e[3], x[3], y[3], b[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      e[k] = __ldg(S + (size_t)k * nt + c);
      x[k] = __ldg(S + (size_t)(3 + k) * nt + c);
      y[k] = __ldg(S + (size_t)(6 + k) * nt + c);
      b[k] = __ldg(m.b + (size_t)k * nt + c);
      acc[2] = fmin(acc[2], e[k]);
      acc[3] = fmax(acc[3], e[k]);
    }
    {
      const double h3[3] = {e[0] - b[0], e[1] - b[1], e[2] - b[2]};
      double mh[3];
      mh_apply3(h3, j2d, mh);
      acc[0] += (mh[0] + mh[1]) + mh[2];
      double hq6[6], eq[6], xq[6], yq[6];
      hq(h3, hq6);
      hq(e, eq);
      hq(x, xq);
      hq(y, yq);
      double en = 0.0;
#pragma unroll
      for (int q = 0; q < 6; ++q)
        en += j2d * (0.5 * g * eq[q] * eq[q] + 0.5 * (xq[q] * xq[q] + yq[q] * yq[q]) / hq6[q]) * QW[q];
      acc[1] += en;
    }
    // 1^T (K (x) J2D Mjz) f = J2D sum_lev sum_b (MHQ jz)_b f[lev][b]   (sum_a K = 1, sum_a BARY_a = 1)
    for (int l = 0; l < L; ++l) {
      double jz[3], w[3];
      layer_jz(b, e, m.fracs[l], m.fracs[l + 1], jz);
      mhq_vec(jz, w);
      const double v1 = j2d * ((w[0] + w[1]) + w[2]);
      acc[4] += 2.0 * v1;
#pragma unroll
      for (int lev = 0; lev < 2; ++lev)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const size_t o = ((size_t)(3 * lev + k) * L + l) * nt + c;
          const double wk = j2d * w[k];
          const double tv = __ldg(T + o);
          acc[5] += wk * __ldg(u + o);
          acc[6] += wk * __ldg(u + P6 + o);
          acc[7] += wk * tv;
          acc[8] = fmin(acc[8], tv);
          acc[9] = fmax(acc[9], tv);
        }
    }
  }
  __shared__ double red[DG_N][DG_BS];
#pragma unroll
  for (int i = 0; i < DG_N; ++i) red[i][t] = acc[i];
  __syncthreads();
  for (int s = DG_BS / 2; s > 0; s >>= 1) {
    if (t < s) {
#pragma unroll
      for (int i = 0; i < DG_N; ++i) {
        const double a = red[i][t], o = red[i][t + s];
        red[i][t] = (i == 2 || i == 8) ? fmin(a, o) : (i == 3 || i == 9) ? fmax(a, o) : a + o;
      }
    }
    __syncthreads();
  }
  if (t < DG_N) part[(size_t)blockIdx.x * DG_N + t] = red[t][0];
}

__global__ void k_diag_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  const int i = threadIdx.x;
  if (i >= DG_N) return;
  double a = (i == 2 || i == 8) ? DBL_MAX : (i == 3 || i == 9) ? -DBL_MAX : 0.0;
  for (int k = 0; k < nb; ++k) {
    const double v = part[(size_t)k * DG_N + i];
    a = (i == 2 || i == 8) ? fmin(a, v) : (i == 3 || i == 9) ? fmax(a, v) : a + v;
  }
  out[i] = a;
}

}  // namespace pdg

using namespace pdg;

extern "C" {

int pdg_step_diagnostics(pdg_ctx* ctx, const double* S, const double* u, const double* T, double g, double* work,
                         double* out, void* stream) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  const int nb = nsm * 4;   // fixed grid: the reduction order does not depend on the column count
  cudaStream_t s = (cudaStream_t)stream;
  k_diag_partial<<<nb, DG_BS, 0, s>>>(ctx->view(), S, u, T, g, work);
  if (check_launch(ctx)) return PDG_ERR_CUDA;
  k_diag_final<<<1, 32, 0, s>>>(work, nb, out);
  return check_launch(ctx);
}

int pdg_diagnostics_work_doubles(pdg_ctx* ctx) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  return nsm * 4 * DG_N;
}

}  // extern "C"
