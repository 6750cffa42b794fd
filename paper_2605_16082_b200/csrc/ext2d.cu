// 2D external mode: fused free-surface + depth-momentum residuals, Mh^-1 and the SSP-RK3
// stage update in ONE thread-per-triangle kernel (external2d.py:128-353).
//
// Gather-only: a triangle reads its neighbours' edge-node values and computes its own copy
// of every edge flux (mirrored quadrature order, dg.py:69-75), so no atomics or colouring
// are needed and results do not depend on the partition of columns across threads/GPUs.
// HBM traffic per triangle per stage: state 72 B (+ neighbour values, L2 hits under the
// Hilbert order) + base state 72 B + geometry 188 B + forcing 48 B + write 72 B.
#include "ctx.cuh"

namespace pdg {

struct Ext2DIn {
  const double *eta, *qx, *qy;  // C3 state evaluated
  const double* f3d2d;          // [2][3][nt] or null
  const double* source;         // C3 or null
  const double* patm;           // C3 or null
  int has_bc;
  double eta_bc, g, rho0;
};

// residuals (before Mh^-1) of the free-surface and depth-momentum equations for column c
template <class ColT, bool FAST = false>
__device__ __forceinline__ void ext2d_residual(const DMesh& m, const ColT& C, int c, const Ext2DIn& a,
                                               double re[3], double rx[3], double ry[3],
                                               double* own = nullptr) {  // optional: the own state [3][3]
  const int nt = m.nt;
  const double g = a.g;
  double e[3], x[3], y[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    e[i] = __ldg(a.eta + i * nt + c);
    x[i] = __ldg(a.qx + i * nt + c);
    y[i] = __ldg(a.qy + i * nt + c);
  }
  if (own) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      own[i] = e[i];
      own[3 + i] = x[i];
      own[6 + i] = y[i];
    }
  }
  // ---- volume terms (external2d.py:145-148, 204-218)
  double xq = 0.0, yq = 0.0;
  {
    double tx[6], ty[6];
    hq(x, tx);
    hq(y, ty);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      xq += tx[q] * QW[q];
      yq += ty[q] * QW[q];
    }
  }
  const double j2d = C.j2d;
#pragma unroll
  for (int i = 0; i < 3; ++i) re[i] = j2d * (C.dx[i] * xq + C.dy[i] * yq);
  const double gx = (e[0] * C.dx[0] + e[1] * C.dx[1]) + e[2] * C.dx[2];
  const double gy = (e[0] * C.dy[0] + e[1] * C.dy[1]) + e[2] * C.dy[2];
  double hphi[3] = {0.0, 0.0, 0.0};
  {
    double h3[3] = {e[0] - C.b[0], e[1] - C.b[1], e[2] - C.b[2]};
    double hqv[6];
    hq(h3, hqv);
    double hmin = hqv[0];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      hmin = fmin(hmin, hqv[q]);
      const double w = hqv[q] * QW[q];
#pragma unroll
      for (int i = 0; i < 3; ++i) hphi[i] += w * BARY[q][i];
    }
    if (hmin <= 0.0) report(m.err, PDG_ERR_DRY, c, 0, hmin);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    rx[i] = -(g * j2d * gx * hphi[i]);
    ry[i] = -(g * j2d * gy * hphi[i]);
  }
  if (a.patm) {
    double pa[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) pa[i] = a.patm[i * nt + c];
    const double px = (pa[0] * C.dx[0] + pa[1] * C.dx[1]) + pa[2] * C.dx[2];
    const double py = (pa[0] * C.dy[0] + pa[1] * C.dy[1]) + pa[2] * C.dy[2];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rx[i] -= j2d * px * hphi[i] / a.rho0;
      ry[i] -= j2d * py * hphi[i] / a.rho0;
    }
  }
  // ---- edges (external2d.py:150-180, 220-251)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int v0 = EV0(k), v1 = EV1(k);
    const double nx = C.nx[k], ny = C.ny[k];
    double ei[2], xi[2], yi[2], bi[2], ee[2], xe[2], ye[2], be[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      ei[h] = e[v0] * ES[h][0] + e[v1] * ES[h][1];
      xi[h] = x[v0] * ES[h][0] + x[v1] * ES[h][1];
      yi[h] = y[v0] * ES[h][0] + y[v1] * ES[h][1];
      bi[h] = C.b[v0] * ES[h][0] + C.b[v1] * ES[h][1];
    }
    if (C.tag[k] == 0) {
      const int e2 = C.nb[k], k2 = C.nk[k];
      const int n0 = EV0(k2) * nt + e2, n1 = EV1(k2) * nt + e2;
      const double ea = __ldg(a.eta + n0), eb = __ldg(a.eta + n1), xa = __ldg(a.qx + n0), xb = __ldg(a.qx + n1);
      const double ya = __ldg(a.qy + n0), yb = __ldg(a.qy + n1), ba = ldg(m.b + n0), bb = ldg(m.b + n1);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ee[h] = ea * ES[h][1] + eb * ES[h][0];
        xe[h] = xa * ES[h][1] + xb * ES[h][0];
        ye[h] = ya * ES[h][1] + yb * ES[h][0];
        be[h] = ba * ES[h][1] + bb * ES[h][0];
      }
    } else if (C.tag[k] == 2) {  // open: prescribed (or interior) level, transparent transport
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        ee[h] = a.has_bc ? a.eta_bc : ei[h];
        xe[h] = xi[h];
        ye[h] = yi[h];
        be[h] = bi[h];
      }
    } else {  // wall: mirror the normal transport
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double qn = nx * xi[h] + ny * yi[h];
        ee[h] = ei[h];
        xe[h] = xi[h] - 2.0 * qn * nx;
        ye[h] = yi[h] - 2.0 * qn * ny;
        be[h] = bi[h];
      }
    }
    const double je = 0.5 * C.el[k];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const double hi = ei[h] - bi[h], he = ee[h] - be[h];
      if (hi <= 0.0 || he <= 0.0) report(m.err, PDG_ERR_DRY, -1, 0, fmin(hi, he));
      const double cel = FAST ? dsqrt_bf(g * fmax(hi, he)) : sqrt(g * fmax(hi, he));  // max(sqrt(g h))
      const double fe = nx * 0.5 * (xi[h] + xe[h]) + ny * 0.5 * (yi[h] + ye[h]) + cel * 0.5 * (ei[h] - ee[h]);
      const double hm = 0.5 * (hi + he);
      const double de = 0.5 * (ei[h] - ee[h]);
      const double fx = -(g * nx * hm * de) + cel * 0.5 * (xi[h] - xe[h]);
      const double fy = -(g * ny * hm * de) + cel * 0.5 * (yi[h] - ye[h]);
      const double we = je * fe, wx = je * fx, wy = je * fy;
      re[v0] -= we * ES[h][0];
      re[v1] -= we * ES[h][1];
      rx[v0] -= wx * ES[h][0];
      rx[v1] -= wx * ES[h][1];
      ry[v0] -= wy * ES[h][0];
      ry[v1] -= wy * ES[h][1];
    }
  }
  if (a.f3d2d) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      rx[i] += __ldg(a.f3d2d + i * nt + c);
      ry[i] += __ldg(a.f3d2d + (3 + i) * nt + c);
    }
  }
  if (a.source) {
    double s[3], ms[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) s[i] = a.source[i * nt + c];
    mh_apply3(s, j2d, ms);
#pragma unroll
    for (int i = 0; i < 3; ++i) re[i] += ms[i];
  }
}

__global__ void k_ext2d_eval(DMesh m, Ext2DIn a, const int* __restrict__ els, int n, int mode,
                             double* __restrict__ oe, double* __restrict__ ox, double* __restrict__ oy) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = els ? els[i] : i;
  Col C;
  load_col(m, c, C);
  double re[3], rx[3], ry[3];
  ext2d_residual(m, C, c, a, re, rx, ry);
  if (mode == 0) {
    if (C.j2d <= 0.0) report(m.err, PDG_ERR_SINGULAR_MASS, c, 0, C.j2d);
    double t[3];
    mh_inv3(re, C.j2d, t);
#pragma unroll
    for (int k = 0; k < 3; ++k) re[k] = t[k];
    mh_inv3(rx, C.j2d, t);
#pragma unroll
    for (int k = 0; k < 3; ++k) rx[k] = t[k];
    mh_inv3(ry, C.j2d, t);
#pragma unroll
    for (int k = 0; k < 3; ++k) ry[k] = t[k];
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    oe[k * n + i] = re[k];
    ox[k * n + i] = rx[k];
    oy[k * n + i] = ry[k];
  }
}

// one SSP-RK3 stage: X = state evaluated, S0 = substep start (3 fields x C3), Y = output.
// STAGE 0: Y = S0 + dt d(X);  1: Y = 3/4 S0 + 1/4 (X + dt d);  2: Y = S0/3 + 2/3 (X + dt d), qbar += Y.q
// els (optional): the columns to update (partitioned runs split owned columns into those next to
// ghost columns and the interior, so the halo exchange overlaps the interior update)
// PDL: programmatic dependent launch -- the next stage's blocks may start while this grid drains;
// they load the (static) geometry, then wait (griddepcontrol.wait) for this grid's results
template <int STAGE, int BS = 256, int MINB = 2, bool PDL = false>
__global__ void __launch_bounds__(BS, MINB) k_rk_stage(DMesh m, Ext2DIn a, const double* S0,
                                                     double* Y, double dt, double* __restrict__ qbar,
                                                     const int* __restrict__ els = nullptr, int n_els = 0) {
  if constexpr (PDL) asm volatile("griddepcontrol.launch_dependents;");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = m.nt;
  if (i >= (els ? n_els : m.nown)) return;
  const int c = els ? els[i] : i;
  Col2 C;
  if constexpr (PDL) {
    load_col2(m, c, C);
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  // issue the substep-start and Qbar loads first: they are independent of the flux work below,
  // so their latency overlaps it instead of being exposed at the end (stages 1, 2)
  double s0[3][3], qb[2][3];
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int k = 0; k < 3; ++k)
      s0[f][k] = STAGE == 0 ? 0.0 : STAGE == 1 ? __ldg(S0 + (size_t)(f * 3 + k) * nt + c) : S0[(size_t)(f * 3 + k) * nt + c];
  if (STAGE == 2) {
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int k = 0; k < 3; ++k) qb[f][k] = qbar[(size_t)(f * 3 + k) * nt + c];
  }
  if constexpr (!PDL) load_col2(m, c, C);
  double r[3][3], xo[9];
  ext2d_residual<Col2, true>(m, C, c, a, r[0], r[1], r[2], xo);
  const double* X = nullptr;
  (void)X;
  const double f6 = 6.0 * drcp(C.j2d);
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double d[3];
    mh_inv3f(r[f], f6, d);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const size_t o = (size_t)(f * 3 + k) * nt + c;
      double y;
      if (STAGE == 0) {
        y = xo[f * 3 + k] + dt * d[k];   // X == S0
      } else if (STAGE == 1) {
        y = 0.75 * s0[f][k] + 0.25 * (xo[f * 3 + k] + dt * d[k]);
      } else {
        y = s0[f][k] * (1.0 / 3.0) + (2.0 / 3.0) * (xo[f * 3 + k] + dt * d[k]);
      }
      Y[o] = y;
      if (STAGE == 2 && f > 0) qbar[(size_t)((f - 1) * 3 + k) * nt + c] = qb[f - 1][k] + y;
    }
  }
}

// qbar /= m;  f2d = (Q_end - Q0)/(m dt) - Mh^-1 f3d2d   (external2d.py:343-352)
__global__ void k_subcycle_final(DMesh m, const double* __restrict__ S, const double* __restrict__ q0,
                                 const double* __restrict__ f3d2d, int msub, double dtfull, double* __restrict__ qbar,
                                 double* __restrict__ f2d) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int nt = m.nt;
  if (c >= m.nown) return;
  const double j2d = m.j2d[c];
#pragma unroll
  for (int comp = 0; comp < 2; ++comp) {
    double fm[3] = {0.0, 0.0, 0.0};
    if (f3d2d) {
      double v[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) v[k] = f3d2d[(comp * 3 + k) * nt + c];
      mh_inv3(v, j2d, fm);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const size_t o = (size_t)(comp * 3 + k) * nt + c;
      qbar[o] = qbar[o] / (double)msub;
      double f = (S[(size_t)((1 + comp) * 3 + k) * nt + c] - q0[o]) / dtfull;
      if (f3d2d) f = f - fm[k];
      f2d[o] = f;
    }
  }
}

// check_cfl (external2d.py:271-283): block partials of (min H, argmin column, max H)
__global__ void k_cfl_partial(DMesh m, const double* __restrict__ eta, double* __restrict__ part) {
  __shared__ double smin[256], smax[256];
  __shared__ long long sarg[256];
  const int nt = m.nt;
  double mn = 1e300, mx = -1e300;
  long long arg = 0x7fffffffffffffffLL;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < m.nown; c += gridDim.x * blockDim.x) {
    double rowmin = 1e300;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double h = eta[k * nt + c] - m.b[k * nt + c];
      rowmin = fmin(rowmin, h);
      mx = fmax(mx, h);
    }
    if (rowmin < mn || (rowmin == mn && c < arg)) {
      mn = rowmin;
      arg = c;
    }
  }
  smin[threadIdx.x] = mn;
  smax[threadIdx.x] = mx;
  sarg[threadIdx.x] = arg;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const int o = threadIdx.x + s;
      if (smin[o] < smin[threadIdx.x] || (smin[o] == smin[threadIdx.x] && sarg[o] < sarg[threadIdx.x])) {
        smin[threadIdx.x] = smin[o];
        sarg[threadIdx.x] = sarg[o];
      }
      smax[threadIdx.x] = fmax(smax[threadIdx.x], smax[o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[3 * blockIdx.x] = smin[0];
    part[3 * blockIdx.x + 1] = (double)sarg[0];
    part[3 * blockIdx.x + 2] = smax[0];
  }
}

__global__ void k_cfl_final(DMesh m, const double* __restrict__ part, int nb, double g, double dt, double min_edge,
                            double* ratio) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double mn = 1e300, mx = -1e300, arg = 0;
  for (int i = 0; i < nb; ++i) {
    if (part[3 * i] < mn || (part[3 * i] == mn && part[3 * i + 1] < arg)) {
      mn = part[3 * i];
      arg = part[3 * i + 1];
    }
    mx = fmax(mx, part[3 * i + 2]);
  }
  if (mn <= 0.0) {
    report(m.err, PDG_ERR_DRY, (long long)arg, 0, mn);
    if (ratio) ratio[0] = 0.0;
    return;
  }
  const double r = dt * sqrt(g * mx) / min_edge;
  if (ratio) ratio[0] = r;
  if (r > 1.0 / 3.0) report(m.err, PDG_ERR_CFL, 0, 0, r);
}

__global__ void k_apply_mh(const double* __restrict__ v, const double* __restrict__ j2d, int n, int nc, int inverse,
                           double* __restrict__ out, pdg_err* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double j = j2d[i];
  if (inverse && j <= 0.0) report(err, PDG_ERR_SINGULAR_MASS, i, 0, j);
  for (int c = 0; c < nc; ++c) {
    double x[3], y[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) x[k] = v[(size_t)(c * 3 + k) * n + i];
    if (inverse)
      mh_inv3(x, j, y);
    else
      mh_apply3(x, j, y);
#pragma unroll
    for (int k = 0; k < 3; ++k) out[(size_t)(c * 3 + k) * n + i] = y[k];
  }
}

}  // namespace pdg

using namespace pdg;

static int run_cfl(pdg_ctx* ctx, const double* eta, double g, double dt, double* ratio, cudaStream_t s) {
  DMesh m = ctx->view();
  const int nb = 128;
  k_cfl_partial<<<nb, 256, 0, s>>>(m, eta, ctx->red);
  if (check_launch(ctx)) return PDG_ERR_CUDA;
  k_cfl_final<<<1, 32, 0, s>>>(m, ctx->red, nb, g, dt, ctx->min_edge, ratio);
  return check_launch(ctx);
}

extern "C" {

int pdg_ext2d_eval(pdg_ctx* ctx, const double* eta, const double* qx, const double* qy, const double* f3d2d,
                   const double* source, const double* patm, int has_bc, double eta_bc, double g, double rho0,
                   const int* els, int n_els, int mode, double* oe, double* ox, double* oy, void* stream) {
  cudaSetDevice(ctx->device);
  Ext2DIn a{eta, qx, qy, f3d2d, source, patm, has_bc, eta_bc, g, rho0};
  const int n = els ? n_els : ctx->nown;
  if (n == 0) return PDG_OK;
  k_ext2d_eval<<<nblocks(n, 128), 128, 0, (cudaStream_t)stream>>>(ctx->view(), a, els, n, mode, oe, ox, oy);
  return check_launch(ctx);
}

int pdg_ext2d_cfl(pdg_ctx* ctx, const double* eta, double g, double dt, double* ratio_dev, void* stream) {
  cudaSetDevice(ctx->device);
  return run_cfl(ctx, eta, g, dt, ratio_dev, (cudaStream_t)stream);
}

int pdg_ext2d_subcycle(pdg_ctx* ctx, double* S, int msub, double dt, double g, double rho0, const double* f3d2d,
                       const double* source, const double* patm, const double* bc_vals, double* qbar, double* f2d,
                       int check_cfl, void* stream) {
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = ctx->nt;
  DMesh m = ctx->view();
  if (check_cfl && run_cfl(ctx, S, g, dt, ctx->red + 4000, s)) return PDG_ERR_CUDA;
  double* W1 = ctx->ws2d;
  double* W2 = W1 + (size_t)9 * nt;
  double* q0 = W2 + (size_t)9 * nt;
  if (cudaMemcpyAsync(q0, S + (size_t)3 * nt, (size_t)6 * nt * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return PDG_ERR_CUDA;
  if (cudaMemsetAsync(qbar, 0, (size_t)6 * nt * sizeof(double), s) != cudaSuccess) return PDG_ERR_CUDA;
  const int variant = tune_get(TUNE_RK);
  const int bs = variant == 2 || variant == 3 || variant == 5 || variant == 6 || variant == 8 ? 128 : 256,
            nb = nblocks(ctx->nown, bs);
  // variant 8: as 2, with programmatic dependent launch between the stage kernels
  auto pdl = [&](auto kern, auto... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(bs);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, args...);
  };
#define RK_LAUNCH(ST, ...)                                                              \
  switch (variant) {                                                                    \
    case 8: pdl(k_rk_stage<ST, 128, 4, true>, __VA_ARGS__, (const int*)nullptr, 0); break; \
    case 2: k_rk_stage<ST, 128, 4><<<nb, bs, 0, s>>>(__VA_ARGS__); break;               \
    case 3: k_rk_stage<ST, 128, 3><<<nb, bs, 0, s>>>(__VA_ARGS__); break;               \
    case 4: k_rk_stage<ST, 256, 1><<<nb, bs, 0, s>>>(__VA_ARGS__); break;               \
    case 5: k_rk_stage<ST, 128, 6><<<nb, bs, 0, s>>>(__VA_ARGS__); break;               \
    case 6: k_rk_stage<ST, 128, 8><<<nb, bs, 0, s>>>(__VA_ARGS__); break;               \
    default: k_rk_stage<ST, 256, 2><<<nb, bs, 0, s>>>(__VA_ARGS__); break;              \
  }
  for (int it = 0; it < msub; ++it) {
    const int hb = bc_vals != nullptr;
    Ext2DIn a{S, S + (size_t)3 * nt, S + (size_t)6 * nt, f3d2d, source, patm, hb, hb ? bc_vals[3 * it] : 0.0, g, rho0};
    RK_LAUNCH(0, m, a, S, W1, dt, qbar)
    if (check_launch(ctx)) return PDG_ERR_CUDA;
    Ext2DIn a1{W1, W1 + (size_t)3 * nt, W1 + (size_t)6 * nt, f3d2d, source, patm, hb,
               hb ? bc_vals[3 * it + 1] : 0.0, g, rho0};
    RK_LAUNCH(1, m, a1, S, W2, dt, qbar)
    if (check_launch(ctx)) return PDG_ERR_CUDA;
    Ext2DIn a2{W2, W2 + (size_t)3 * nt, W2 + (size_t)6 * nt, f3d2d, source, patm, hb,
               hb ? bc_vals[3 * it + 2] : 0.0, g, rho0};
    RK_LAUNCH(2, m, a2, S, S, dt, qbar)
    if (check_launch(ctx)) return PDG_ERR_CUDA;
  }
#undef RK_LAUNCH
  k_subcycle_final<<<nb, bs, 0, s>>>(m, S, q0, f3d2d, msub, msub * dt, qbar, f2d);
  return check_launch(ctx);
}

// ---- per-RK-stage entries (partitioned runs exchange the stage state between stages) ----
int pdg_ext2d_subcycle_begin(pdg_ctx* ctx, const double* S, double g, double dt, int check_cfl, double* qbar,
                             void* stream) {
  cudaSetDevice(ctx->device);
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = ctx->nt;
  if (check_cfl && run_cfl(ctx, S, g, dt, ctx->red + 4000, s)) return PDG_ERR_CUDA;
  double* q0 = ctx->ws2d + (size_t)18 * nt;
  if (cudaMemcpyAsync(q0, S + (size_t)3 * nt, (size_t)6 * nt * sizeof(double), cudaMemcpyDeviceToDevice, s) !=
      cudaSuccess)
    return PDG_ERR_CUDA;
  if (cudaMemsetAsync(qbar, 0, (size_t)6 * nt * sizeof(double), s) != cudaSuccess) return PDG_ERR_CUDA;
  return PDG_OK;
}

// one SSP-RK3 stage: X = state evaluated, S0 = substep start, Y = output (stage 2 may write Y = S0)
int pdg_ext2d_rk_stage(pdg_ctx* ctx, int stage, const double* X, const double* S0, double* Y, double dt, double g,
                       double rho0, const double* f3d2d, const double* source, const double* patm, int has_bc,
                       double eta_bc, double* qbar, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = ctx->nt;
  DMesh m = ctx->view();
  const int bs = 256, nb = nblocks(ctx->nown, bs);
  Ext2DIn a{X, X + (size_t)3 * nt, X + (size_t)6 * nt, f3d2d, source, patm, has_bc, eta_bc, g, rho0};
  if (stage == 0)
    k_rk_stage<0><<<nb, bs, 0, s>>>(m, a, S0, Y, dt, qbar);
  else if (stage == 1)
    k_rk_stage<1><<<nb, bs, 0, s>>>(m, a, S0, Y, dt, qbar);
  else
    k_rk_stage<2><<<nb, bs, 0, s>>>(m, a, S0, Y, dt, qbar);
  (void)bs;
  return check_launch(ctx);
}

// the same stage over an explicit column list (partitioned runs: boundary / interior columns)
int pdg_ext2d_rk_stage_cols(pdg_ctx* ctx, int stage, const double* X, const double* S0, double* Y, double dt,
                            double g, double rho0, const double* f3d2d, double* qbar, const int* els, int n_els,
                            void* stream) {
  if (n_els <= 0) return PDG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int nt = ctx->nt;
  DMesh m = ctx->view();
  const int nb = nblocks(n_els, 128);
  Ext2DIn a{X, X + (size_t)3 * nt, X + (size_t)6 * nt, f3d2d, nullptr, nullptr, 0, 0.0, g, rho0};
  if (tune_get(TUNE_RK) == 8) {   // programmatic dependent launch (see pdg_ext2d_subcycle)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nb);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    if (stage == 0)
      cudaLaunchKernelEx(&cfg, k_rk_stage<0, 128, 4, true>, m, a, S0, Y, dt, qbar, els, n_els);
    else if (stage == 1)
      cudaLaunchKernelEx(&cfg, k_rk_stage<1, 128, 4, true>, m, a, S0, Y, dt, qbar, els, n_els);
    else
      cudaLaunchKernelEx(&cfg, k_rk_stage<2, 128, 4, true>, m, a, S0, Y, dt, qbar, els, n_els);
    return check_launch(ctx);
  }
  if (stage == 0)
    k_rk_stage<0, 128, 4><<<nb, 128, 0, s>>>(m, a, S0, Y, dt, qbar, els, n_els);
  else if (stage == 1)
    k_rk_stage<1, 128, 4><<<nb, 128, 0, s>>>(m, a, S0, Y, dt, qbar, els, n_els);
  else
    k_rk_stage<2, 128, 4><<<nb, 128, 0, s>>>(m, a, S0, Y, dt, qbar, els, n_els);
  return check_launch(ctx);
}

int pdg_ext2d_subcycle_end(pdg_ctx* ctx, const double* S, const double* f3d2d, int msub, double dt, double* qbar,
                           double* f2d, void* stream) {
  const int nt = ctx->nt;
  double* q0 = ctx->ws2d + (size_t)18 * nt;
  k_subcycle_final<<<nblocks(ctx->nown, 256), 256, 0, (cudaStream_t)stream>>>(ctx->view(), S, q0, f3d2d, msub,
                                                                              msub * dt, qbar, f2d);
  return check_launch(ctx);
}

int pdg_apply_mh(const double* v, const double* j2d, int n, int nc, int inverse, double* out, pdg_err* err,
                 void* stream) {
  if (n == 0) return PDG_OK;
  k_apply_mh<<<nblocks(n, 256), 256, 0, (cudaStream_t)stream>>>(v, j2d, n, nc, inverse, out, err);
  return check_launch_noctx();
}

}  // extern "C"
