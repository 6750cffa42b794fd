// Device building blocks shared by the 3D assemblies (internal3d.py) and the fused stepper.
//
// Execution model: ONE THREAD PER COLUMN looping over layers.  A warp covers 32 consecutive
// (Hilbert-ordered) columns, so every per-layer load of a P6 plane is a coalesced 256-byte
// run; per-column 2D data stays in registers across the whole layer loop; vertical sweeps
// (r, w, w~, block Thomas) are carried in registers between layer iterations.
#pragma once
#include "common.cuh"

namespace pdg {

// 32-bit plane index (k * L + l) * nt + c: one field array never exceeds 2^32 words (checked at
// pdg_ctx_set_layers), and unsigned arithmetic keeps the address math in single IMADs
__device__ __forceinline__ unsigned pix(int k, int l, int c, int L, int nt) {
  return ((unsigned)k * (unsigned)L + (unsigned)l) * (unsigned)nt + (unsigned)c;
}
// the 36-plane prism-mass arrays (API only) reach 36 * L * nt words: 64-bit offsets
__device__ __forceinline__ size_t pix36(int rs, int l, int c, int L, int nt) {
  return ((size_t)rs * (size_t)L + (size_t)l) * (size_t)nt + (size_t)c;
}
// per-thread asynchronous global -> shared copies (LDGSTS): the staged kernels issue the next
// layer's words one or two layers ahead and wait for them only when the layer is consumed
__device__ __forceinline__ void cp_async8(double* sdst, const double* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// ---- Blackwell bulk-async copies (TMA engine, 1-D) with mbarrier completion ---------------------
// One elected thread arms a slot's mbarrier with the byte count and issues cp.async.bulk copies of
// whole contiguous plane segments (a block's columns of one node plane: 1 KB at 128 columns); the
// copy engine moves them into shared memory without per-thread LDGSTS and signals the barrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of the slot (the previous readers) before the async-proxy refill
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// TMA bulk prefetch of a contiguous global range into L2 (16-byte aligned, size a multiple of 16):
// one instruction warms a whole plane segment of a block's columns for the next layer
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ void ld6(const double* __restrict__ f, int l, int c, int L, int nt, double v[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = f[pix(k, l, c, L, nt)];
}
__device__ __forceinline__ void st6(double* __restrict__ f, int l, int c, int L, int nt, const double v[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) f[pix(k, l, c, L, nt)] = v[k];
}

// read-only-path (ld.global.nc) variants for kernels whose inputs never alias their outputs
__device__ __forceinline__ void ld6g(const double* f, int l, int c, int L, int nt, double v[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = __ldg(f + pix(k, l, c, L, nt));
}
__device__ __forceinline__ void ld_nb4g(const double* f, int k2, int e2, int l, int L, int nt, double n4[4]) {
  const int a = EV0(k2), b = EV1(k2);
  n4[0] = __ldg(f + pix(a, l, e2, L, nt));
  n4[1] = __ldg(f + pix(b, l, e2, L, nt));
  n4[2] = __ldg(f + pix((3 + a), l, e2, L, nt));
  n4[3] = __ldg(f + pix((3 + b), l, e2, L, nt));
}

// the same loads with the plane stride ln = L * nt passed in (the caller hides it from the
// optimiser so the per-node plane offsets are re-formed instead of held live across the layer loop)
__device__ __forceinline__ void ld6g_o(const double* f, unsigned lo, unsigned ln, double v[6]) {
#pragma unroll
  for (int k = 0; k < 6; ++k) v[k] = __ldg(f + (k * ln + lo));
}
__device__ __forceinline__ void ld_nb4g_o(const double* f, int k2, unsigned le2, unsigned ln, double n4[4]) {
  const unsigned a = EV0(k2), b = EV1(k2);
  n4[0] = __ldg(f + (a * ln + le2));
  n4[1] = __ldg(f + (b * ln + le2));
  n4[2] = __ldg(f + ((3 + a) * ln + le2));
  n4[3] = __ldg(f + ((3 + b) * ln + le2));
}

// L1 prefetch of the 6 node planes of layer l (issued one layer ahead: the thread-per-column
// kernels run at ~8 warps/SM, too few to hide HBM latency, and have no registers to spare for
// software pipelining -- a prefetch costs no register)
__device__ __forceinline__ void pf6(const double* f, int l, int c, int L, int nt) {
#pragma unroll
  for (int k = 0; k < 6; ++k) asm volatile("prefetch.global.L1 [%0];" ::"l"(f + pix(k, l, c, L, nt)));
}
__device__ __forceinline__ void pf_nb4(const double* f, int k2, int e2, int l, int L, int nt) {
  const int a = EV0(k2), b = EV1(k2);
  asm volatile("prefetch.global.L1 [%0];" ::"l"(f + pix(a, l, e2, L, nt)));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(f + pix(b, l, e2, L, nt)));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(f + pix((3 + a), l, e2, L, nt)));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(f + pix((3 + b), l, e2, L, nt)));
}

// the 4 lateral nodes (t0, t1, b0, b1) of the neighbour prism across local edge k2 of column e2
__device__ __forceinline__ void ld_nb4(const double* __restrict__ f, int k2, int e2, int l, int L, int nt,
                                       double n4[4]) {
  const int a = EV0(k2), b = EV1(k2);
  n4[0] = f[pix(a, l, e2, L, nt)];
  n4[1] = f[pix(b, l, e2, L, nt)];
  n4[2] = f[pix((3 + a), l, e2, L, nt)];
  n4[3] = f[pix((3 + b), l, e2, L, nt)];
}

// own lateral trace on edge k at the 2v x 2h face points (internal3d.py:229-258, mirror=False)
__device__ __forceinline__ void tr_own(const double v[6], int k, double t[2][2]) {
  const int a = EV0(k), b = EV1(k);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double ht = v[a] * ES[h][0] + v[b] * ES[h][1];
    const double hb = v[3 + a] * ES[h][0] + v[3 + b] * ES[h][1];
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) t[vv][h] = VS[vv][0] * ht + VS[vv][1] * hb;
  }
}
// neighbour trace at the same physical points (mirrored edge-point order)
__device__ __forceinline__ void tr_nb(const double n4[4], double t[2][2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double ht = n4[0] * ES[h][1] + n4[1] * ES[h][0];
    const double hb = n4[2] * ES[h][1] + n4[3] * ES[h][0];
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) t[vv][h] = VS[vv][0] * ht + VS[vv][1] * hb;
  }
}
// zeta-independent corner data on the two edge points
__device__ __forceinline__ void tr2_own(const double c3[3], int k, double t[2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) t[h] = c3[EV0(k)] * ES[h][0] + c3[EV1(k)] * ES[h][1];
}
__device__ __forceinline__ void tr2_nb(double a, double b, double t[2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) t[h] = a * ES[h][1] + b * ES[h][0];
}
// corner data duplicated on both levels, traced like a prism field
__device__ __forceinline__ void tr_dup(const double t2[2], double t[2][2]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) t[vv][h] = VS[vv][0] * t2[h] + VS[vv][1] * t2[h];
}

// acc[node] += s * sum_vh VS[v][lev] ES[h][hn] x[v][h] over the 4 lateral nodes of edge k
// (internal3d.py:261-272; s = sign * Jedge)
__device__ __forceinline__ void lat_add(double acc[6], int k, const double x[2][2], double s) {
#pragma unroll
  for (int lev = 0; lev < 2; ++lev)
#pragma unroll
    for (int hn = 0; hn < 2; ++hn) {
      double t = 0.0;
#pragma unroll
      for (int vv = 0; vv < 2; ++vv)
#pragma unroll
        for (int h = 0; h < 2; ++h) t += VS[vv][lev] * ES[h][hn] * x[vv][h];
      acc[3 * lev + (hn == 0 ? EV0(k) : EV1(k))] += s * t;
    }
}

// the projection of lat_add without the accumulation: p[lev][hn] = sum_vh VS[v][lev] ES[h][hn] x[v][h]
// (a vector face field n_d x is then projected once and added with the factors s n_d)
__device__ __forceinline__ void lat_proj(const double x[2][2], double p[2][2]) {
#pragma unroll
  for (int lev = 0; lev < 2; ++lev)
#pragma unroll
    for (int hn = 0; hn < 2; ++hn) {
      double t = 0.0;
#pragma unroll
      for (int vv = 0; vv < 2; ++vv)
#pragma unroll
        for (int h = 0; h < 2; ++h) t += VS[vv][lev] * ES[h][hn] * x[vv][h];
      p[lev][hn] = t;
    }
}
__device__ __forceinline__ void lat_put(double acc[6], int k, const double p[2][2], double s) {
#pragma unroll
  for (int lev = 0; lev < 2; ++lev)
#pragma unroll
    for (int hn = 0; hn < 2; ++hn) acc[3 * lev + (hn == 0 ? EV0(k) : EV1(k))] += s * p[lev][hn];
}

// per-column neighbour data of one interior edge, loaded once per column
struct EdgeNb {
  int e2, k2;
  double stab[2];  // 0.5 [[eta]] max(c) at the two edge points (internal3d.py:296-301)
  double hm[2];    // 0.5 (H_own + H_nbr) at the edge points: {Jz} = (f_b - f_t)/2 * hm on sigma layers
  double hn[2];    // neighbour depth H at its two edge corners (own traversal order)
};

__device__ __forceinline__ void edge_setup(const DMesh& m, const Col& C, const double eta[3],
                                           const double* __restrict__ eta_g, int k, double g, EdgeNb& E) {
  const int nt = m.nt;
  E.e2 = C.nb[k];
  E.k2 = C.nk[k];
  if (C.tag[k] != 0) return;
  const int i0 = EV0(E.k2) * nt + E.e2, i1 = EV1(E.k2) * nt + E.e2;
  const double eta0 = eta_g[i0], eta1 = eta_g[i1];
  const double b0 = ldg(m.b + i0), b1 = ldg(m.b + i1);
  E.hn[0] = eta0 - b0;
  E.hn[1] = eta1 - b1;
  double ei[2], ee[2], bi[2], be[2];
  tr2_own(eta, k, ei);
  tr2_own(C.b, k, bi);
  tr2_nb(eta0, eta1, ee);
  tr2_nb(b0, b1, be);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double hi = ei[h] - bi[h], he = ee[h] - be[h];
    // max(sqrt(g hi), sqrt(g he)) == sqrt(g max(hi, he)) exactly (sqrt is monotone, correctly rounded)
    E.stab[h] = 0.5 * (ei[h] - ee[h]) * sqrt(g * fmax(hi, he));
    E.hm[h] = 0.5 * (hi + he);
  }
}

// combine own and neighbour lateral nodes so one trace gives the interface mean:
// own trace uses (o0, o1) with ES[h][0..1], the mirrored neighbour (n0, n1) with ES[h][1..0]
__device__ __forceinline__ void tr_mean(const double o[6], int k, const double n4[4], double t[2][2]) {
  const int a = EV0(k), b = EV1(k);
  const double c0 = o[a] + n4[1], c1 = o[b] + n4[0], c2 = o[3 + a] + n4[3], c3 = o[3 + b] + n4[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double ht = c0 * ES[h][0] + c1 * ES[h][1];
    const double hb = c2 * ES[h][0] + c3 * ES[h][1];
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) t[vv][h] = 0.5 * (VS[vv][0] * ht + VS[vv][1] * hb);
  }
}

// half jump 0.5 (own - nbr) at the face points from combined nodes
__device__ __forceinline__ void tr_jump(const double o[6], int k, const double n4[4], double t[2][2]) {
  const int a = EV0(k), b = EV1(k);
  const double c0 = o[a] - n4[1], c1 = o[b] - n4[0], c2 = o[3 + a] - n4[3], c3 = o[3 + b] - n4[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const double ht = c0 * ES[h][0] + c1 * ES[h][1];
    const double hb = c2 * ES[h][0] + c3 * ES[h][1];
#pragma unroll
    for (int vv = 0; vv < 2; ++vv) t[vv][h] = 0.5 * (VS[vv][0] * ht + VS[vv][1] * hb);
  }
}

// stabilised lateral flux factor n.{q} + {Jz/H} max(c) [[eta]] on interior edge k
// (internal3d.py:275-314).  On sigma layers Jz/H = (f_b - f_t)/2 =: jm for every column.
__device__ __forceinline__ void lat_factor(const Col& C, const EdgeNb& E, int k, double jm, const double qo[2][6],
                                           const double qn[2][4], double fac[2][2]) {
  double o[6], n4[4];
#pragma unroll
  for (int i = 0; i < 6; ++i) o[i] = C.nx[k] * qo[0][i] + C.ny[k] * qo[1][i];
#pragma unroll
  for (int i = 0; i < 4; ++i) n4[i] = C.nx[k] * qn[0][i] + C.ny[k] * qn[1][i];
  double t[2][2];
  tr_mean(o, k, n4, t);
#pragma unroll
  for (int vv = 0; vv < 2; ++vv)
#pragma unroll
    for (int h = 0; h < 2; ++h) fac[vv][h] = t[vv][h] + jm * E.stab[h];
}

// bilinear P1 x P1 integral over the prism against phi_z: S[m] = sum_{l1,l2} K3[m][l1][l2] a_l1^T MHQ b_l2
// (= sum_vq QW VS[v][m] a(v,q) b(v,q), exact for the 12-point rule)
__device__ __forceinline__ void mhq_vec(const double x[3], double y[3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) y[a] = MHQ[a][0] * x[0] + MHQ[a][1] * x[1] + MHQ[a][2] * x[2];
}

// iso-zeta divergence test term: acc[lev*3+i] += J2D (dphx_i S[lev][0] + dphy_i S[lev][1])
__device__ __forceinline__ void iso_add(const Col& C, const double S[2][2], double acc[6]) {
#pragma unroll
  for (int lev = 0; lev < 2; ++lev)
#pragma unroll
    for (int i = 0; i < 3; ++i) acc[3 * lev + i] += C.j2d * (C.dx[i] * S[lev][0] + C.dy[i] * S[lev][1]);
}

// values of a prism nodal field at the 12 tensor points: out[v][q]
__device__ __forceinline__ void at_pts(const double f[6], double out[2][6]) {
  double t[6], b[6];
  hq(f, t);
  hq(f + 3, b);
#pragma unroll
  for (int vv = 0; vv < 2; ++vv)
#pragma unroll
    for (int q = 0; q < 6; ++q) out[vv][q] = VS[vv][0] * t[q] + VS[vv][1] * b[q];
}

// S[m][d] = sum_vq QW VS[v][m] a[v][q] b_d[v][q]   (volume advection against phi_z grad_h phi_h)
__device__ __forceinline__ void adv_moment(const double a[2][6], const double bx[2][6], const double by[2][6],
                                           double S[2][2]) {
#pragma unroll
  for (int mm = 0; mm < 2; ++mm) {
    double sx = 0.0, sy = 0.0;
#pragma unroll
    for (int vv = 0; vv < 2; ++vv)
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        const double w = QW[q] * VS[vv][mm] * a[vv][q];
        sx += w * bx[vv][q];
        sy += w * by[vv][q];
      }
    S[mm][0] = sx;
    S[mm][1] = sy;
  }
}

}  // namespace pdg
