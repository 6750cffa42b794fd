// Mesh2D setup on the GPU (mesh.py:79-127, 187-228): geometry, edge pairing, Hilbert permutation.
//
// Integer maps are bit-exact with the reference: edge pairing is a STABLE radix sort of the
// (min, max) vertex keys with the flat (element, edge) index as value, so equal keys keep the
// reference's dict insertion order and runs pair (1st,2nd), (3rd,4th), ... exactly like its
// seen/pop loop; the Hilbert order is a stable radix sort of the curve distance of the
// quantised centroid, whose float steps are rounded in numpy's order (_rn intrinsics, no FMA).
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace pdg {

__global__ void k_mesh_geometry(int nt, const double* __restrict__ vx, const double* __restrict__ vy,
                                const double* __restrict__ vb, const long long* __restrict__ tri, double* X, double* Y,
                                double* B, double* j2d, double* dphx, double* dphy, double* elen, double* enx,
                                double* eny, pdg_err* err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nt) return;
  double x[3], y[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const long long v = tri[3 * (size_t)e + i];
    x[i] = vx[v];
    y[i] = vy[v];
    X[3 * (size_t)e + i] = x[i];
    Y[3 * (size_t)e + i] = y[i];
    B[3 * (size_t)e + i] = vb[v];
  }
  // J2D = (x1-x0)(y2-y0) - (x2-x0)(y1-y0)           (mesh.py:85)
  const double J = __dsub_rn(__dmul_rn(__dsub_rn(x[1], x[0]), __dsub_rn(y[2], y[0])),
                             __dmul_rn(__dsub_rn(x[2], x[0]), __dsub_rn(y[1], y[0])));
  j2d[e] = J;
  if (J <= 0.0) report(err, 8, e, 0, J);
  // grad phi_i = (y_j - y_k, x_k - x_j) / J2D, (i, j, k) cyclic   (mesh.py:89-93)
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3, k = (i + 2) % 3;
    dphx[3 * (size_t)e + i] = __ddiv_rn(__dsub_rn(y[j], y[k]), J);
    dphy[3 * (size_t)e + i] = __ddiv_rn(__dsub_rn(x[k], x[j]), J);
  }
  // edges k = (k, k+1): length and outward normal (dy, -dx)/len       (mesh.py:95-101)
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const double ex = __dsub_rn(x[EV1(k)], x[EV0(k)]), ey = __dsub_rn(y[EV1(k)], y[EV0(k)]);
    const double len = hypot(ex, ey);
    if (len <= 0.0) report(err, PDG_ERR_NONPOS_LENGTH, e, k, len);
    elen[3 * (size_t)e + k] = len;
    enx[3 * (size_t)e + k] = __ddiv_rn(ey, len);
    eny[3 * (size_t)e + k] = __ddiv_rn(-ex, len);
  }
}

__global__ void k_edge_keys(int nt, long long nv, const long long* __restrict__ tri, unsigned long long* keys,
                            int* vals) {
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= 3 * nt) return;
  const int e = f / 3, k = f % 3;
  const long long a = tri[3 * (size_t)e + EV0(k)], b = tri[3 * (size_t)e + EV1(k)];
  const long long lo = a < b ? a : b, hi = a < b ? b : a;
  keys[f] = (unsigned long long)lo * (unsigned long long)nv + (unsigned long long)hi;
  vals[f] = f;
}

// head index of each run of equal keys (then a max-scan propagates it along the run)
__global__ void k_run_heads(int n, const unsigned long long* __restrict__ k, int* head) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  head[i] = (i == 0 || k[i] != k[i - 1]) ? i : 0;
}

__global__ void k_pair(int n, const unsigned long long* __restrict__ k, const int* __restrict__ v,
                       const int* __restrict__ runstart, long long* nbr, long long* nbrk, long long* btag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int rank = i - runstart[i];
  if ((rank & 1) == 0 && i + 1 < n && k[i + 1] == k[i]) {
    const int f1 = v[i], f2 = v[i + 1];
    nbr[f1] = f2 / 3;
    nbrk[f1] = f2 % 3;
    nbr[f2] = f1 / 3;
    nbrk[f2] = f1 % 3;
    btag[f1] = 0;
    btag[f2] = 0;
  }
}

__global__ void k_adj_init(int n, long long* nbr, long long* nbrk, long long* btag) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  nbr[i] = -1;
  nbrk[i] = -1;
  btag[i] = 1;  // BTAG_WALL
}

__global__ void k_centroids(int nt, const double* __restrict__ X, const double* __restrict__ Y, double* cx, double* cy) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nt) return;
  const size_t o = 3 * (size_t)e;
  cx[e] = __ddiv_rn(__dadd_rn(__dadd_rn(X[o], X[o + 1]), X[o + 2]), 3.0);
  cy[e] = __ddiv_rn(__dadd_rn(__dadd_rn(Y[o], Y[o + 1]), Y[o + 2]), 3.0);
}

// mesh.py:187-207 on the quantised centroid (mesh.py:217-224)
__global__ void k_hilbert(int nt, int order, const double* __restrict__ cx, const double* __restrict__ cy,
                          const double* __restrict__ mm, unsigned long long* d, int* idx) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nt) return;
  const long long n = 1LL << order;
  const double xmin = mm[0], xmax = mm[1], ymin = mm[2], ymax = mm[3];
  const double sx = fmax(__dsub_rn(xmax, xmin), 1e-300), sy = fmax(__dsub_rn(ymax, ymin), 1e-300);
  const double fn = (double)(n - 1);
  long long ix = (long long)__dmul_rn(__ddiv_rn(__dsub_rn(cx[e], xmin), sx), fn);
  long long iy = (long long)__dmul_rn(__ddiv_rn(__dsub_rn(cy[e], ymin), sy), fn);
  ix = ix < n - 1 ? ix : n - 1;
  iy = iy < n - 1 ? iy : n - 1;
  long long dd = 0;
  for (long long s = n >> 1; s > 0; s >>= 1) {
    const long long rx = (ix & s) > 0, ry = (iy & s) > 0;
    dd += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        ix = (n - 1) - ix;
        iy = (n - 1) - iy;
      }
      const long long t = ix;
      ix = iy;
      iy = t;
    }
  }
  d[e] = (unsigned long long)dd;
  idx[e] = e;
}

__global__ void k_minmax_final(const double* part, int nb, double* mm) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double a = 1e308, b = -1e308, c = 1e308, d = -1e308;
  for (int i = 0; i < nb; ++i) {
    a = fmin(a, part[4 * i]);
    b = fmax(b, part[4 * i + 1]);
    c = fmin(c, part[4 * i + 2]);
    d = fmax(d, part[4 * i + 3]);
  }
  mm[0] = a;
  mm[1] = b;
  mm[2] = c;
  mm[3] = d;
}

__global__ void k_minmax(int n, const double* __restrict__ cx, const double* __restrict__ cy, double* part) {
  __shared__ double s[4][256];
  double a = 1e308, b = -1e308, c = 1e308, d = -1e308;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    a = fmin(a, cx[i]);
    b = fmax(b, cx[i]);
    c = fmin(c, cy[i]);
    d = fmax(d, cy[i]);
  }
  s[0][threadIdx.x] = a;
  s[1][threadIdx.x] = b;
  s[2][threadIdx.x] = c;
  s[3][threadIdx.x] = d;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      s[0][threadIdx.x] = fmin(s[0][threadIdx.x], s[0][threadIdx.x + h]);
      s[1][threadIdx.x] = fmax(s[1][threadIdx.x], s[1][threadIdx.x + h]);
      s[2][threadIdx.x] = fmin(s[2][threadIdx.x], s[2][threadIdx.x + h]);
      s[3][threadIdx.x] = fmax(s[3][threadIdx.x], s[3][threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int q = 0; q < 4; ++q) part[4 * blockIdx.x + q] = s[q][0];
}

__global__ void k_widen(int n, const int* a, long long* o) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) o[i] = a[i];
}

struct MaxOp {
  __device__ int operator()(int a, int b) const { return a > b ? a : b; }
};

}  // namespace pdg

using namespace pdg;

static int bits_for(unsigned long long maxkey) {
  int b = 1;
  while (b < 64 && (maxkey >> b) != 0ULL) ++b;
  return b;
}

extern "C" {

// geometry + adjacency of a triangle mesh; every array is a DEVICE pointer in the reference
// (nt, 3) layout (Mesh2D fields).  tri: int64 (nt, 3); vx, vy, vb: (nv).
int pdg_mesh_build(int nt, long long nv, const double* vx, const double* vy, const double* vb, const long long* tri,
                   double* x, double* y, double* b, double* j2d, double* dphx, double* dphy, double* elen,
                   double* enx, double* eny, long long* nbr, long long* nbrk, long long* btag, pdg_err* err,
                   void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nt == 0) return PDG_OK;
  k_mesh_geometry<<<nblocks(nt, 128), 128, 0, s>>>(nt, vx, vy, vb, tri, x, y, b, j2d, dphx, dphy, elen, enx, eny,
                                                   err);
  const int n = 3 * nt;
  unsigned long long *k0, *k1;
  int *v0, *v1, *head, *run;
  void* tmp = nullptr;
  size_t tb = 0, tb2 = 0;
  if (cudaMallocAsync(&k0, n * sizeof(unsigned long long), s) || cudaMallocAsync(&k1, n * sizeof(unsigned long long), s) ||
      cudaMallocAsync(&v0, n * sizeof(int), s) || cudaMallocAsync(&v1, n * sizeof(int), s) ||
      cudaMallocAsync(&head, n * sizeof(int), s) || cudaMallocAsync(&run, n * sizeof(int), s))
    return PDG_ERR_CUDA;
  k_edge_keys<<<nblocks(n, 256), 256, 0, s>>>(nt, nv, tri, k0, v0);
  const int bits = bits_for((unsigned long long)(nv > 0 ? nv : 1) * (unsigned long long)(nv > 0 ? nv : 1));
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, v1, n, 0, bits, s);
  cub::DeviceScan::InclusiveScan(nullptr, tb2, head, run, MaxOp(), n, s);
  tb = tb > tb2 ? tb : tb2;
  if (cudaMallocAsync(&tmp, tb, s)) return PDG_ERR_CUDA;
  cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, v1, n, 0, bits, s);   // stable
  k_run_heads<<<nblocks(n, 256), 256, 0, s>>>(n, k1, head);
  cub::DeviceScan::InclusiveScan(tmp, tb, head, run, MaxOp(), n, s);
  k_adj_init<<<nblocks(n, 256), 256, 0, s>>>(n, nbr, nbrk, btag);
  k_pair<<<nblocks(n, 256), 256, 0, s>>>(n, k1, v1, run, nbr, nbrk, btag);
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(k0, s);
  cudaFreeAsync(k1, s);
  cudaFreeAsync(v0, s);
  cudaFreeAsync(v1, s);
  cudaFreeAsync(head, s);
  cudaFreeAsync(run, s);
  return check_launch_noctx();
}

// hilbert_reorder's permutation (mesh.py:210-228): perm[new] = old, stable in the curve distance.
int pdg_hilbert_perm(int nt, int order, const double* x, const double* y, long long* perm, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (nt == 0) return PDG_OK;
  double *cx, *cy, *part, *mm;
  unsigned long long *d0, *d1;
  int *i0, *i1;
  const int nb = 128;
  if (cudaMallocAsync(&cx, nt * sizeof(double), s) || cudaMallocAsync(&cy, nt * sizeof(double), s) ||
      cudaMallocAsync(&part, 4 * nb * sizeof(double), s) || cudaMallocAsync(&mm, 4 * sizeof(double), s) ||
      cudaMallocAsync(&d0, nt * sizeof(unsigned long long), s) || cudaMallocAsync(&d1, nt * sizeof(unsigned long long), s) ||
      cudaMallocAsync(&i0, nt * sizeof(int), s) || cudaMallocAsync(&i1, nt * sizeof(int), s))
    return PDG_ERR_CUDA;
  k_centroids<<<nblocks(nt, 256), 256, 0, s>>>(nt, x, y, cx, cy);
  k_minmax<<<nb, 256, 0, s>>>(nt, cx, cy, part);
  k_minmax_final<<<1, 32, 0, s>>>(part, nb, mm);
  k_hilbert<<<nblocks(nt, 256), 256, 0, s>>>(nt, order, cx, cy, mm, d0, i0);
  void* tmp = nullptr;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, d0, d1, i0, i1, nt, 0, 2 * order, s);
  if (cudaMallocAsync(&tmp, tb, s)) return PDG_ERR_CUDA;
  cub::DeviceRadixSort::SortPairs(tmp, tb, d0, d1, i0, i1, nt, 0, 2 * order, s);   // stable argsort
  cudaFreeAsync(tmp, s);
  k_widen<<<nblocks(nt, 256), 256, 0, s>>>(nt, i1, perm);
  cudaFreeAsync(cx, s);
  cudaFreeAsync(cy, s);
  cudaFreeAsync(part, s);
  cudaFreeAsync(mm, s);
  cudaFreeAsync(d0, s);
  cudaFreeAsync(d1, s);
  cudaFreeAsync(i0, s);
  cudaFreeAsync(i1, s);
  return check_launch_noctx();
}

}  // extern "C"
