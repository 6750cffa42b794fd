// Layout conversion between the reference's row layouts and the device planes, for the host I/O
// path of the drop-in (set_state / get_state, internal3d.py / external2d.py array conventions).
//
//   rows   [ncols][L][nk]  : a column range of a (P, nk) prism field (p = c L + l) or, with L = 1,
//                            of an (nt, nk) 2D field -- exactly the bytes of the host chunk
//   planes [nk][L][nt]     : the device layout (col3d.cuh pix)
//
// A host chunk is copied to a device staging buffer by DMA and then rearranged by these kernels
// (and the reverse on the way out), so the PCIe copies stay plain contiguous transfers.  Tiled
// through shared memory: a block moves 32 columns x TL layers x nk values; reads are contiguous
// runs of TL nk doubles per column, writes are 256-byte runs of 32 columns per (node, layer).
#include "ctx.cuh"

namespace pdg {
constexpr int HT_C = 32;   // columns per tile
constexpr int HT_L = 8;    // layers per tile
constexpr int HT_T = 256;  // threads

template <bool TO_PLANES>
__global__ void __launch_bounds__(HT_T) k_rows_planes(const double* __restrict__ src, double* __restrict__ dst,
                                                      int ncols, int L, int nk, int nt, int c0) {
  extern __shared__ double tile[];  // [HT_C][HT_L * nk + 1]
  const int w = HT_L * nk + 1;
  const int cb = blockIdx.x * HT_C, lb = blockIdx.y * HT_L;
  const int nc = min(HT_C, ncols - cb), nl = min(HT_L, L - lb);
  const int run = nl * nk;  // contiguous values per column in the rows layout
  if (TO_PLANES) {
    for (int i = threadIdx.x; i < nc * run; i += HT_T) {
      const int col = i / run, j = i - col * run;
      tile[col * w + j] = src[((size_t)(cb + col) * L + lb) * nk + j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < HT_C * run; i += HT_T) {
      const int col = i % HT_C, j = i / HT_C;   // j = l * nk + k
      if (col >= nc) continue;
      const int l = j / nk, k = j - l * nk;
      dst[((size_t)k * L + lb + l) * nt + c0 + cb + col] = tile[col * w + j];
    }
  } else {
    for (int i = threadIdx.x; i < HT_C * run; i += HT_T) {
      const int col = i % HT_C, j = i / HT_C;
      if (col >= nc) continue;
      const int l = j / nk, k = j - l * nk;
      tile[col * w + j] = src[((size_t)k * L + lb + l) * nt + c0 + cb + col];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < nc * run; i += HT_T) {
      const int col = i / run, j = i - col * run;
      dst[((size_t)(cb + col) * L + lb) * nk + j] = tile[col * w + j];
    }
  }
}

static int launch_rp(bool to_planes, const double* src, double* dst, int ncols, int L, int nk, int nt, int c0,
                     void* stream) {
  if (ncols <= 0 || L <= 0 || nk <= 0) return PDG_OK;
  if (nk > 16 || c0 < 0 || c0 + ncols > nt) return PDG_ERR_SHAPE;
  const dim3 grid((ncols + HT_C - 1) / HT_C, (L + HT_L - 1) / HT_L);
  const size_t sm = (size_t)HT_C * (HT_L * nk + 1) * sizeof(double);
  if (to_planes)
    k_rows_planes<true><<<grid, HT_T, sm, (cudaStream_t)stream>>>(src, dst, ncols, L, nk, nt, c0);
  else
    k_rows_planes<false><<<grid, HT_T, sm, (cudaStream_t)stream>>>(src, dst, ncols, L, nk, nt, c0);
  return check_launch_noctx();
}
}  // namespace pdg

using namespace pdg;
extern "C" {
int pdg_rows_to_planes(const double* rows, int ncols, int L, int nk, double* planes, int nt, int c0, void* stream) {
  return launch_rp(true, rows, planes, ncols, L, nk, nt, c0, stream);
}
int pdg_planes_to_rows(const double* planes, int nt, int c0, int ncols, int L, int nk, double* rows, void* stream) {
  return launch_rp(false, planes, rows, ncols, L, nk, nt, c0, stream);
}
// device-to-device copy on the caller's stream (the step's 2D working-state copies: the stepper
// graph holds only library launches and copies, no framework kernels)
int pdg_copy_d2d(void* dst, const void* src, long long bytes, void* stream) {
  if (bytes <= 0) return PDG_OK;
  return cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) == cudaSuccess
             ? PDG_OK
             : PDG_ERR_CUDA;
}

}  // extern "C"
