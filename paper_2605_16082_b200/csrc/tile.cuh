// Tile staging shared by the tiled kernels (3D column kernels, the 2D RK stage): StagePlanes and
// TileStage (moved from int3d.cu).
#pragma once
#include "col3d.cuh"

namespace pdg {

// staged planes: word w of a column at layer l is p[w][l * nt + col] (p[w] = plane base + node offset)
struct StagePlanes {
  const double* p[30];
};

// ---------------------------------------------------------------------------------------------
// Tile staging shared by the tiled column kernels: NW words per column of layer l (word w at
// sp.p[w][l nt + col]) for the block's TW columns and its halo, copied with per-thread cp.async
// into smem laid out [NW][tj] (tj = TW + max halo).  The halo copies are split so that every
// thread issues about the same number of them.
template <int NW, int TW>
struct TileStage {
  int t, c, nh, h0, hj, hw0, hw1, hcol;
  bool act;
  __device__ __forceinline__ void init(const DMesh& m, const int* __restrict__ halo, const int* __restrict__ hoff) {
    t = threadIdx.x;
    c = blockIdx.x * TW + t;
    act = c < m.nown;
    h0 = hoff[blockIdx.x];
    nh = hoff[blockIdx.x + 1] - h0;
    const int nparts = nh > 0 ? max(1, TW / nh) : 1;
    const int wpp = (NW + nparts - 1) / nparts;
    const int part = nh > 0 ? t / nh : nparts;
    hj = nh > 0 ? t - part * nh : 0;
    hw0 = part < nparts ? part * wpp : NW;
    hw1 = min(NW, hw0 + wpp);
    hcol = part < nparts ? halo[h0 + hj] : 0;
  }
  // lo = l * nt: plane offsets stay below 2^32 words (col3d.cuh pix), so one 32-bit offset per
  // column is added to each plane pointer
  __device__ __forceinline__ void issue(double* s, int tj, const StagePlanes& sp, unsigned lo,
                                        const int* __restrict__ halo) const {
    if (act) {
      const unsigned oc = lo + (unsigned)c;
#pragma unroll
      for (int w = 0; w < NW; ++w) cp_async8(s + w * tj + t, sp.p[w] + oc);
    }
    const unsigned oh = lo + (unsigned)hcol;
    for (int w = hw0; w < hw1; ++w) cp_async8(s + w * tj + TW + hj, sp.p[w] + oh);
    for (int j = TW + t; j < nh; j += TW) {
      const unsigned oj = lo + (unsigned)halo[h0 + j];
      for (int w = 0; w < NW; ++w) cp_async8(s + w * tj + TW + j, sp.p[w] + oj);
    }
    cp_async_commit();
  }
};

}  // namespace pdg
