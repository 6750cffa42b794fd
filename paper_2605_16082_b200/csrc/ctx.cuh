// Context object behind the opaque pdg_ctx handle (host side).
#pragma once
#include <vector>

#include "common.cuh"

struct pdg_ctx {
  int device = 0;
  int nt = 0;
  int nown = 0;   // owned (computed) columns: 0..nown-1; the rest are ghost columns (partitioned runs)
  int L = 0;
  double min_edge = 0.0;
  double *j2d = nullptr, *dphx = nullptr, *dphy = nullptr, *elen = nullptr, *enx = nullptr, *eny = nullptr,
         *b = nullptr, *fracs = nullptr;
  int *nbr = nullptr, *nbrk = nullptr, *btag = nullptr, *ninfo = nullptr;
  pdg_err* err = nullptr;     // device error word
  double* red = nullptr;      // reduction scratch (device)
  double* ws2d = nullptr;     // 2D subcycle workspace: 2 stage states + q0
  double* ws3d = nullptr;     // 3D workspace (block-Thomas propagation tiles), momentum solves
  size_t ws3d_doubles = 0;
  double* ws3t = nullptr;     // a second one for the tracer solves, so the two can run concurrently
  size_t ws3t_doubles = 0;
  long long launches = 0;
  std::vector<double> fracs_host;
  // tile maps of the shared-memory-staged face kernels (int3d.cu k_*_t): for tiles of tw
  // consecutive owned columns, the neighbour slot of every (edge, column) and each tile's halo;
  // one map per tile width (64, 128)
  std::vector<int> nbr_host, btag_host;   // (nt,3) row-major host copies
  struct TileMap {
    int tw = 0, nown = -1, nh_max = 0;
    int *tslot = nullptr, *halo = nullptr, *hoff = nullptr;
  } tiles[2];

  pdg::DMesh view() const {
    pdg::DMesh m;
    m.nt = nt;
    m.nown = nown;
    m.L = L;
    m.j2d = j2d;
    m.dphx = dphx;
    m.dphy = dphy;
    m.elen = elen;
    m.enx = enx;
    m.eny = eny;
    m.b = b;
    m.nbr = nbr;
    m.nbrk = nbrk;
    m.btag = btag;
    m.fracs = fracs;
    m.ninfo = ninfo;
    m.err = err;
    return m;
  }
  // per-column sigma-layer constants of the kh == 0 vertical kernels ([8][nt], columns.cu k_vcol)
  double* vc = nullptr;
  double* vcol() {
    if (!vc && cudaMalloc(&vc, (size_t)8 * nt * sizeof(double)) != cudaSuccess) vc = nullptr;
    return vc;
  }
  // grows the 3D workspace (never on the hot path once sized)
  static double* grow(double*& p, size_t& have, size_t n) {
    if (n > have) {
      if (p) cudaFree(p);
      p = nullptr;
      if (cudaMalloc(&p, n * sizeof(double)) != cudaSuccess) {
        have = 0;
        return nullptr;
      }
      have = n;
    }
    return p;
  }
  double* ws3(size_t n, int ncomp = 2) { return ncomp == 1 ? grow(ws3t, ws3t_doubles, n) : grow(ws3d, ws3d_doubles, n); }
};

namespace pdg {
// builds / reuses the tile map of width tw (64 or 128; host work, never during capture); nullptr on failure
const pdg_ctx::TileMap* ensure_tiles(pdg_ctx* ctx, int tw);
int check_launch(pdg_ctx* ctx);  // returns PDG_OK or PDG_ERR_CUDA and counts the launch
int check_launch_noctx();
}  // namespace pdg
