// Context lifetime, mesh upload (reference (nt,3) host layout -> device SoA), error word.
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.cuh"

static thread_local char g_errbuf[512] = "";
static int g_tune[pdg::TUNE_NKEYS] = {1, 1, 1, 3, 4, 8, 8, 4, 0, 128, 0, 128, 1, 1, 0, 0};  // measured: scripts/tune.py

namespace pdg {
int tune_get(int key) { return (key >= 0 && key < TUNE_NKEYS) ? g_tune[key] : 1; }
}  // namespace pdg
static long long g_noctx_launches = 0;

namespace pdg {
int check_launch(pdg_ctx* ctx) {
  if (ctx) ctx->launches++;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_errbuf, sizeof(g_errbuf), "%s", cudaGetErrorString(e));
    return PDG_ERR_CUDA;
  }
  return PDG_OK;
}
int check_launch_noctx() {
  g_noctx_launches++;
  return check_launch(nullptr);
}
}  // namespace pdg

template <typename T>
static int upload_soa3(const T* host_nt3, int nt, T** dev) {
  // (nt,3) -> [3][nt]
  std::vector<T> tmp((size_t)3 * nt);
  for (int c = 0; c < nt; ++c)
    for (int k = 0; k < 3; ++k) tmp[(size_t)k * nt + c] = host_nt3[(size_t)c * 3 + k];
  if (cudaMalloc(dev, tmp.size() * sizeof(T)) != cudaSuccess) return PDG_ERR_CUDA;
  if (cudaMemcpy(*dev, tmp.data(), tmp.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return PDG_ERR_CUDA;
  return PDG_OK;
}

static int upload_int3(const int64_t* host_nt3, int nt, int** dev) {
  std::vector<int> tmp((size_t)3 * nt);
  for (int c = 0; c < nt; ++c)
    for (int k = 0; k < 3; ++k) tmp[(size_t)k * nt + c] = (int)host_nt3[(size_t)c * 3 + k];
  if (cudaMalloc(dev, tmp.size() * sizeof(int)) != cudaSuccess) return PDG_ERR_CUDA;
  if (cudaMemcpy(*dev, tmp.data(), tmp.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess)
    return PDG_ERR_CUDA;
  return PDG_OK;
}

extern "C" {

int pdg_ctx_create(const pdg_mesh_desc* d, int device, pdg_ctx** out) {
  *out = nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return pdg::check_launch(nullptr), PDG_ERR_CUDA;
  pdg_ctx* c = new pdg_ctx();
  c->device = device;
  c->nt = d->nt;
  c->nown = d->nt;
  c->min_edge = d->min_edge;
  int nt = d->nt;
  int rc = PDG_OK;
  rc |= cudaMalloc(&c->j2d, nt * sizeof(double)) != cudaSuccess;
  rc |= cudaMemcpy(c->j2d, d->j2d, nt * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess;
  rc |= upload_soa3(d->dphx, nt, &c->dphx);
  rc |= upload_soa3(d->dphy, nt, &c->dphy);
  rc |= upload_soa3(d->elen, nt, &c->elen);
  rc |= upload_soa3(d->enx, nt, &c->enx);
  rc |= upload_soa3(d->eny, nt, &c->eny);
  rc |= upload_soa3(d->b, nt, &c->b);
  rc |= upload_int3(d->nbr, nt, &c->nbr);
  c->nbr_host.resize((size_t)3 * nt);
  c->btag_host.resize((size_t)3 * nt);
  for (size_t i = 0; i < (size_t)3 * nt; ++i) {
    c->nbr_host[i] = (int)d->nbr[i];
    c->btag_host[i] = (int)d->btag[i];
  }
  rc |= upload_int3(d->nbrk, nt, &c->nbrk);
  rc |= upload_int3(d->btag, nt, &c->btag);
  {
    std::vector<int> info((size_t)3 * nt);
    for (int e = 0; e < nt; ++e)
      for (int k = 0; k < 3; ++k) {
        const long long nb = d->nbr[(size_t)e * 3 + k], nk = d->nbrk[(size_t)e * 3 + k], tg = d->btag[(size_t)e * 3 + k];
        info[(size_t)k * nt + e] = (int)(((nb > 0 ? nb : 0) << 4) | ((nk > 0 ? nk : 0) << 2) | (tg & 3));
      }
    rc |= cudaMalloc(&c->ninfo, info.size() * sizeof(int)) != cudaSuccess;
    rc |= cudaMemcpy(c->ninfo, info.data(), info.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess;
  }
  rc |= cudaMalloc(&c->err, sizeof(pdg_err)) != cudaSuccess;
  rc |= cudaMemset(c->err, 0, sizeof(pdg_err)) != cudaSuccess;
  rc |= cudaMalloc(&c->red, 4096 * sizeof(double)) != cudaSuccess;
  rc |= cudaMalloc(&c->ws2d, (size_t)(9 + 9 + 6) * nt * sizeof(double)) != cudaSuccess;
  if (rc) {
    snprintf(g_errbuf, sizeof(g_errbuf), "pdg_ctx_create: %s", cudaGetErrorString(cudaGetLastError()));
    pdg_ctx_destroy(c);
    return PDG_ERR_CUDA;
  }
  *out = c;
  return PDG_OK;
}

int pdg_ctx_destroy(pdg_ctx* c) {
  if (!c) return PDG_OK;
  void* ptrs[] = {c->j2d, c->dphx, c->dphy, c->elen, c->enx, c->eny, c->b, c->fracs, c->nbr, c->nbrk, c->btag,
                  c->ninfo, c->err, c->red, c->ws2d, c->ws3d, c->ws3t, c->tiles[0].tslot, c->tiles[0].halo,
                  c->tiles[0].hoff, c->tiles[1].tslot, c->tiles[1].halo, c->tiles[1].hoff,
                  c->vc};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete c;
  return PDG_OK;
}

int pdg_ctx_set_layers(pdg_ctx* c, int L, const double* fracs) {
  if (L < 1) return PDG_ERR_SHAPE;
  if ((long long)6 * L * c->nt >= (1LL << 32)) return PDG_ERR_SHAPE;  // 32-bit plane indices (col3d.cuh pix)
  if (c->fracs) cudaFree(c->fracs);
  c->fracs = nullptr;
  if (cudaMalloc(&c->fracs, (L + 1) * sizeof(double)) != cudaSuccess) return PDG_ERR_CUDA;
  if (cudaMemcpy(c->fracs, fracs, (L + 1) * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
    return PDG_ERR_CUDA;
  c->fracs_host.assign(fracs, fracs + L + 1);
  c->L = L;
  return PDG_OK;
}

}  // extern "C"

namespace pdg {
// Tiles of tw consecutive owned columns.  tslot[k][c] = e2 - c0 when the neighbour across edge k
// lies in c's own tile, tw + h when it is the tile's h-th halo column (first-seen order), -1 on
// boundary edges.  A face kernel stages the tile's and the halo's planes of a layer in shared
// memory and gathers every neighbour trace from there (no atomics, no scattered HBM reads).
const pdg_ctx::TileMap* ensure_tiles(pdg_ctx* c, int tw) {
  if (tw != 64 && tw != 128) return nullptr;
  pdg_ctx::TileMap& T = c->tiles[tw == 64 ? 0 : 1];
  if (T.tw == tw && T.nown == c->nown && T.tslot) return &T;
  const int nt = c->nt, nown = c->nown, ntile = (nown + tw - 1) / tw;
  std::vector<int> slot((size_t)3 * nt, -1), halo, hoff(ntile + 1, 0);
  int nh_max = 0;
  std::vector<int> seen;
  for (int b = 0; b < ntile; ++b) {
    const int c0 = b * tw, c1 = std::min(nown, c0 + tw);
    seen.clear();
    for (int e = c0; e < c1; ++e)
      for (int k = 0; k < 3; ++k) {
        if (c->btag_host[(size_t)e * 3 + k] != 0) continue;
        const int e2 = c->nbr_host[(size_t)e * 3 + k];
        if (e2 >= c0 && e2 < c1) {
          slot[(size_t)k * nt + e] = e2 - c0;
          continue;
        }
        int h = -1;
        for (size_t j = 0; j < seen.size(); ++j)
          if (seen[j] == e2) h = (int)j;
        if (h < 0) {
          h = (int)seen.size();
          seen.push_back(e2);
        }
        slot[(size_t)k * nt + e] = tw + h;
      }
    halo.insert(halo.end(), seen.begin(), seen.end());
    hoff[b + 1] = (int)halo.size();
    nh_max = std::max(nh_max, (int)seen.size());
  }
  if (halo.empty()) halo.push_back(0);
  for (int* p : {T.tslot, T.halo, T.hoff})
    if (p) cudaFree(p);
  T.tslot = T.halo = T.hoff = nullptr;
  T.tw = 0;
  int rc = 0;
  rc |= cudaMalloc(&T.tslot, slot.size() * sizeof(int)) != cudaSuccess;
  rc |= cudaMalloc(&T.halo, halo.size() * sizeof(int)) != cudaSuccess;
  rc |= cudaMalloc(&T.hoff, hoff.size() * sizeof(int)) != cudaSuccess;
  if (rc) return nullptr;
  rc |= cudaMemcpy(T.tslot, slot.data(), slot.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess;
  rc |= cudaMemcpy(T.halo, halo.data(), halo.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess;
  rc |= cudaMemcpy(T.hoff, hoff.data(), hoff.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess;
  if (rc) return nullptr;
  T.tw = tw;
  T.nown = nown;
  T.nh_max = nh_max;
  return &T;
}
}  // namespace pdg

extern "C" {

int pdg_ctx_set_owned(pdg_ctx* c, int nown) {
  if (nown < 0 || nown > c->nt) return PDG_ERR_SHAPE;
  c->nown = nown;
  return PDG_OK;
}

int pdg_last_error(pdg_ctx* c, void* stream, int* code, long long* i0, long long* i1, double* val) {
  pdg_err h;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemcpyAsync(&h, c->err, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess) return PDG_ERR_CUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) {
    snprintf(g_errbuf, sizeof(g_errbuf), "%s", cudaGetErrorString(cudaGetLastError()));
    return PDG_ERR_CUDA;
  }
  if (h.code != 0) cudaMemsetAsync(c->err, 0, sizeof(pdg_err), s);
  *code = h.code;
  *i0 = h.i0;
  *i1 = h.i1;
  *val = h.val;
  return PDG_OK;
}

const char* pdg_cuda_error_string(void) { return g_errbuf; }

int pdg_tune(int key, int value) {
  if (key < 0 || key >= pdg::TUNE_NKEYS) return PDG_ERR_SHAPE;
  int old = g_tune[key];
  if (value >= 0) g_tune[key] = value;
  return old;
}

long long pdg_launch_count(pdg_ctx* c) { return c ? c->launches : g_noctx_launches; }

}  // extern "C"
