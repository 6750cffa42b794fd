// Halo exchange of a horizontally partitioned run over NCCL (pdg_comm_init,
// pdg_halo_*; SPEC.md:574-587 halo_exchange / boundary-first overlap).
//
// One process per GPU.  The library binds the NCCL the process already uses (torch's pip NCCL,
// 2.28.x) at run time with dlopen (pdg_comm_load), so one process never holds two NCCLs and the
// .so has no link-time NCCL dependency.  A halo plan holds, per peer rank, the device index lists
// of the owned columns to send and of the ghost slots to fill, and message buffers sized for the
// largest exchange.  An exchange is
//     start:  pack (one kernel for every field and peer, grid.y = peer) on the caller's stream ->
//             event -> grouped ncclSend/ncclRecv to every peer on the plan's communication stream
//     finish: the caller's stream waits for the communication -> unpack (one kernel)
// everything stream ordered, so the caller launches interior work between start and finish and
// the whole partitioned step can be captured in one CUDA graph (NCCL point-to-point operations
// are capturable; the event fork/join becomes graph edges).
#include <dlfcn.h>

#include <cstdio>
#include <algorithm>
#include <cstring>

#include <vector>

#include "ctx.cuh"

namespace {
// the few NCCL types the exchange uses (stable ABI, nccl.h)
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat64 = 8;

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
char g_nccl_err[256] = "";

template <typename F>
bool bind(F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(g_nccl.h, name));
  return f != nullptr;
}
int nccl_fail(ncclResult_t r) {
  snprintf(g_nccl_err, sizeof(g_nccl_err), "NCCL error %d: %s", r,
           g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "?");
  return PDG_ERR_CUDA;
}
}  // namespace

struct pdg_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, device = 0;
  cudaStream_t cs = nullptr;  // communication stream (high priority)
};

namespace pdg {
struct HaloFields {
  const double* f[8];
  long long np[8];
};
struct HaloPeerDev {                    // per peer: index lists and message buffers (device)
  const int* sidx;
  const int* ridx;
  int nsend, nrecv;
  double* sbuf;
  double* rbuf;
};
// every field's boundary values for every peer (blockIdx.y = peer) into its [planes][nsend] buffer
__global__ void k_halo_pack_all(HaloFields F, int nt, const HaloPeerDev* __restrict__ pd, long long tot) {
  const HaloPeerDev q = pd[blockIdx.y];
  const int n = q.nsend;
  const long long total = tot * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long p = t / n;
    const int c = (int)(t - p * n);
    int f = 0;
    while (p >= F.np[f]) p -= F.np[f++];
    q.sbuf[t] = F.f[f][p * nt + q.sidx[c]];
  }
}
__global__ void k_halo_unpack_all(HaloFields F, int nt, const HaloPeerDev* __restrict__ pd, long long tot) {
  const HaloPeerDev q = pd[blockIdx.y];
  const int n = q.nrecv;
  const long long total = tot * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long p = t / n;
    const int c = (int)(t - p * n);
    int f = 0;
    while (p >= F.np[f]) p -= F.np[f++];
    const_cast<double*>(F.f[f])[p * nt + q.ridx[c]] = q.rbuf[t];
  }
}
}  // namespace pdg

struct pdg_halo_plan {
  pdg_comm* c = nullptr;
  int nt = 0, max_planes = 0;
  std::vector<int> peers, nsend, nrecv;
  std::vector<int*> sidx, ridx;         // device index lists (copies owned by the plan)
  std::vector<double*> sbuf, rbuf;      // [max_planes][n] per peer
  pdg::HaloPeerDev* pdev = nullptr;     // the same, per peer, for the all-peer kernels (device)
  int max_send = 0, max_recv = 0;
  cudaEvent_t packed = nullptr, done = nullptr;
  long long planes = 0;                 // planes of the exchange in flight
};

static bool halo_fields(int nf, double* const* fields, const long long* nplanes, pdg::HaloFields& F, long long& tot) {
  if (nf < 1 || nf > 8) return false;
  tot = 0;
  for (int f = 0; f < 8; ++f) {
    F.f[f] = f < nf ? fields[f] : nullptr;
    F.np[f] = f < nf ? nplanes[f] : (1LL << 62);
    if (f < nf) tot += nplanes[f];
  }
  return true;
}

using namespace pdg;
extern "C" {

const char* pdg_comm_error_string(void) { return g_nccl_err; }

int pdg_comm_load(const char* libnccl_path) {
  if (g_nccl.h) return PDG_OK;
  g_nccl.h = dlopen(libnccl_path, RTLD_NOW | RTLD_GLOBAL);
  if (!g_nccl.h) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "dlopen(%s) failed: %s", libnccl_path, dlerror());
    return PDG_ERR_CUDA;
  }
  const bool ok = bind(g_nccl.GetUniqueId, "ncclGetUniqueId") && bind(g_nccl.CommInitRank, "ncclCommInitRank") &&
                  bind(g_nccl.CommDestroy, "ncclCommDestroy") && bind(g_nccl.Send, "ncclSend") &&
                  bind(g_nccl.Recv, "ncclRecv") && bind(g_nccl.GroupStart, "ncclGroupStart") &&
                  bind(g_nccl.GroupEnd, "ncclGroupEnd") && bind(g_nccl.GetErrorString, "ncclGetErrorString");
  if (!ok) {
    snprintf(g_nccl_err, sizeof(g_nccl_err), "%s lacks the NCCL point-to-point API", libnccl_path);
    dlclose(g_nccl.h);
    g_nccl = NcclApi{};
    return PDG_ERR_CUDA;
  }
  return PDG_OK;
}

int pdg_comm_unique_id(void* id128) {
  if (!g_nccl.h) return PDG_ERR_CUDA;
  ncclUniqueId id;
  const ncclResult_t r = g_nccl.GetUniqueId(&id);
  if (r != 0) return nccl_fail(r);
  memcpy(id128, &id, sizeof(id));
  return PDG_OK;
}

int pdg_comm_init(const void* id128, int rank, int nranks, int device, pdg_comm** out) {
  if (!g_nccl.h) return PDG_ERR_CUDA;
  if (rank < 0 || rank >= nranks) return PDG_ERR_SHAPE;
  cudaSetDevice(device);
  auto* c = new pdg_comm;
  c->rank = rank;
  c->nranks = nranks;
  c->device = device;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  const ncclResult_t r = g_nccl.CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    delete c;
    return nccl_fail(r);
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if (cudaStreamCreateWithPriority(&c->cs, cudaStreamNonBlocking, hi) != cudaSuccess) {
    g_nccl.CommDestroy(c->comm);
    delete c;
    return PDG_ERR_CUDA;
  }
  *out = c;
  return PDG_OK;
}

int pdg_comm_destroy(pdg_comm* c) {
  if (!c) return PDG_OK;
  if (c->cs) cudaStreamDestroy(c->cs);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  delete c;
  return PDG_OK;
}

int pdg_halo_plan_destroy(pdg_halo_plan* p) {
  if (!p) return PDG_OK;
  for (auto* q : p->sidx) cudaFree(q);
  for (auto* q : p->ridx) cudaFree(q);
  for (auto* q : p->sbuf) cudaFree(q);
  for (auto* q : p->rbuf) cudaFree(q);
  cudaFree(p->pdev);
  if (p->packed) cudaEventDestroy(p->packed);
  if (p->done) cudaEventDestroy(p->done);
  delete p;
  return PDG_OK;
}

// send_idx / recv_idx: HOST arrays of HOST int32 lists (the plan copies them to the device)
int pdg_halo_plan_create(pdg_comm* c, int nt, int npeers, const int* peers, const int* nsend,
                         const int* const* send_idx, const int* nrecv, const int* const* recv_idx, int max_planes,
                         pdg_halo_plan** out) {
  if (!c || npeers < 0 || max_planes < 1) return PDG_ERR_SHAPE;
  cudaSetDevice(c->device);
  auto* p = new pdg_halo_plan;
  p->c = c;
  p->nt = nt;
  p->max_planes = max_planes;
  bool ok = cudaEventCreateWithFlags(&p->packed, cudaEventDisableTiming) == cudaSuccess &&
            cudaEventCreateWithFlags(&p->done, cudaEventDisableTiming) == cudaSuccess;
  for (int i = 0; ok && i < npeers; ++i) {
    if (peers[i] < 0 || peers[i] >= c->nranks) ok = false;
    p->peers.push_back(peers[i]);
    p->nsend.push_back(nsend[i]);
    p->nrecv.push_back(nrecv[i]);
    int *si = nullptr, *ri = nullptr;
    double *sb = nullptr, *rb = nullptr;
    ok = ok && cudaMalloc(&si, sizeof(int) * (nsend[i] + 1)) == cudaSuccess &&
         cudaMalloc(&ri, sizeof(int) * (nrecv[i] + 1)) == cudaSuccess &&
         cudaMalloc(&sb, sizeof(double) * ((size_t)max_planes * nsend[i] + 1)) == cudaSuccess &&
         cudaMalloc(&rb, sizeof(double) * ((size_t)max_planes * nrecv[i] + 1)) == cudaSuccess;
    p->sidx.push_back(si);
    p->ridx.push_back(ri);
    p->sbuf.push_back(sb);
    p->rbuf.push_back(rb);
    if (ok && nsend[i]) ok = cudaMemcpy(si, send_idx[i], sizeof(int) * nsend[i], cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && nrecv[i]) ok = cudaMemcpy(ri, recv_idx[i], sizeof(int) * nrecv[i], cudaMemcpyHostToDevice) == cudaSuccess;
  }
  if (ok) {
    std::vector<HaloPeerDev> d;
    for (int i = 0; i < npeers; ++i) {
      d.push_back({p->sidx[i], p->ridx[i], p->nsend[i], p->nrecv[i], p->sbuf[i], p->rbuf[i]});
      p->max_send = std::max(p->max_send, p->nsend[i]);
      p->max_recv = std::max(p->max_recv, p->nrecv[i]);
    }
    ok = cudaMalloc(&p->pdev, sizeof(HaloPeerDev) * (npeers + 1)) == cudaSuccess &&
         (npeers == 0 ||
          cudaMemcpy(p->pdev, d.data(), sizeof(HaloPeerDev) * npeers, cudaMemcpyHostToDevice) == cudaSuccess);
  }
  if (!ok) {
    pdg_halo_plan_destroy(p);
    return PDG_ERR_CUDA;
  }
  *out = p;
  return PDG_OK;
}

// pack every field's boundary values for every peer, then post the grouped sends / receives on the
// communication stream (after the pack).  fields: HOST array of nf DEVICE pointers, nplanes[f]
// planes of nt doubles each.
int pdg_halo_start(pdg_halo_plan* p, int nf, double* const* fields, const long long* nplanes, void* stream) {
  if (!p) return PDG_ERR_SHAPE;
  HaloFields F;
  long long tot = 0;
  if (!halo_fields(nf, fields, nplanes, F, tot) || tot > p->max_planes) return PDG_ERR_SHAPE;
  const cudaStream_t s = (cudaStream_t)stream;
  const int np = (int)p->peers.size();
  if (np > 0 && p->max_send > 0) {
    const int nb = (int)std::min<long long>((tot * p->max_send + 255) / 256, std::max(1, 4 * 148 / np));
    k_halo_pack_all<<<dim3(nb, np), 256, 0, s>>>(F, p->nt, p->pdev, tot);
    if (cudaGetLastError() != cudaSuccess) return PDG_ERR_CUDA;
  }
  p->planes = tot;
  if (cudaEventRecord(p->packed, s) != cudaSuccess) return PDG_ERR_CUDA;
  const cudaStream_t cs = p->c->cs;
  if (cudaStreamWaitEvent(cs, p->packed, 0) != cudaSuccess) return PDG_ERR_CUDA;
  ncclResult_t r = g_nccl.GroupStart();
  if (r != 0) return nccl_fail(r);
  for (size_t i = 0; i < p->peers.size(); ++i) {
    if (p->nrecv[i] && (r = g_nccl.Recv(p->rbuf[i], (size_t)tot * p->nrecv[i], kNcclFloat64, p->peers[i], p->c->comm, cs)))
      break;
    if (p->nsend[i] && (r = g_nccl.Send(p->sbuf[i], (size_t)tot * p->nsend[i], kNcclFloat64, p->peers[i], p->c->comm, cs)))
      break;
  }
  const ncclResult_t r2 = g_nccl.GroupEnd();
  if (r != 0) return nccl_fail(r);
  if (r2 != 0) return nccl_fail(r2);
  if (cudaEventRecord(p->done, cs) != cudaSuccess) return PDG_ERR_CUDA;
  return PDG_OK;
}

// the caller's stream waits for the transfers and fills the ghost slots
int pdg_halo_finish(pdg_halo_plan* p, int nf, double* const* fields, const long long* nplanes, void* stream) {
  if (!p) return PDG_ERR_SHAPE;
  const cudaStream_t s = (cudaStream_t)stream;
  if (cudaStreamWaitEvent(s, p->done, 0) != cudaSuccess) return PDG_ERR_CUDA;
  HaloFields F;
  long long tot = 0;
  if (!halo_fields(nf, fields, nplanes, F, tot) || tot != p->planes) return PDG_ERR_SHAPE;
  const int np = (int)p->peers.size();
  if (np > 0 && p->max_recv > 0) {
    const int nb = (int)std::min<long long>((tot * p->max_recv + 255) / 256, std::max(1, 4 * 148 / np));
    k_halo_unpack_all<<<dim3(nb, np), 256, 0, s>>>(F, p->nt, p->pdev, tot);
    if (cudaGetLastError() != cudaSuccess) return PDG_ERR_CUDA;
  }
  return PDG_OK;
}

// SURVEY.md section 8b names: blocking exchanges of the 2D sub-cycle state (the three C3 fields
// eta, Qx, Qy: 9 planes, the all-rings plan) and of ring-1 3D fields (start + finish)
int pdg_halo_2d(pdg_halo_plan* p, double* state9, void* stream) {
  double* f[1] = {state9};
  const long long np[1] = {9};
  const int rc = pdg_halo_start(p, 1, f, np, stream);
  return rc != PDG_OK ? rc : pdg_halo_finish(p, 1, f, np, stream);
}
int pdg_halo_3d(pdg_halo_plan* p, int nf, double* const* fields, const long long* nplanes, void* stream) {
  const int rc = pdg_halo_start(p, nf, fields, nplanes, stream);
  return rc != PDG_OK ? rc : pdg_halo_finish(p, nf, fields, nplanes, stream);
}

}  // extern "C"
