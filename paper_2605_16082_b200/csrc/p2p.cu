// Device-initiated halo exchange over NVLink peer memory ("LSA peer stores
// (2D)"; SPEC.md:574-587 halo_exchange).  No NCCL and no host involvement.
//
// Every rank owns one device buffer ("inbox") holding, per peer it receives from, an epoch flag
// and a double-buffered receive window [2][max_planes][nrecv].  The buffer is mapped by the peers
// (CUDA IPC between processes; the raw pointer for ranks that share a process).  An exchange is
// two launches whatever the number of peers (grid.y = peer):
//     start:  the blocks of peer i pack the boundary columns of every field and STORE them
//             straight into peer i's window (parity = epoch & 1) through the peer pointer; the
//             last of them to finish publishes the new epoch in peer i's flag (release, system
//             scope) -- pack, transfer and signal in one launch;
//     finish: the blocks of peer i wait (acquire, system scope) until its flag reaches the
//             expected epoch and scatter the window into the ghost slots; the last of them
//             advances the expected epoch.
// The epochs live in device memory (sent / expected counters advanced by the kernels), so the
// launches carry no per-exchange host values and a captured CUDA graph can be replayed.
// Two windows suffice: ghost rings are symmetric (a rank that sends to a peer also receives from
// it), so a sender cannot run two exchanges ahead of a receiver that still reads a window.
#include <algorithm>
#include <cstring>
#include <vector>

#include "ctx.cuh"

namespace {
constexpr int kFlagBytes = 128;  // one flag per cache line

struct Peer {
  int rank = 0, nsend = 0, nrecv = 0;
  int* sidx = nullptr;            // own columns to send (device)
  int* ridx = nullptr;            // own ghost slots to fill (device)
  long long win_off = 0;          // offset of my receive window for this peer in MY inbox (bytes)
  long long flag_off = 0;         // offset of my flag for this peer in MY inbox (bytes)
  char* remote = nullptr;         // the peer's inbox (mapped)
  bool ipc_opened = false;
  long long rwin_off = 0, rflag_off = 0;  // my window / flag inside the PEER's inbox
};
}  // namespace

namespace pdg {
// what the all-peer kernels need per peer (device array, refreshed by pdg_p2p_connect)
struct PeerDev {
  const int* sidx;
  const int* ridx;
  int nsend, nrecv;
  double* rwin;          // my window in the peer's inbox
  unsigned* rflag;       // my flag in the peer's inbox
  const double* win;     // the peer's window in my inbox
  const unsigned* flag;  // the peer's flag in my inbox
};
}  // namespace pdg

struct pdg_p2p {
  int nt = 0, max_planes = 0, device = 0;
  std::vector<Peer> peers;
  char* inbox = nullptr;
  size_t inbox_bytes = 0;
  unsigned* counters = nullptr;   // [2][npeers] sent / expected epochs (device)
  unsigned* done = nullptr;       // [2][npeers] blocks finished pushing / pulling the current epoch
  pdg::PeerDev* pdev = nullptr;   // [npeers] (device)
  int max_send = 0, max_recv = 0;
  long long planes = 0;           // planes of the exchange in flight (host check)
};

namespace pdg {
constexpr unsigned long long kP2PTimeoutNs = 60ull * 1000000000ull;
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

struct P2PFields {
  const double* f[8];
  long long np[8];
  int nf;
};

// every peer in one launch: blockIdx.y = peer, blockIdx.x strides over its (plane, column) words
__global__ void k_p2p_push_all(P2PFields F, int nt, const PeerDev* __restrict__ pd, long long wplanes,
                               long long tot, unsigned* sent, unsigned* done) {
  const int i = blockIdx.y;
  const PeerDev q = pd[i];
  const unsigned epoch = sent[i] + 1;   // advanced only by the last block of this peer
  const int n = q.nsend > 0 ? q.nsend : 1;
  double* win = q.rwin + (epoch & 1u) * (wplanes * q.nsend);
  const long long total = tot * q.nsend;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long p = t / n;
    const int c = (int)(t - p * n);
    int f = 0;
    while (p >= F.np[f]) p -= F.np[f++];
    win[t] = F.f[f][p * nt + q.sidx[c]];
  }
  // one system-scope fence per peer, not per block: each block orders its stores at GPU scope
  // (the barrier makes them the fencing thread's, a fence is cumulative) before counting itself
  // done; the last block -- which has observed every count -- fences at system scope and releases
  // the flag, so the peer's acquire sees every block's stores (a per-block MEMBAR.SYS measured
  // 16 us per push launch against 5 us for the pull)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(done + i, 1u);
    if (prev == gridDim.x - 1) {   // every block of this peer has stored and fenced: publish
      __threadfence_system();
      done[i] = 0u;
      sent[i] = epoch;
      st_release_sys(q.rflag, epoch);
    }
  }
}

__global__ void k_p2p_pull_all(P2PFields F, int nt, const PeerDev* __restrict__ pd, long long wplanes,
                               long long tot, unsigned* expected, unsigned* done) {
  const int i = blockIdx.y;
  const PeerDev q = pd[i];
  const unsigned want = expected[i] + 1;   // advanced only by the last block of this peer
  if (threadIdx.x == 0) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys(q.flag) < want) {
      __nanosleep(200);
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > kP2PTimeoutNs) __trap();
    }
  }
  __syncthreads();
  const int n = q.nrecv > 0 ? q.nrecv : 1;
  const double* win = q.win + (want & 1u) * (wplanes * q.nrecv);
  const long long total = tot * q.nrecv;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    long long p = t / n;
    const int c = (int)(t - p * n);
    int f = 0;
    while (p >= F.np[f]) p -= F.np[f++];
    const_cast<double*>(F.f[f])[p * nt + q.ridx[c]] = __ldcg(win + t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(done + i, 1u);
    if (prev == gridDim.x - 1) {   // every block of this peer has read `want`: advance it
      done[i] = 0u;
      expected[i] = want;
    }
  }
}
}  // namespace pdg

using namespace pdg;

static bool fields_of(int nf, double* const* fields, const long long* nplanes, P2PFields& F, long long& tot) {
  if (nf < 1 || nf > 8) return false;
  F.nf = nf;
  tot = 0;
  for (int f = 0; f < nf; ++f) {
    F.f[f] = fields[f];
    F.np[f] = nplanes[f];
    tot += nplanes[f];
  }
  for (int f = nf; f < 8; ++f) {
    F.f[f] = nullptr;
    F.np[f] = 1LL << 62;
  }
  return true;
}

extern "C" {

int pdg_p2p_destroy(pdg_p2p* p) {
  if (!p) return PDG_OK;
  cudaSetDevice(p->device);
  for (auto& q : p->peers) {
    cudaFree(q.sidx);
    cudaFree(q.ridx);
    if (q.ipc_opened) cudaIpcCloseMemHandle(q.remote);
  }
  cudaFree(p->inbox);
  cudaFree(p->counters);
  cudaFree(p->done);
  cudaFree(p->pdev);
  delete p;
  return PDG_OK;
}

// peers / nsend / send_idx / nrecv / recv_idx: HOST arrays (the plan copies the lists)
int pdg_p2p_create(int nt, int npeers, const int* peers, const int* nsend, const int* const* send_idx,
                   const int* nrecv, const int* const* recv_idx, int max_planes, int device, pdg_p2p** out) {
  if (npeers < 0 || max_planes < 1 || nt < 0) return PDG_ERR_SHAPE;
  cudaSetDevice(device);
  auto* p = new pdg_p2p;
  p->nt = nt;
  p->max_planes = max_planes;
  p->device = device;
  size_t off = (size_t)npeers * kFlagBytes;
  bool ok = true;
  for (int i = 0; ok && i < npeers; ++i) {
    Peer q;
    q.rank = peers[i];
    q.nsend = nsend[i];
    q.nrecv = nrecv[i];
    q.flag_off = (long long)i * kFlagBytes;
    q.win_off = (long long)off;
    off += ((size_t)2 * max_planes * nrecv[i] * sizeof(double) + 255) & ~(size_t)255;
    ok = cudaMalloc(&q.sidx, sizeof(int) * (q.nsend + 1)) == cudaSuccess &&
         cudaMalloc(&q.ridx, sizeof(int) * (q.nrecv + 1)) == cudaSuccess;
    if (ok && q.nsend) ok = cudaMemcpy(q.sidx, send_idx[i], sizeof(int) * q.nsend, cudaMemcpyHostToDevice) == cudaSuccess;
    if (ok && q.nrecv) ok = cudaMemcpy(q.ridx, recv_idx[i], sizeof(int) * q.nrecv, cudaMemcpyHostToDevice) == cudaSuccess;
    p->peers.push_back(q);
  }
  p->inbox_bytes = off + 256;
  ok = ok && cudaMalloc(&p->inbox, p->inbox_bytes) == cudaSuccess &&
       cudaMemset(p->inbox, 0, (size_t)npeers * kFlagBytes + 256) == cudaSuccess &&
       cudaMalloc(&p->counters, sizeof(unsigned) * (2 * npeers + 1)) == cudaSuccess &&
       cudaMemset(p->counters, 0, sizeof(unsigned) * (2 * npeers + 1)) == cudaSuccess &&
       cudaMalloc(&p->done, sizeof(unsigned) * (2 * npeers + 1)) == cudaSuccess &&
       cudaMemset(p->done, 0, sizeof(unsigned) * (2 * npeers + 1)) == cudaSuccess &&
       cudaMalloc(&p->pdev, sizeof(PeerDev) * (npeers + 1)) == cudaSuccess;
  for (const auto& q : p->peers) {
    p->max_send = std::max(p->max_send, q.nsend);
    p->max_recv = std::max(p->max_recv, q.nrecv);
  }
  if (!ok) {
    pdg_p2p_destroy(p);
    return PDG_ERR_CUDA;
  }
  *out = p;
  return PDG_OK;
}

// what the peers need to map my inbox: the IPC handle (64 bytes; ipc_handle may be null), the raw
// device pointer (same-process ranks), and per peer slot the offsets of my window and flag for it
int pdg_p2p_local(pdg_p2p* p, void* ipc_handle, void** raw, long long* win_off, long long* flag_off) {
  if (!p) return PDG_ERR_SHAPE;
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, p->inbox) != cudaSuccess) return PDG_ERR_CUDA;
    memcpy(ipc_handle, &h, sizeof(h));
  }
  if (raw) *raw = p->inbox;
  for (size_t i = 0; i < p->peers.size(); ++i) {
    win_off[i] = p->peers[i].win_off;
    flag_off[i] = p->peers[i].flag_off;
  }
  return PDG_OK;
}

// map peer slot `slot`'s inbox: from its IPC handle (another process), or its raw pointer (same
// process; ipc_handle null); win_off / flag_off locate MY window and flag inside it
int pdg_p2p_connect(pdg_p2p* p, int slot, const void* ipc_handle, void* raw, long long win_off, long long flag_off) {
  if (!p || slot < 0 || slot >= (int)p->peers.size()) return PDG_ERR_SHAPE;
  Peer& q = p->peers[slot];
  cudaSetDevice(p->device);
  if (ipc_handle) {
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    void* ptr = nullptr;
    if (cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return PDG_ERR_CUDA;
    q.remote = (char*)ptr;
    q.ipc_opened = true;
  } else {
    q.remote = (char*)raw;
  }
  q.rwin_off = win_off;
  q.rflag_off = flag_off;
  PeerDev d{q.sidx, q.ridx, q.nsend, q.nrecv, (double*)(q.remote + win_off), (unsigned*)(q.remote + flag_off),
            (const double*)(p->inbox + q.win_off), (const unsigned*)(p->inbox + q.flag_off)};
  if (cudaMemcpy(p->pdev + slot, &d, sizeof(d), cudaMemcpyHostToDevice) != cudaSuccess) return PDG_ERR_CUDA;
  return PDG_OK;
}

int pdg_p2p_start(pdg_p2p* p, int nf, double* const* fields, const long long* nplanes, void* stream) {
  if (!p) return PDG_ERR_SHAPE;
  P2PFields F;
  long long tot = 0;
  if (!fields_of(nf, fields, nplanes, F, tot) || tot > p->max_planes) return PDG_ERR_SHAPE;
  const cudaStream_t s = (cudaStream_t)stream;
  const int np = (int)p->peers.size();
  for (const auto& q : p->peers)
    if (!q.remote) return PDG_ERR_SHAPE;
  if (np > 0) {
    const int nb = (int)std::min<long long>(std::max<long long>(1, (tot * p->max_send + 255) / 256),
                                            std::max(1, 4 * 148 / np));
    k_p2p_push_all<<<dim3(nb, np), 256, 0, s>>>(F, p->nt, p->pdev, p->max_planes, tot, p->counters, p->done);
  }
  p->planes = tot;
  return check_launch_noctx();
}

int pdg_p2p_finish(pdg_p2p* p, int nf, double* const* fields, const long long* nplanes, void* stream) {
  if (!p) return PDG_ERR_SHAPE;
  P2PFields F;
  long long tot = 0;
  if (!fields_of(nf, fields, nplanes, F, tot) || tot != p->planes) return PDG_ERR_SHAPE;
  const cudaStream_t s = (cudaStream_t)stream;
  const int np = (int)p->peers.size();
  if (np > 0) {
    const int nb = (int)std::min<long long>(std::max<long long>(1, (tot * p->max_recv + 255) / 256),
                                            std::max(1, 4 * 148 / np));
    k_p2p_pull_all<<<dim3(nb, np), 256, 0, s>>>(F, p->nt, p->pdev, p->max_planes, tot, p->counters + np,
                                                 p->done + np);
  }
  return check_launch_noctx();
}

}  // extern "C"
