"""Horizontal domain decomposition and halo exchange (no reference code exists).

decompose(mesh, P): contiguous ranges of the Hilbert order balanced by prism count (weights =
layers per column) with a greedy prefix split, plus a one-ring ghost layer = every column that
shares an edge with an owned column.  Local numbering: owned columns first
(in global order), then ghosts (ascending global id).  The send/recv maps of every pair of
ranks list the same global ids in the same (ascending) order, so a halo message is a plain
[plane][i] block.

Because every assembly kernel is gather-only, a partitioned run reproduces the P = 1 run
bitwise (tests/test_partition*.py).

Transports: `DistHalo` (one process per GPU, torch.distributed send/recv -- NCCL over NVLink on
the GPU box, gloo on CPU) and `VirtualGroup` (P ranks in one process on one device; messages are
device-to-device copies) -- the latter makes the partitioned path testable on a single GPU.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np

from .errors import MapMismatch, TooManyRanks

GHOST_DEPTH = 3   # ghost rings of a partition: the 2D sub-cycle exchanges once per substep


@dataclass
class Part:
    rank: int
    nparts: int
    lo: int                     # owned global range [lo, hi)
    hi: int
    ghosts: np.ndarray          # global ids of ghost columns (ascending; all rings)
    send: dict = field(default_factory=dict)   # peer -> local indices (owned) to send (all rings)
    recv: dict = field(default_factory=dict)   # peer -> local indices (ghost slots) to fill (all rings)
    ring: np.ndarray = None     # ring (1..depth) of every ghost
    send1: dict = field(default_factory=dict)  # the same restricted to ring-1 ghosts (3D exchanges)
    recv1: dict = field(default_factory=dict)

    @property
    def n_own(self) -> int:
        return self.hi - self.lo

    @property
    def local(self) -> np.ndarray:
        """global ids of the local columns (owned then ghosts)."""
        return np.concatenate([np.arange(self.lo, self.hi), self.ghosts])


def _clamp_bounds(raw, n, P):
    """Apply the non-empty / capacity clamps to the raw split points (sequential in k)."""
    bounds = [0]
    for k in range(1, P):
        b = int(raw[k - 1]) + 1
        b = max(b, bounds[-1] + 1)            # never an empty part
        b = min(b, n - (P - k))
        bounds.append(b)
    bounds.append(n)
    return np.asarray(bounds, dtype=np.int64)


def split_ranges(weights, P, device=None):
    """Greedy prefix split: boundary k is the first prefix whose weight reaches k W / P (exact integers).
    device: the prefix sum and split search run on that GPU (csrc/partition.cu pdg_split_search)."""
    w = np.asarray(weights, dtype=np.int64)
    n = w.size
    if P < 1:
        raise ValueError("P must be >= 1")
    if P > n:
        raise TooManyRanks(f"{P} ranks for {n} columns")
    if device is not None:
        import ctypes

        import torch

        from . import _lib
        from .device import ptr, stream_ptr
        with torch.cuda.device(device):
            wd = torch.as_tensor(w, device=device)
            raw = np.zeros(max(P - 1, 1), np.int64)
            _lib.check(_lib.lib().pdg_split_search(ptr(wd), n, P, raw.ctypes.data_as(ctypes.c_void_p), stream_ptr()),
                       "split_search")
        return _clamp_bounds(raw, n, P)
    cum = np.cumsum(w)
    W = int(cum[-1])
    raw = [int(np.searchsorted(cum * P, k * W, side="left")) for k in range(1, P)]
    return _clamp_bounds(raw, n, P)


def _rings_host(nbr, nt, lo, hi, depth):
    local = np.zeros(nt, bool)
    local[lo:hi] = True
    front = np.arange(lo, hi)
    rings = []
    for _ in range(depth):
        nb = nbr[front].ravel()
        nb = np.unique(nb[nb >= 0])
        nb = nb[~local[nb]]
        local[nb] = True
        rings.append(nb)
        front = nb
    ghosts = np.concatenate(rings) if rings else np.zeros(0, np.int64)
    ring = np.concatenate([np.full(g.size, k + 1, np.int32) for k, g in enumerate(rings)]) if rings else \
        np.zeros(0, np.int32)
    order = np.argsort(ghosts, kind="stable")
    return ghosts[order], ring[order]


def _rings_device(dm, lo, hi, depth):
    import ctypes

    import torch

    from . import _lib
    from .device import ptr, stream_ptr
    cap = max(dm.nt - (hi - lo), 1)
    with torch.cuda.device(dm.device):
        g = torch.empty(cap, dtype=torch.int32, device=dm.device)
        r = torch.empty(cap, dtype=torch.int32, device=dm.device)
        n = ctypes.c_int()
        _lib.check(_lib.lib().pdg_partition_rings(dm.h, lo, hi, depth, ptr(g), ptr(r), ctypes.byref(n), stream_ptr()),
                   "partition_rings")
        return g[:n.value].cpu().numpy().astype(np.int64), r[:n.value].cpu().numpy().astype(np.int32)


def decompose(mesh, P: int, layers=None, depth: int = 1, device=None):
    """list of Part for ranks 0..P-1.

    depth > 1 adds ghost rings: ring k+1 = the edge neighbours of ring k not already local.  The
    2D sub-cycle then exchanges once per substep (its three RK stages run redundantly on rings
    1-2 and 1) while the 3D fields only ever need ring 1 (send1 / recv1).

    device: run the O(nt) parts -- the weight prefix sum / split search and every rank's ring
    search -- on that GPU (csrc/partition.cu; bit-exact with the host path, which stays for the
    CPU-only multi-process tests)."""
    nt = mesh.nt
    weights = np.ones(nt, np.int64) if layers is None else np.asarray(layers, np.int64)
    b = split_ranges(weights, P, device=device)
    owner = np.repeat(np.arange(P), np.diff(b))
    parts = []
    if device is not None:
        import torch

        from .device import DeviceMesh
        dm = DeviceMesh(mesh, torch.device(device).index)
        rings_of = lambda lo, hi: _rings_device(dm, lo, hi, depth)  # noqa: E731
    else:
        nbr = np.asarray(mesh.nbr)
        rings_of = lambda lo, hi: _rings_host(nbr, nt, lo, hi, depth)  # noqa: E731
    for r in range(P):
        lo, hi = int(b[r]), int(b[r + 1])
        ghosts, ring = rings_of(lo, hi)
        parts.append(Part(r, P, lo, hi, ghosts, ring=ring))
    for r, p in enumerate(parts):
        for s in np.unique(owner[p.ghosts]) if p.ghosts.size else []:
            s = int(s)
            mine = owner[p.ghosts] == s
            sel = p.ghosts[mine]                                      # ascending global ids
            p.recv[s] = (p.n_own + np.flatnonzero(mine)).astype(np.int32)
            parts[s].send[r] = (sel - parts[s].lo).astype(np.int32)
            one = mine & (p.ring == 1)
            if one.any():
                p.recv1[s] = (p.n_own + np.flatnonzero(one)).astype(np.int32)
                parts[s].send1[r] = (p.ghosts[one] - parts[s].lo).astype(np.int32)
    for p in parts:
        for s, idx in p.recv.items():
            if parts[s].send.get(p.rank) is None or parts[s].send[p.rank].size != idx.size:
                raise MapMismatch(f"ranks {s} -> {p.rank}")
    return parts


def local_mesh(mesh, part: Part):
    """Mesh arrays of the local columns (owned + ghosts); neighbours remapped to local ids
    (-1 where a ghost's neighbour is not local -- never read: only owned columns are computed)."""
    gl = part.local
    g2l = np.full(mesh.nt, -1, dtype=np.int64)
    g2l[gl] = np.arange(gl.size)
    lm = SimpleNamespace()
    for k in ("j2d", "dphx", "dphy", "elen", "enx", "eny", "b", "x", "y", "nbrk", "btag"):
        setattr(lm, k, np.ascontiguousarray(np.asarray(getattr(mesh, k))[gl]))
    nbr = np.asarray(mesh.nbr)[gl]
    lm.nbr = np.where(nbr >= 0, g2l[np.maximum(nbr, 0)], -1).astype(np.int64)
    lm.nt = gl.size
    lm.min_edge = float(mesh.min_edge)
    lm.global_ids = gl
    lm.tri = np.asarray(mesh.tri)[gl]
    return lm


# ----------------------------------------------------------------------------- exchange

class _Maps:
    """Device copies of one rank's send / recv index lists (all rings, and ring 1 only)."""

    def __init__(self, part: Part, device, deep=True):
        import torch
        self.part = part
        src_s, src_r = (part.send, part.recv) if deep else (part.send1, part.recv1)
        self.send = {s: torch.as_tensor(v, device=device) for s, v in sorted(src_s.items())}
        self.recv = {s: torch.as_tensor(v, device=device) for s, v in sorted(src_r.items())}


def _pack(fields, nt, idx, buf):
    """fields: tensors whose last dim-run is [..][nt] (planes of nt columns); buf: 1-D [sum nplanes * n].
    CUDA tensors use the pdg_halo_pack kernel; CPU tensors (gloo tests) torch indexing."""
    off = 0
    n = idx.numel()
    for f in fields:
        npl = f.numel() // nt
        if f.is_cuda:
            import ctypes
            from . import _lib
            from .device import stream_ptr
            _lib.check(_lib.lib().pdg_halo_pack(ctypes.c_void_p(f.data_ptr()), npl, nt,
                                                ctypes.c_void_p(idx.data_ptr()), n,
                                                ctypes.c_void_p(buf.data_ptr() + 8 * off), stream_ptr()), "pack")
        else:
            buf[off:off + npl * n] = f.reshape(npl, nt)[:, idx.long()].reshape(-1)
        off += npl * n


def _unpack(fields, nt, idx, buf):
    off = 0
    n = idx.numel()
    for f in fields:
        npl = f.numel() // nt
        if f.is_cuda:
            import ctypes
            from . import _lib
            from .device import stream_ptr
            _lib.check(_lib.lib().pdg_halo_unpack(ctypes.c_void_p(buf.data_ptr() + 8 * off), npl, nt,
                                                  ctypes.c_void_p(idx.data_ptr()), n,
                                                  ctypes.c_void_p(f.data_ptr()), stream_ptr()), "unpack")
        else:
            f.view(npl, nt)[:, idx.long()] = buf[off:off + npl * n].reshape(npl, n)
        off += npl * n


class DistHalo:
    """One rank of a torch.distributed job (NCCL on GPUs, gloo on CPU for the host-side tests).
    `deep` messages fill every ghost ring (2D sub-cycle state and forcing), the others ring 1."""

    def __init__(self, part: Part, nt_local: int, device):
        import torch.distributed as dist
        self.maps = {True: _Maps(part, device, True), False: _Maps(part, device, False)}
        self.nt = nt_local
        self.device = device
        self.exchanges = 0
        # gloo cannot send CUDA tensors: stage the packed messages through host memory (lets the
        # multi-process path run -- and be tested -- with several ranks sharing one GPU)
        self.host_staging = dist.is_initialized() and dist.get_backend() == "gloo" and device.type == "cuda"
        self._plans = {}   # (planes per column, deep) -> (buffers, P2P ops), reused every step

    def exchange(self, fields, deep=False):
        self.start(fields, deep)
        self.finish(fields, deep)

    def _plan(self, tot, deep):
        """Message buffers and the P2P op list for `tot` planes per column, allocated once: an
        exchange is always finished before the next one starts, so reuse is stream-ordered."""
        import torch
        import torch.distributed as dist
        plan = self._plans.get((tot, deep))
        if plan is None:
            mp = self.maps[deep]
            sends = {p: torch.empty(tot * idx.numel(), dtype=torch.float64, device=self.device)
                     for p, idx in mp.send.items()}
            recvs = {p: torch.empty(tot * idx.numel(), dtype=torch.float64,
                                    device="cpu" if self.host_staging else self.device)
                     for p, idx in mp.recv.items()}
            hsend = {p: torch.empty(b.numel(), dtype=torch.float64, pin_memory=True) for p, b in sends.items()} \
                if self.host_staging else sends
            ops = []
            for peer in sorted(set(sends) | set(recvs)):
                if peer in sends:
                    ops.append(dist.P2POp(dist.isend, hsend[peer], peer))
                if peer in recvs:
                    ops.append(dist.P2POp(dist.irecv, recvs[peer], peer))
            plan = self._plans[(tot, deep)] = (sends, hsend, recvs, ops)
        return plan

    def start(self, fields, deep=True):
        """Pack the owned boundary values and post the sends / receives (asynchronous: with NCCL the
        transfer runs on its own stream while the caller launches interior work)."""
        import torch.distributed as dist
        tot = sum(f.numel() // self.nt for f in fields)
        sends, hsend, recvs, ops = self._plan(tot, deep)
        for peer, idx in self.maps[deep].send.items():
            _pack(fields, self.nt, idx, sends[peer])
            if self.host_staging:
                hsend[peer].copy_(sends[peer])
        works = dist.batch_isend_irecv(ops) if ops else []
        self._pending = (recvs, works, deep)

    def finish(self, fields, deep=True):
        """Wait for the posted transfers (a stream dependency with NCCL) and fill the ghost slots."""
        recvs, works, deep = self._pending
        for w in works:
            w.wait()
        for peer, idx in self.maps[deep].recv.items():
            buf = recvs[peer].to(self.device) if self.host_staging else recvs[peer]
            _unpack(fields, self.nt, idx, buf)
        self._pending = None
        self.exchanges += 1


class VirtualGroup:
    """P ranks in one process on one device: halo messages are device-to-device copies (pack into a
    message buffer, unpack on the receiving rank).  Buffers are allocated once per message shape,
    so an exchange is allocation-free and stream ordered: a whole P-rank step can be one graph."""

    capturable = True

    def __init__(self, parts, nts, device):
        self.maps = {d: [_Maps(p, device, d) for p in parts] for d in (True, False)}
        self.nts = nts
        self.device = device
        self.exchanges = 0
        self._bufs = {}

    def _buffers(self, deep, tots):
        import torch
        key = (deep, tuple(tots))
        bufs = self._bufs.get(key)
        if bufs is None:
            bufs = {(r, peer): torch.empty(tots[r] * idx.numel(), dtype=torch.float64, device=self.device)
                    for r, mp in enumerate(self.maps[deep]) for peer, idx in mp.send.items()}
            self._bufs[key] = bufs
        return bufs

    def exchange_all(self, fields_per_rank, deep=False):
        maps = self.maps[deep]
        tots = [sum(f.numel() // self.nts[r] for f in fields) for r, fields in enumerate(fields_per_rank)]
        msgs = self._buffers(deep, tots)
        for r, (mp, fields) in enumerate(zip(maps, fields_per_rank)):
            for peer, idx in mp.send.items():
                _pack(fields, self.nts[r], idx, msgs[(r, peer)])
        for r, (mp, fields) in enumerate(zip(maps, fields_per_rank)):
            for peer, idx in mp.recv.items():
                _unpack(fields, self.nts[r], idx, msgs[(peer, r)])
        self.exchanges += 1


# ----------------------------------------------------------------------------- NCCL through the C ABI

_NCCL = {}


def nccl_library_path():
    """The libnccl the process already uses (torch's), so one process never holds two NCCLs."""
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                if "libnccl.so" in line:
                    return line.split()[-1]
    except OSError:
        pass
    import os
    try:
        import nvidia.nccl
        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    except ImportError:
        pass
    return "libnccl.so.2"


def nccl_comm(rank: int, nranks: int, device: int):
    """This process's pdg_comm (csrc/comm.cu), created once: rank 0 draws the NCCL unique id and
    torch.distributed broadcasts it (nranks == 1 needs no process group)."""
    import ctypes
    from . import _lib
    key = (rank, nranks, device)
    if key in _NCCL:
        return _NCCL[key]
    lb = _lib.lib()
    if lb.pdg_comm_load(nccl_library_path().encode()) != 0:
        raise RuntimeError("pdg_comm_load: " + lb.pdg_comm_error_string().decode())
    uid = (ctypes.c_char * 128)()
    if rank == 0 and lb.pdg_comm_unique_id(uid) != 0:
        raise RuntimeError("pdg_comm_unique_id: " + lb.pdg_comm_error_string().decode())
    if nranks > 1:
        import torch.distributed as dist
        obj = [bytes(uid) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctypes.memmove(uid, obj[0], 128)
    h = ctypes.c_void_p()
    if lb.pdg_comm_init(uid, rank, nranks, device, ctypes.byref(h)) != 0:
        raise RuntimeError("pdg_comm_init: " + lb.pdg_comm_error_string().decode())
    _NCCL[key] = h
    return h


class NcclHalo:
    """One rank's halo exchange through the library (csrc/comm.cu):
    start = pack kernels + grouped ncclSend / ncclRecv on a communication stream, finish = stream
    wait + unpack.  No host synchronisation and no allocation after the plans are built, so the
    partitioned step (2D exchanges once per substep, boundary-first) is captured in one CUDA graph
    per rank like the single-GPU step."""

    capturable = True

    def __init__(self, part: Part, nt_local: int, device, L: int, comm=None, peers_of=None):
        import ctypes
        from . import _lib
        self.part, self.nt, self.device = part, nt_local, device
        self.exchanges = 0
        self.comm = comm if comm is not None else nccl_comm(part.rank, part.nparts, device.index or 0)
        lb = _lib.lib()
        self._keep = []
        self.plans = {}
        # ring-1 messages carry at most u and T (18 L planes per column); deep ones the 2D state (9)
        for deep, maxp in ((True, 9), (False, 18 * L)):
            snd, rcv = (part.send, part.recv) if deep else (part.send1, part.recv1)
            peers = sorted(set(snd) | set(rcv))
            arrs = []
            for d in (snd, rcv):
                lists = [np.ascontiguousarray(d.get(q, np.zeros(0, np.int32)), dtype=np.int32) for q in peers]
                arrs.append(lists)
            self._keep.append(arrs)
            n = len(peers)
            IntArr = ctypes.c_int * max(n, 1)
            PtrArr = ctypes.POINTER(ctypes.c_int) * max(n, 1)
            sp = PtrArr(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in arrs[0]])
            rp = PtrArr(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in arrs[1]])
            h = ctypes.c_void_p()
            _lib.check(lb.pdg_halo_plan_create(self.comm, nt_local, n, IntArr(*peers),
                                               IntArr(*[a.size for a in arrs[0]]), sp,
                                               IntArr(*[a.size for a in arrs[1]]), rp, maxp, ctypes.byref(h)),
                       "pdg_halo_plan_create")
            self.plans[deep] = h
        self._args = {}

    def _fields(self, fields):
        import ctypes
        key = tuple((f.data_ptr(), f.numel()) for f in fields)
        a = self._args.get(key)
        if a is None:
            a = ((ctypes.c_void_p * len(fields))(*[f.data_ptr() for f in fields]),
                 (ctypes.c_longlong * len(fields))(*[f.numel() // self.nt for f in fields]))
            self._args[key] = a
        return a

    def exchange(self, fields, deep=False):
        self.start(fields, deep)
        self.finish(fields, deep)

    def start(self, fields, deep=True):
        from . import _lib
        from .device import stream_ptr
        fp, npl = self._fields(fields)
        rc = _lib.lib().pdg_halo_start(self.plans[deep], len(fields), fp, npl, stream_ptr())
        if rc != 0:
            raise RuntimeError("pdg_halo_start: " + _lib.lib().pdg_comm_error_string().decode())

    def finish(self, fields, deep=True):
        from . import _lib
        from .device import stream_ptr
        fp, npl = self._fields(fields)
        _lib.check(_lib.lib().pdg_halo_finish(self.plans[deep], len(fields), fp, npl, stream_ptr()), "halo_finish")
        self.exchanges += 1


# ----------------------------------------------------------------------------- NVLink peer stores

class P2PPlan:
    """One rank's device-initiated exchange plan for one message shape (csrc/p2p.cu): an inbox of
    per-peer epoch flags and double-buffered windows that the peers write into directly."""

    def __init__(self, send, recv, nt, device, max_planes):
        import ctypes
        from . import _lib
        self.peers = sorted(set(send) | set(recv))
        lists = []
        for d in (send, recv):
            lists.append([np.ascontiguousarray(d.get(q, np.zeros(0, np.int32)), dtype=np.int32) for q in self.peers])
        self._keep = lists
        n = len(self.peers)
        IntArr = ctypes.c_int * max(n, 1)
        PtrArr = ctypes.POINTER(ctypes.c_int) * max(n, 1)
        sp = PtrArr(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in lists[0]])
        rp = PtrArr(*[a.ctypes.data_as(ctypes.POINTER(ctypes.c_int)) for a in lists[1]])
        self.h = ctypes.c_void_p()
        idx = device.index if device.index is not None else 0
        _lib.check(_lib.lib().pdg_p2p_create(nt, n, IntArr(*self.peers), IntArr(*[a.size for a in lists[0]]), sp,
                                             IntArr(*[a.size for a in lists[1]]), rp, max_planes, idx,
                                             ctypes.byref(self.h)), "pdg_p2p_create")

    def local(self, ipc: bool):
        """(64-byte IPC handle or None, raw inbox pointer, {peer: (window offset, flag offset)})."""
        import ctypes
        from . import _lib
        n = max(len(self.peers), 1)
        handle = (ctypes.c_char * 64)() if ipc else None
        raw = ctypes.c_void_p()
        wo, fo = (ctypes.c_longlong * n)(), (ctypes.c_longlong * n)()
        _lib.check(_lib.lib().pdg_p2p_local(self.h, handle, ctypes.byref(raw), wo, fo), "pdg_p2p_local")
        offs = {q: (wo[i], fo[i]) for i, q in enumerate(self.peers)}
        return (bytes(handle) if ipc else None), raw.value, offs

    def connect(self, peer, handle, raw, offs_of_peer, me):
        """Map `peer`'s inbox (IPC handle, or raw pointer in this process); my window / flag in it
        are at the offsets the peer computed for me."""
        import ctypes
        from . import _lib
        wo, fo = offs_of_peer[me]
        hb = (ctypes.c_char * 64).from_buffer_copy(handle) if handle is not None else None
        _lib.check(_lib.lib().pdg_p2p_connect(self.h, self.peers.index(peer), hb, ctypes.c_void_p(raw), wo, fo),
                   "pdg_p2p_connect")

    def run(self, which, fields, nt):
        import ctypes
        from . import _lib
        from .device import stream_ptr
        fp = (ctypes.c_void_p * len(fields))(*[f.data_ptr() for f in fields])
        npl = (ctypes.c_longlong * len(fields))(*[f.numel() // nt for f in fields])
        fn = _lib.lib().pdg_p2p_start if which == "start" else _lib.lib().pdg_p2p_finish
        _lib.check(fn(self.h, len(fields), fp, npl, stream_ptr()), "pdg_p2p_" + which)

    def __del__(self):
        try:
            from . import _lib
            _lib.lib().pdg_p2p_destroy(self.h)
        except Exception:
            pass


def _p2p_plans(part, nt, device, L):
    # ring-1 messages carry at most u and T (18 L planes per column); deep ones the 2D state (9)
    return {True: P2PPlan(part.send, part.recv, nt, device, 9),
            False: P2PPlan(part.send1, part.recv1, nt, device, 18 * L)}


class P2PHalo:
    """One rank's halo exchange by NVLink peer stores (csrc/p2p.cu): the
    peers' inboxes are mapped with CUDA IPC (handles all-gathered over torch.distributed once);
    start = one push kernel per peer (pack + remote stores + epoch release), finish = one pull
    kernel per peer (epoch acquire + unpack).  No NCCL, no host synchronisation: the rank's step
    is captured in one CUDA graph like the single-GPU step."""

    capturable = True

    def __init__(self, part: Part, nt_local: int, device, L: int):
        import torch.distributed as dist
        self.nt, self.exchanges = nt_local, 0
        self.plans = _p2p_plans(part, nt_local, device, L)
        mine = {d: pl.local(ipc=True) for d, pl in self.plans.items()}
        allinfo = [None] * dist.get_world_size()
        dist.all_gather_object(allinfo, {d: (h, o) for d, (h, _, o) in mine.items()})
        for d, pl in self.plans.items():
            for q in pl.peers:
                h, offs = allinfo[q][d]
                pl.connect(q, h, 0, offs, part.rank)
        dist.barrier()

    def exchange(self, fields, deep=False):
        self.start(fields, deep)
        self.finish(fields, deep)

    def start(self, fields, deep=True):
        self.plans[deep].run("start", fields, self.nt)

    def finish(self, fields, deep=True):
        self.plans[deep].run("finish", fields, self.nt)
        self.exchanges += 1


class P2PGroup:
    """P ranks in one process on one device, exchanging through the peer-store protocol with raw
    pointers (the same push / pull kernels, epochs and windows as P2PHalo without IPC)."""

    capturable = True

    def __init__(self, parts, nts, device, L):
        self.nts = nts
        self.exchanges = 0
        self.plans = [_p2p_plans(p, nt, device, L) for p, nt in zip(parts, nts)]
        info = [{d: pl.local(ipc=False) for d, pl in r.items()} for r in self.plans]
        for r, pls in enumerate(self.plans):
            for d, pl in pls.items():
                for q in pl.peers:
                    _, raw, offs = info[q][d]
                    pl.connect(q, None, raw, offs, r)

    def exchange_all(self, fields_per_rank, deep=False):
        for r, fields in enumerate(fields_per_rank):
            self.plans[r][deep].run("start", fields, self.nts[r])
        for r, fields in enumerate(fields_per_rank):
            self.plans[r][deep].run("finish", fields, self.nts[r])
        self.exchanges += 1


class PartitionedRun:
    """P partitions of one mesh, each an ImexStepper over its owned + ghost columns.

    transport "virtual": all ranks in this process on one device (VirtualGroup);
    transport "p2p-virtual": the same, exchanging through the peer-store kernels (P2PGroup);
    transport "nccl": this process is rank `rank`; the library's NCCL plans (NcclHalo);
    transport "p2p": this process is rank `rank`; NVLink peer stores (P2PHalo, CUDA IPC);
    transport "dist": this process is rank `rank` of a torch.distributed job (DistHalo).
    """

    def __init__(self, mesh, L, params, dt, m, kv, nu_v, P, transport="virtual", rank=None, device=None):
        import torch
        from .stepper import ImexStepper
        self.mesh, self.L, self.P = mesh, L, P
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.parts = decompose(mesh, P, np.full(mesh.nt, L), depth=GHOST_DEPTH, device=dev)
        self.local = [local_mesh(mesh, p) for p in self.parts]
        ranks = range(P) if transport in ("virtual", "p2p-virtual") else [rank]
        self.ranks = list(ranks)
        self.st = {r: ImexStepper(self.local[r], L, params, dt, m, kv, nu_v, part=self.parts[r], device=dev.index)
                   for r in ranks}
        if transport == "virtual":
            self.group = VirtualGroup(self.parts, [lm.nt for lm in self.local], dev)
        elif transport == "p2p-virtual":   # all ranks here, peer-store protocol with raw pointers
            self.group = P2PGroup(self.parts, [lm.nt for lm in self.local], dev, L)
        elif transport == "p2p":     # NVLink peer stores between processes (CUDA IPC inboxes)
            self.group = None
            self.st[rank].halo = P2PHalo(self.parts[rank], self.local[rank].nt, dev, L)
        elif transport == "nccl":    # the library's NCCL halo plans (csrc/comm.cu): graph-captured steps
            self.group = None
            self.st[rank].halo = NcclHalo(self.parts[rank], self.local[rank].nt, dev, L)
        else:                        # torch.distributed send / recv (gloo tests, un-graphed)
            self.group = None
            self.st[rank].halo = DistHalo(self.parts[rank], self.local[rank].nt, dev)
        self.use_graph = True
        self.graphs = {}
        self.dev = dev
        self._skip_exchanges = set()   # tests only: exchange names to leave out (a broken schedule)

    @property
    def schedule_check(self) -> bool:
        """Debug mode: ghost slots are poisoned (NaN) while their exchange is pending
        and every eager step ends with ScheduleViolation if a poisoned value reached an owned one."""
        return any(st.schedule_check for st in self.st.values())

    @schedule_check.setter
    def schedule_check(self, on: bool):
        for st in self.st.values():
            st.schedule_check = bool(on)

    def set_state(self, eta, qx, qy, ux, uy, T, t=0.0):
        L = self.L
        for r, st in self.st.items():
            gl = self.local[r].global_ids
            pr = (gl[:, None] * L + np.arange(L)[None, :]).ravel()
            st.set_state(eta[gl], qx[gl], qy[gl], ux[pr], uy[pr], T[pr], t)

    def get_state(self):
        """Global numpy state gathered from the owned columns (virtual transport: all ranks here)."""
        L, nt = self.L, self.mesh.nt
        out = dict(eta=np.zeros((nt, 3)), qx=np.zeros((nt, 3)), qy=np.zeros((nt, 3)), ux=np.zeros((nt * L, 6)),
                   uy=np.zeros((nt * L, 6)), T=np.zeros((nt * L, 6)))
        for r, st in self.st.items():
            p = self.parts[r]
            s = st.get_state()
            own = slice(0, p.n_own)
            out["eta"][p.lo:p.hi] = s["eta"][own]
            out["qx"][p.lo:p.hi] = s["qx"][own]
            out["qy"][p.lo:p.hi] = s["qy"][own]
            for k in ("ux", "uy", "T"):
                out[k][p.lo * L:p.hi * L] = s[k][:p.n_own * L]
            out["t"] = s["t"]
        return out

    def _lockstep(self):
        """One step of every virtual rank: the ranks' step generators advance together and every
        exchange point is one VirtualGroup exchange (the 'start' of a boundary-first exchange is
        a no-op on one device: the copies happen at its 'finish', after the interior work)."""
        gens = {r: st._step_gen(st.t) for r, st in self.st.items()}
        while True:
            fields, phases, done = [], set(), 0
            for r in self.ranks:          # every rank runs the same phase, then one exchange
                try:
                    ph, f, name = next(gens[r])
                    phases.add((ph, name))
                    fields.append(f)
                except StopIteration:
                    done += 1
            if done:
                if done != len(self.ranks):
                    raise MapMismatch("ranks reached different exchange points")
                break
            if len(phases) != 1:
                raise MapMismatch(f"ranks at different exchange phases {phases}")
            ph, name = phases.pop()
            if name in self._skip_exchanges:      # tests: a deliberately broken schedule
                continue
            if ph not in ("start", "start1"):     # one device: a boundary-first exchange moves at its join
                self.group.exchange_all(fields, deep=ph in ("finish", "deep"))

    def _capture(self, key):
        """One CUDA graph of the whole P-rank lockstep step (the stepper's capture recipe)."""
        import gc

        import torch
        side = torch.cuda.Stream(device=self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        saved = {r: st.S.clone() for r, st in self.st.items()}
        n_before = self.group.exchanges
        with torch.cuda.stream(side):
            self._lockstep()                       # sizes workspaces and message buffers
            for r, st in self.st.items():
                st.S.copy_(saved[r])
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        gc.collect()
        gcflag = gc.isenabled()
        gc.disable()
        try:
            n0 = self.group.exchanges
            with torch.cuda.graph(g):
                self._lockstep()
            self._graph_exchanges = self.group.exchanges - n0
            self.group.exchanges = n_before      # warm-up and recording moved nothing: replays count
        finally:
            if gcflag:
                gc.enable()
        self.graphs[key] = g
        return g

    def step(self, n=1):
        if self.group is None:            # one rank of a multi-process job: its stepper drives the halo
            for st in self.st.values():
                st.step(n)
            return
        for _ in range(n):
            varies = any(st.p.tau_x1 is not None for st in self.st.values())
            if self.use_graph and not varies and not self.schedule_check:
                key = next(iter(self.st.values())).cur
                g = self.graphs.get(key)
                if g is None:
                    g = self._capture(key)
                g.replay()
                self.group.exchanges += self._graph_exchanges
            else:
                self._lockstep()
            for st in self.st.values():
                st._advance()
            if self.schedule_check:
                for st in self.st.values():
                    st.check_schedule()

    def check(self):
        for st in self.st.values():
            st.check()


# ----------------------------------------------------------------------------- scaling plumbing

PAPER_EXCHANGES_PER_STEP = 100    # PAPER.md section 4.2: "approximately 100 halo exchanges" at m = 20


def exchanges_per_step(m: int) -> int:
    """Halo exchanges of one partitioned internal step, derived from the step plan (stepper._stage):
    per stage q, F3D->2D (all rings), mis and (u, T); per external substep one exchange of the 2D
    state over all ghost rings (three rings: the RK stages run on owned + rings 1-2 / 1 / 0).
    m = 20 -> 2 x 4 + 10 + 20 = 38 (the paper's one-ring scheme: ~100)."""
    return 2 * 4 + m // 2 + m


def amdahl_report(times: dict, path: str | None = None) -> dict:
    """Least-squares fit T(P) = a + b / P over a rank-count sweep: a is the serial /
    latency share, b the parallel work.  times: {P: seconds per step} (>= 2 rank counts).  Writes
    P,T,T_fit,a,b,r2 rows to `path` when given; returns {"a", "b", "r2", "rows"}."""
    P = np.asarray(sorted(times), dtype=float)
    if P.size < 2:
        raise ValueError("amdahl_report needs >= 2 rank counts")
    T = np.asarray([times[int(p)] if int(p) in times else times[p] for p in sorted(times)], dtype=float)
    X = np.stack([np.ones_like(P), 1.0 / P], axis=1)
    (a, b), *_ = np.linalg.lstsq(X, T, rcond=None)
    fit = a + b / P
    ss_res = float(((T - fit) ** 2).sum())
    ss_tot = float(((T - T.mean()) ** 2).sum())
    r2 = 1.0 - ss_res / ss_tot if ss_tot > 0 else (1.0 if ss_res <= 1e-30 else 0.0)
    rows = [(int(p), float(t), float(f)) for p, t, f in zip(P, T, fit)]
    if path is not None:
        with open(path, "w") as fh:
            fh.write("P,T,T_fit,a,b,r2\n")
            for p, t, f in rows:
                fh.write(f"{p},{t!r},{f!r},{float(a)!r},{float(b)!r},{r2!r}\n")
    return {"a": float(a), "b": float(b), "r2": r2, "rows": rows}
