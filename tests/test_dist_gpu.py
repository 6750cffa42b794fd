"""bench.py's multi-process path (torchrun, one rank per partition) on one GPU with gloo host-staged halos:
the final state equals the single-process run bitwise."""
import glob
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp, nproc, halo=None):
    out = os.path.join(tmp, f"s{nproc}{halo or ''}")
    base = [sys.executable, "bench.py", "--config", "c3", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-e2e",
            "--dump", out, "--phase-csv", out + ".phases.csv"]
    if nproc == 1:
        cmd = base
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
               "--master-addr", "127.0.0.1", "--master-port", "29517"] + base[1:] + ["--gpus", str(nproc),
                                                                                      "--backend", "gloo"]
        if halo:
            cmd += ["--halo", halo]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    parts = [np.load(f) for f in sorted(glob.glob(out + ".*.npz"))]
    gid = np.concatenate([p["gid"] for p in parts])
    order = np.argsort(gid)
    return {k: np.concatenate([p[k] for p in parts])[order] if k == "eta" else None for k in ("eta",)}, parts


def test_two_process_partition_matches_single(tmp_path):
    one, p1 = _run(str(tmp_path), 1)
    two, p2 = _run(str(tmp_path), 2)
    assert np.array_equal(one["eta"], two["eta"])
    L = 20
    for k in ("T", "ux"):
        a = p1[0][k]
        b = np.concatenate([p[k] for p in p2])   # rank ranges are contiguous and ascending
        assert np.array_equal(a, b), k
    # SPEC.md:616 phase timings of every rank: step,rank,phase,micros with the boundary-first phases
    for r in range(2):
        rows = open(os.path.join(str(tmp_path), f"s2.phases.csv.{r}")).read().splitlines()
        assert rows[0] == "step,rank,phase,micros"
        names = {x.split(",")[2] for x in rows[1:]}
        assert {"boundary:state2d", "pack+post:state2d", "interior:state2d", "join+unpack:state2d",
                "exchange:q", "exchange:uT", "exchange:mis"} <= names, names
        assert all(float(x.split(",")[3]) >= 0.0 and x.split(",")[1] == str(r) for x in rows[1:])


def test_two_process_peer_store_halos(tmp_path):
    """The device-initiated transport between processes (csrc/p2p.cu, partition.P2PHalo): each
    rank maps the other's inbox through CUDA IPC (handles all-gathered over gloo) and its step is
    graph-captured; two processes share the one GPU here.  Bitwise equal to the single process."""
    one, p1 = _run(str(tmp_path), 1)
    two, p2 = _run(str(tmp_path), 2, halo="p2p")
    assert np.array_equal(one["eta"], two["eta"])
    for k in ("T", "ux"):
        a = p1[0][k]
        b = np.concatenate([p[k] for p in p2])
        assert np.array_equal(a, b), k
