"""ctypes binding of libprismdg_b200.so (include/prismdg_b200.h).

There is no fallback: if the library is missing or a CUDA device is absent,
every compute entry raises.  The library is built in-tree by
`python -m paper_2605_16082_b200.build` (or __graft_entry__.build()).
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PDG_LIB selects an alternative in-tree build (A/B experiments); default: the in-tree library
LIB_PATH = os.environ.get("PDG_LIB") or os.path.join(_HERE, "libprismdg_b200.so")

P = ctypes.c_void_p
I = ctypes.c_int
D = ctypes.c_double
LL = ctypes.c_longlong


class MeshDesc(ctypes.Structure):
    _fields_ = [("nt", I), ("j2d", P), ("dphx", P), ("dphy", P), ("elen", P), ("enx", P), ("eny", P), ("b", P),
                ("nbr", P), ("nbrk", P), ("btag", P), ("min_edge", D)]


# name -> (restype, argtypes)
_SIGS = {
    "pdg_ctx_create": (I, [ctypes.POINTER(MeshDesc), I, ctypes.POINTER(P)]),
    "pdg_ctx_destroy": (I, [P]),
    "pdg_ctx_set_layers": (I, [P, I, P]),
    "pdg_last_error": (I, [P, P, ctypes.POINTER(I), ctypes.POINTER(LL), ctypes.POINTER(LL), ctypes.POINTER(D)]),
    "pdg_cuda_error_string": (ctypes.c_char_p, []),
    "pdg_launch_count": (LL, [P]),
    "pdg_tune": (I, [I, I]),
    "pdg_ctx_set_owned": (I, [P, I]),
    "pdg_mesh_build": (I, [I, LL] + [P] * 16 + [P]),
    "pdg_hilbert_perm": (I, [I, I, P, P, P, P]),
    "pdg_ext2d_subcycle_begin": (I, [P, P, D, D, I, P, P]),
    "pdg_ext2d_rk_stage": (I, [P, I, P, P, P, D, D, D, P, P, P, I, D, P, P]),
    "pdg_ext2d_subcycle_end": (I, [P, P, P, I, D, P, P, P]),
    "pdg_ext2d_rk_stage_cols": (I, [P, I, P, P, P, D, D, D, P, P, P, I, P]),
    "pdg_split_search": (I, [P, I, I, P, P]),
    "pdg_partition_rings": (I, [P, I, I, I, P, P, ctypes.POINTER(I), P]),
    "pdg_halo_pack": (I, [P, LL, I, P, I, P, P]),
    "pdg_halo_unpack": (I, [P, LL, I, P, I, P, P]),
    "pdg_comm_load": (I, [ctypes.c_char_p]),
    "pdg_comm_error_string": (ctypes.c_char_p, []),
    "pdg_comm_unique_id": (I, [P]),
    "pdg_comm_init": (I, [P, I, I, I, ctypes.POINTER(P)]),
    "pdg_comm_destroy": (I, [P]),
    "pdg_halo_plan_create": (I, [P, I, I, P, P, P, P, P, I, ctypes.POINTER(P)]),
    "pdg_halo_plan_destroy": (I, [P]),
    "pdg_halo_start": (I, [P, I, P, P, P]),
    "pdg_halo_finish": (I, [P, I, P, P, P]),
    "pdg_halo_2d": (I, [P, P, P]),
    "pdg_copy_d2d": (I, [P, P, LL, P]),
    "pdg_halo_3d": (I, [P, I, P, P, P]),
    "pdg_p2p_create": (I, [I, I, P, P, P, P, P, I, I, P]),
    "pdg_p2p_destroy": (I, [P]),
    "pdg_p2p_local": (I, [P, P, P, P, P]),
    "pdg_p2p_connect": (I, [P, I, P, P, LL, LL]),
    "pdg_p2p_start": (I, [P, I, P, P, P]),
    "pdg_p2p_finish": (I, [P, I, P, P, P]),
    "pdg_rows_to_planes": (I, [P, I, I, I, P, I, I, P]),
    "pdg_planes_to_rows": (I, [P, I, I, I, I, I, P, P]),
    "pdg_ext2d_eval": (I, [P, P, P, P, P, P, P, I, D, D, D, P, I, I, P, P, P, P]),
    "pdg_ext2d_subcycle": (I, [P, P, I, D, D, D, P, P, P, P, P, P, I, P]),
    "pdg_ext2d_cfl": (I, [P, P, D, D, P, P]),
    "pdg_apply_mh": (I, [P, P, I, I, I, P, P, P]),
    "pdg_eos": (I, [P, P, LL, D, D, D, D, P, P]),
    # internal3d (csrc/int3d.cu)
    "pdg_prism_mass": (I, [P, P, P, I, P, P]),
    "pdg_project_transport": (I, [P, P, P, P, P, P, I, P, P, P, P]),
    "pdg_column_sum": (I, [I, I, I, P, P, P]),
    "pdg_total_thickness": (I, [P, P, P, P]),
    "pdg_mismatch": (I, [P, P, P, P, P, P]),
    "pdg_consistent_transport": (I, [P, P, P, P, P, I, P, P]),
    "pdg_lateral_flux_factor": (I, [P, P, P, D, P, I, P, P]),
    "pdg_compute_r": (I, [P, P, P, I, D, D, D, P, I, P, P]),
    "pdg_compute_w": (I, [P, P, P, P, P, P, P, I, P, P]),
    "pdg_compute_wtilde": (I, [P, P, P, P, P, D, P, I, P, P]),
    "pdg_horizontal_rhs": (I, [P, P, P, I, P, P, P, P, D, D, I, P, I, P, P]),
    "pdg_horizontal_diffusion": (I, [P, P, P, I, D, I, D, I, P, I, P, P]),
    "pdg_mass_terms": (I, [I, I, P, P, P, D, D, P, P]),
    "pdg_stress_rhs": (I, [P, P, P, D, D, D, P, I, P, P]),
    "pdg_step_f3d2d": (I, [P, P, P, P, P, D, D, D, D, D, D, P, P]),
    "pdg_step_f3d2d_rsum": (I, [P, P, P, P, P, P, D, D, D, D, D, D, P, P]),
    "pdg_step_r": (I, [P, P, P, D, D, D, P, P, P, P]),
    "pdg_step_rhs": (I, [P, I, P, P, P, P, P, P, P, P, P, D, D, D, D, D, D, D, P, P]),
    "pdg_step_rhs_ut": (I, [P, P, P, P, P, P, P, P, P, P, P, P, D, D, D, D, D, D, D, P, P, P]),
    "pdg_step_rhs_ut_w": (I, [P, P, P, P, P, P, P, P, P, P, P, P, D, D, D, D, D, D, D, P, P, P, P]),
    # columns (csrc/columns.cu)
    "pdg_solve_sweep": (I, [I, I, I, I, P, P, P, P, P, P]),
    "pdg_solve_banded": (I, [I, I, I, P, P, P, P, P, P, P, P, P]),
    "pdg_apply_banded": (I, [I, I, I, P, P, P, P, P, P]),
    "pdg_build_implicit": (I, [LL, P, P, P, P, D, P, P, P, P]),
    "pdg_mass_op": (I, [I, I, I, I, P, P, P, P, P]),
    "pdg_solve_tridiagonal": (I, [I, I, P, P, P, P, P, P, P, P]),
    "pdg_assemble_vertical": (I, [P, P, P, P, D, D, D, I, P, I, P, P, P, P]),
    "pdg_step_vertical": (I, [P, I, I, P, P, P, D, P, D, D, D, I, D, P, P, P, P]),
    "pdg_step_vertical_cols": (I, [P, I, I, P, P, P, D, P, D, D, D, I, D, P, P, P, P, I, P]),
    "pdg_step_diagnostics": (I, [P, P, P, P, D, P, P, P]),
    "pdg_diagnostics_work_doubles": (I, [P]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raises if the extension is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension not built: {LIB_PATH} missing "
                               "(run `python -m paper_2605_16082_b200.build`); there is no CPU fallback")
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        # PDG_TUNE="key=value,..." overrides the measured kernel-variant defaults (A/B runs)
        for kv in filter(None, os.environ.get("PDG_TUNE", "").split(",")):
            k, v = kv.split("=")
            l.pdg_tune(int(k), int(v))
        _lib = l
    return _lib


def declare(name, res, args):
    _SIGS[name] = (res, args)
    if _lib is not None:
        fn = getattr(_lib, name)
        fn.restype = res
        fn.argtypes = args


def exported_symbols():
    return list(_SIGS)


def check(rc, what=""):
    """Return status of a C entry: argument errors (PDG_ERR_SHAPE, ...) raise their errors.py
    class eagerly, PDG_ERR_CUDA raises RuntimeError with the CUDA error string."""
    if rc != 0:
        from . import errors
        if rc != errors.ERR_CUDA:
            errors.raise_for_code(rc, what=what)
        msg = lib().pdg_cuda_error_string().decode(errors="replace")
        raise RuntimeError(f"{what}: CUDA error ({rc}) {msg}")
