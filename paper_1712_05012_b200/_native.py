"""ctypes binding of libkfb200.so (the C ABI in include/kfb200.h).

The library is the only compute path of this package: if it is missing, or no
CUDA device is present, every hot-path call raises ``NativeLibraryError``.
There is deliberately no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeLibraryError

LIB_PATH = os.environ.get("KFB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                         "libkfb200.so")   # KFB200_LIB: A/B builds
ABI_VERSION = 14

P = C.c_void_p
I32 = C.c_int32
F64 = C.c_double


class KfChain(C.Structure):
    _fields_ = [("n_atoms", I32), ("n_links", I32), ("n_dof", I32), ("n_res", I32),
                ("n_bb", I32), ("n_side", I32), ("side_depth", I32), ("_pad0", I32)] + [
        (name, P) for name in (
            "link_parent", "link_dof", "link_axis0", "link_body0", "bb_order", "side_order",
            "side_depth_off", "atom_link", "atom_zrel", "link_atom_off", "link_atoms",
            "chi_res_off", "chi_links", "bb_by_dof", "bb_side_res")]


class KfField(C.Structure):
    _fields_ = [
        ("n_atoms", I32), ("uniform_weights", I32), ("dielectric_const", I32), ("solvation", I32),
        ("q32", P), ("R32", P), ("seps32", P), ("q", P), ("R", P), ("eps", P),
        ("tparent", P), ("tgp", P), ("tggp", P), ("tres", P), ("tchain", P), ("class_map", P),
        ("class_slow", P),
        ("w_elec", F64 * 4), ("w_vdw", F64 * 4), ("uniform_value", F64), ("kappa", F64),
        ("cut_pair2", F64), ("thr_elec2", F64), ("thr_vdw2", F64),
        ("cell", F64), ("hash_bits", I32), ("n_stencil", I32), ("stencil", P),
        ("n_samples", I32), ("_pad1", I32), ("samples", P), ("r_off", P), ("r_off2", P),
        ("gamma", P), ("w_int", P), ("quantum", F64), ("delta_r", F64), ("four_pi", F64),
        ("reach_pad", F64), ("solv_atoms", P), ("n_solv", I32), ("precision", I32),
        ("samples_grp", P), ("grp_cone", P), ("n_groups", I32), ("flat", I32),
        ("atom_par", P), ("atom_aux", P), ("r_off_max", F64), ("class_codes", P), ("unit_codes", P)]


class KfStatus(C.Structure):
    _fields_ = [("iter", I32), ("done", I32), ("reason", I32), ("error", I32),
                ("err_iter", I32), ("clash_i", I32), ("clash_j", I32), ("overflow", I32),
                ("dmin_bits", C.c_uint64), ("clash_key", C.c_uint64), ("tau0", F64),
                ("n_pairs", C.c_int64), ("n_pairs_vdw", C.c_int64)]


class KfBatch(C.Structure):
    _fields_ = [("B", I32), ("n_buckets", I32), ("nb_cap", I32), ("record_theta", I32),
                ("max_records", I32), ("pair_chunk", I32), ("api_eval", I32), ("_pad_b", I32)] + [
        (name, P) for name in (
            "theta", "frozen", "link_T", "fk_scratch", "pos", "forces", "cell_key", "cell_cnt", "cell_start",
            "occ", "occ_count", "occ_offset", "chunk_pre", "item_cell", "chunk_count", "chunk_offset",
            "atom_slot", "atom_rank", "sorted_atom", "s_hi", "s_lo",
            "s_pos", "s_par", "s_aux", "s_tree", "cell_box", "work", "e_atom", "pair_count",
            "solv_acc", "solv_ovf", "pair_fj", "cav_atom", "f_exp", "a_exp", "wrench", "side_tot", "bb_suffix", "tau", "energy", "status",
            "rec_energy", "rec_theta")]


class KfStep(C.Structure):
    _fields_ = [("kappa", F64), ("torque_tol", F64), ("torque_tol_rel", F64),
                ("energy_tol", F64), ("max_iters", I32), ("energy_window", I32)]


REASONS = {1: "max_iters", 2: "torque-free", 3: "torque tolerance",
           4: "torque tolerance (relative)", 5: "energy plateau"}
ERR_CLASH, ERR_NONFINITE, ERR_CAPACITY, ERR_EXTENT = 1, 2, 3, 4

# every exported symbol of include/kfb200.h with its argument types
_PROTOS = {
    "kf_abi_version": (I32, []),
    "kf_struct_size": (C.c_size_t, [C.c_int]),
    "kf_last_error": (C.c_char_p, []),
    "kf_device_sm_count": (I32, []),
    "kf_fk": (I32, [P, P, P]),
    "kf_nonbonded": (I32, [P, P, P]),
    "kf_solvation": (I32, [P, P, P]),
    "kf_energy_reduce": (I32, [P, P, C.c_int, P]),
    "kf_torques_step": (I32, [P, P, P, P, P]),
    "kf_fold_iterations": (I32, [P, P, P, P, C.c_int, P]),
    "kf_fold_iterations_eager": (I32, [P, P, P, P, C.c_int, P]),
    "kf_fold_graph_prepare": (I32, [P, P, P, P, C.c_int, P]),
    "kf_graph_cache_clear": (None, []),
    "kf_clash_report": (I32, [P, P, P]),
    "kf_bbox": (I32, [P, C.c_int, P, P]),
    "kf_grid_cells": (I32, [P, C.c_int, P, F64, P, P, P, P]),
    "kf_counting_sort": (I32, [P, C.c_int, C.c_int64, P, P, P, P, P]),
    "kf_neighbor_rows_count": (I32, [P, P, C.c_int, P, P, C.c_int, P, P]),
    "kf_neighbor_rows_fill": (I32, [P, P, C.c_int, P, P, P, C.c_int, P, P, P]),
    "kf_sort_rows": (I32, [P, C.c_int, P, P]),
    "kf_filter_table": (I32, [P, P, P, C.c_int, C.c_int64, F64, C.c_int, P, P, P]),
    "kf_compact_pairs": (I32, [P, P, C.c_int, C.c_int64, P, P, P, P, P, P, P, P]),
    "kf_sum_f64": (I32, [P, C.c_int64, P, P, P]),
    "kf_scan_exclusive_i64": (I32, [P, C.c_int64, P, P, P]),
    "kf_classify_pairs": (I32, [P, P, P, C.c_int64, P, P]),
    "kf_pair_terms": (I32, [P, P, C.c_int, P, P, P, P, C.c_int64, C.c_int, P, P, P, P]),
    "kf_pair_kernel_kind": (I32, [P, P, C.c_int]),
    "kf_scatter_pair_forces": (I32, [P, C.c_int, P, P, P, P, C.c_int64, P, P]),
    "kf_grid_occupied": (I32, [P, P, C.c_int64, P, P, P, P, P]),
    "kf_row_kept_offsets": (I32, [P, C.c_int, P, P, P]),
    "kf_argmin_f64": (I32, [P, C.c_int64, P, P]),
    "kf_sasa_pass": (I32, [P, C.c_int, P, P, P, C.c_int, P, P, F64, C.c_int, P, P, P, P, F64,
                           P, P, P, P, P]),
    "kf_fixed_to_f64": (I32, [P, C.c_int64, F64, P, P]),
    "kf_bin": (I32, [P, P, P]),
    "kf_launch_counter": (C.c_ulonglong, []),
    "kf_peak_flops": (I32, [C.c_int, P, P]),
    "kf_pairs": (I32, [P, P, P]),
    "kf_solvation_forces": (I32, [P, C.c_int, P, P, P, P, C.c_int, P, P, P, P, F64, F64,
                                  C.c_int, P, P, P]),
    "kf_link_wrenches": (I32, [P, P, P, P, P]),
    "kf_joint_torques": (I32, [P, P, P, P, P, P, P]),
    "kf_kcm_step": (I32, [P, P, P, C.c_int, F64, P, P, P]),
}

_lib = None


def lib():
    """Load and validate libkfb200.so once (ABI version and struct layouts)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeLibraryError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (make -C paper_1712_05012_b200/csrc)")
    handle = C.CDLL(LIB_PATH)
    for name, (res, args) in _PROTOS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.kf_abi_version() != ABI_VERSION:
        raise NativeLibraryError("libkfb200 ABI version mismatch")
    for k, cls in enumerate((KfChain, KfField, KfStatus, KfBatch, KfStep)):
        if handle.kf_struct_size(k) != C.sizeof(cls):
            raise NativeLibraryError(f"struct layout mismatch for {cls.__name__}: "
                                     f"C {handle.kf_struct_size(k)} vs ctypes {C.sizeof(cls)}")
    _lib = handle
    return handle


def exported_symbols() -> list:
    return list(_PROTOS)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.kf_last_error().decode() if _lib is not None else "?"
        raise NativeLibraryError(f"{what} failed: {msg}")


def ref(struct) -> C.c_void_p:
    return C.cast(C.pointer(struct), C.c_void_p)
