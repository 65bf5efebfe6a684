"""ctypes binding of libemc.so (include/emc.h).

The library is built in-tree (``python -m paper_2403_12345_b200._build`` or
``__graft_entry__.build()``) and loaded from this directory.  A missing
library or an unusable GPU raises NativeUnavailableError -- there is no CPU
fallback for any transport operation.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import NativeUnavailableError

HERE = os.path.dirname(os.path.abspath(__file__))
ABI_VERSION = 2                     # include/emc.h EMC_ABI_VERSION
LIB_PATH = os.environ.get("EMC_LIBRARY") or os.path.join(HERE, "libemc.so")

N_COUNTERS = 24
N_TIMINGS = 4

_P = C.c_void_p
_I64 = C.c_int64
_I32 = C.c_int32
_D = C.c_double


class EmcLibrary(C.Structure):
    _fields_ = [("n_nuclides", _I64), ("n_points", _I64), ("n_materials", _I64),
                ("n_entries", _I64), ("grid_off", _P), ("grids", _P), ("ch_t", _P),
                ("ch_s", _P), ("ch_c", _P), ("ch_f", _P), ("nu", _P), ("mat_off", _P),
                ("mat_nuc", _P), ("mat_den", _P), ("emin", _D), ("emax", _D)]


class EmcGeometry(C.Structure):
    _fields_ = [("radius", _D), ("r2", _D), ("half_pitch", _D), ("height", _D),
                ("n_axial", _I64), ("zplanes", _P), ("fuel_mats", _P), ("mod_mat", _I64)]


class EmcRunConfig(C.Structure):
    _fields_ = [("particles_per_batch", _I64), ("gid_lo", _I64), ("n_assigned", _I64),
                ("max_in_flight", _I64), ("history", _I32), ("fused", _I32),
                ("use_logs", _I32), ("sort_enabled", _I32), ("sort_every", _I32),
                ("box_guard", _I32), ("seed", C.c_uint64), ("alpha", _D), ("fission_t", _D),
                ("perturb_gid", _I64)]


class EmcBatchArgs(C.Structure):
    _fields_ = [("batch", _I64), ("k_run", _D), ("batch0", _I32), ("score", _I32)]


class EmcBatchResult(C.Structure):
    _fields_ = [("counters", _I64 * N_COUNTERS), ("timings", _D * N_TIMINGS),
                ("n_sites", _I64), ("n_logs", _I64), ("iterations", _I64),
                ("launches", _I64), ("error", _I32), ("reruns", _I32),
                ("error_gid", _I64)]


# every symbol include/emc.h declares: (name, restype, argtypes)
SYMBOLS = {
    "emc_last_error": (C.c_char_p, []),
    "emc_abi_version": (C.c_int, []),
    "emc_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "emc_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "emc_destroy": (None, [_P]),
    "emc_set_stream": (C.c_int, [_P, _P]),
    "emc_upload_library": (C.c_int, [_P, C.POINTER(EmcLibrary)]),
    "emc_upload_geometry": (C.c_int, [_P, C.POINTER(EmcGeometry)]),
    "emc_configure": (C.c_int, [_P, C.POINTER(EmcRunConfig)]),
    "emc_set_geometry_options": (C.c_int, [_P, _I32, _I32]),
    "emc_set_fixed_source": (C.c_int, [_P, _I32, _D]),
    "emc_set_lattice": (C.c_int, [_P, _I32, _D, _P]),
    "emc_set_mesh": (C.c_int, [_P, _I32, _I32, _I32]),
    "emc_mesh_device": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_I64)]),
    "emc_set_source_local": (C.c_int, [_P, _D]),
    "emc_set_source_device": (C.c_int, [_P, C.POINTER(_P), _I64, _D]),
    "emc_set_source_window": (C.c_int, [_P, C.POINTER(_P), _I64, _D, _I64]),
    "emc_run_batch": (C.c_int, [_P, C.POINTER(EmcBatchArgs), C.POINTER(EmcBatchResult)]),
    "emc_reduce_bins": (C.c_int, [_P, _P, _P, _I64]),
    "emc_bank_size": (C.c_int, [_P, C.POINTER(_I64)]),
    "emc_bank_device": (C.c_int, [_P, C.POINTER(_P)]),
    "emc_bank_copy": (C.c_int, [_P, _I64, _I64] + [_P] * 9),
    "emc_xs_lookup": (C.c_int, [_P, _I64, _P, _P, _P, _P, _I32]),
    "emc_grid_index": (C.c_int, [_P, _I64, _P, _P, _P]),
    "emc_upload_union": (C.c_int, [_P, _P, _I64, _P, _P]),
    "emc_set_accel": (C.c_int, [_P, _I32]),
    "emc_group_create": (C.c_int, [_P, _I32, _P]),
    "emc_group_destroy": (None, [_P]),
    "emc_group_reduce_bins": (C.c_int, [_P, _P, _I64]),
    "emc_group_exchange_bank": (C.c_int, [_P, _I64, _D, _P]),
    "emc_locate": (C.c_int, [_P, _I64, _P, _P]),
    "emc_distance": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P]),
    "emc_particle_ops": (C.c_int, [_P, _I64, _P, _P, _P, _P, _P, _P]),
    "emc_sort_queue": (C.c_int, [_P, _I64, _P, _I64, _P, _P, _P]),
    "emc_replay_bins": (C.c_int, [_P, _I64, _P, _P, _I32, _P]),
    "emc_lcg_skip": (C.c_int, [_P, _I64, _P, _P, _P]),
    "emc_libm_eval": (C.c_int, [_P, _I64, _P, _P]),
    "emc_div_eval": (C.c_int, [_P, _I64, _P, _P, _P]),
    "emc_launch_count": (_I64, [_P]),
    "emc_bench_lookup": (C.c_int, [_P, _I64, _P, _P, _I32, _I32, C.POINTER(_D), C.POINTER(_D)]),
}

_LIB = None


def load_library_file() -> C.CDLL:
    """dlopen libemc.so and bind every exported symbol (no GPU needed)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailableError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2403_12345_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SYMBOLS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.emc_abi_version() != ABI_VERSION:
        raise NativeUnavailableError(f"{LIB_PATH} has ABI {lib.emc_abi_version()}, these bindings need "
                                     f"{ABI_VERSION}: rebuild it (python -m paper_2403_12345_b200._build)")
    _LIB = lib
    return lib


def check(rc: int, what: str = "") -> None:
    if rc != 0:
        msg = load_library_file().emc_last_error().decode(errors="replace")
        raise NativeUnavailableError(f"libemc {what} failed (rc={rc}): {msg}") \
            if rc == -1 else RuntimeError(f"libemc {what} failed (rc={rc}): {msg}")


def device_count() -> int:
    lib = load_library_file()
    n = C.c_int(0)
    rc = lib.emc_device_count(C.byref(n))
    if rc != 0:
        return 0
    return n.value


def ptr(a) -> C.c_void_p:
    """data pointer of a numpy array (or None)."""
    return None if a is None else C.c_void_p(a.ctypes.data)
