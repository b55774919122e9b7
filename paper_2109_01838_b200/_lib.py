"""ctypes binding of the C ABI in include/rama_b200.h.

The B200 build has no CPU fallback: importing works anywhere (so host-side
logic can be tested without a GPU), but every compute call raises if the
CUDA library or a CUDA device is missing.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RAMA_LIB (A/B experiments): another build of the same library
LIB_PATH = os.environ.get("RAMA_LIB") or os.path.join(_HERE, "_lib", "librama_b200.so")

_i32p = ctypes.c_void_p  # device pointers travel as void*
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double
_vp = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)
_I32P = ctypes.POINTER(ctypes.c_int32)

RAMA_OK = 0
RAMA_ERR_INVALID = 1
RAMA_ERR_CUDA = 2
RAMA_ERR_NOMEM = 3

MODE_IDS = {"P": 0, "PD": 1, "PD+": 2, "D": 3, "GAEC": 4}
PHASE_NAMES = {0: "contract", 1: "primal-dual", 2: "cleanup", 3: "dual", 4: "gaec"}


class RamaCfg(ctypes.Structure):
    _fields_ = [
        ("mode", ctypes.c_int32),
        ("mp_iterations", ctypes.c_int32),
        ("max_cycle_length", ctypes.c_int32),
        ("max_rounds", ctypes.c_int32),
        ("separation_rounds", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("matching_switch_fraction", ctypes.c_double),
    ]


class RamaRound(ctypes.Structure):
    _fields_ = [
        ("round_index", ctypes.c_int32),
        ("phase", ctypes.c_int32),
        ("nodes", ctypes.c_int64),
        ("edges", ctypes.c_int64),
        ("triplets", ctypes.c_int64),
        ("lb", ctypes.c_double),
        ("lb_valid", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("contracted", ctypes.c_int64),
        ("time_ms", ctypes.c_double),
    ]


# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGS = {
    "rama_version": [],
    "rama_last_error": [],
    "rama_last_launch_count": [],
    "rama_profile_enable": [_i32],
    "rama_profile_read": [_F64P, _F64P, _I64P],
    "rama_profile_kernels": [ctypes.c_char_p, _i64],
    "rama_io_last_error": [],
    "rama_parse_multicut": [_vp, _i64, ctypes.c_char_p, _I64P, _I64P, _vp, _vp, _vp, _i64, _i32],
    "rama_serialize_multicut": [_i64, _vp, _vp, _vp, _i64, _vp, _i64, _I64P, _i32],
    "rama_solve": [_i64, _vp, _vp, _vp, _i64, ctypes.POINTER(RamaCfg), _vp, _F64P, ctypes.POINTER(RamaRound), _i32,
                   _I32P, _vp],
    "rama_solve_ws": [_i64, _vp, _vp, _vp, _i64, ctypes.POINTER(RamaCfg), _vp, _F64P, ctypes.POINTER(RamaRound), _i32,
                      _I32P, _vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), _vp],
    "rama_ws_bytes": [_i64, _i64, ctypes.POINTER(RamaCfg)],
    "rama_release_cache": [],
    "rama_solve_host": [_i64, _vp, _vp, _vp, _i64, ctypes.POINTER(RamaCfg), _vp, _F64P, ctypes.POINTER(RamaRound),
                        _i32, _I32P, _vp],
    "rama_solve_batch": [_i64, _I64P, _I64P, _vp, _vp, _vp, ctypes.POINTER(RamaCfg), _vp, _F64P,
                         ctypes.POINTER(RamaRound), _i32, _I32P, _i32, _vp],
    "rama_canonicalize": [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _I64P, _vp],
    "rama_clustering_cost": [_i64, _vp, _vp, _vp, _i64, _vp, _F64P, _vp],
    "rama_components": [_i64, _vp, _vp, _i64, _vp, _I64P, _vp],
    "rama_contract": [_i64, _vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _I64P, _F64P, _vp],
    "rama_select_matching": [_i64, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _I64P, _vp],
    "rama_select_max_edge": [_i64, _vp, _vp, _vp, _i64, _I64P, _vp],
    "rama_select_forest": [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _I64P, _vp],
    "rama_contraction_step": [_i64, _vp, _vp, _vp, _i64, _i32, _f64, _vp, _vp, _vp, _vp, _I64P, _F64P, _vp],
    "rama_separate": [_i64, _vp, _vp, _vp, _i64, _i32, _vp, _vp, _I64P, _vp],
    "rama_triangulate": [_i64, _vp, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp, _vp, _I64P, _vp, _vp, _I64P, _vp,
                         _vp],
    "rama_extend_separation": [_i64, _i64, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i32, _i64, _i64, _vp, _vp, _vp, _I64P,
                               _vp, _vp, _vp, _I64P, _vp, _I64P, _vp],
    "rama_check_agreement": [_i64, _vp, _i64, _vp, _vp, _f64, _I32P, _vp],
    "rama_message_passing": [_i64, _vp, _i64, _vp, _vp, _i32, _i32, _vp],
    "rama_reparam_costs": [_i64, _vp, _i64, _vp, _vp, _vp, _vp],
    "rama_lower_bound": [_i64, _vp, _i64, _vp, _vp, _F64P, _vp],
}
_RESTYPES = {"rama_last_error": ctypes.c_char_p, "rama_io_last_error": ctypes.c_char_p, "rama_last_launch_count": ctypes.c_int64,
             "rama_profile_kernels": ctypes.c_int64, "rama_ws_bytes": ctypes.c_uint64}

EXPORTED = tuple(_SIGS)

_lib = None
launches = 0  # kernels launched by library calls in this process


def load():
    """Load the in-tree CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                "B200 CUDA library not built (%s); run `python -m paper_2109_01838_b200._build` "
                "-- there is no CPU fallback" % LIB_PATH)
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def call(name, *args):
    """Invoke a C entry point; map status codes to Python exceptions."""
    global launches
    lib = load()
    rc = getattr(lib, name)(*args)
    launches += int(lib.rama_last_launch_count())
    if rc == RAMA_OK:
        return
    msg = lib.rama_last_error().decode(errors="replace")
    if rc == RAMA_ERR_INVALID:
        raise ValueError(msg)
    if rc == RAMA_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError("%s failed (%d): %s" % (name, rc, msg))


def call_host(name, *args):
    """Host-only entry points (MULTICUT I/O): no CUDA device required."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc == RAMA_OK:
        return
    msg = lib.rama_io_last_error().decode(errors="replace")
    if rc == RAMA_ERR_INVALID:
        raise ValueError(msg)
    raise RuntimeError("%s failed (%d): %s" % (name, rc, msg))


# --------------------------------------------------------- torch plumbing

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        if not t.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 build has no CPU fallback")
        _torch = t
    return _torch


def stream():
    return ctypes.c_void_p(torch().cuda.current_stream().cuda_stream)


def dev(arr, dtype):
    """numpy / torch -> contiguous CUDA tensor of dtype."""
    t = torch()
    if isinstance(arr, t.Tensor):
        return arr.to(device="cuda", dtype=dtype).contiguous()
    a = np.ascontiguousarray(arr)
    return t.from_numpy(a).to(device="cuda", dtype=dtype).contiguous()


def i32(arr):
    return dev(arr, torch().int32)


def f64(arr):
    return dev(arr, torch().float64)


def empty_i32(n):
    return torch().empty(max(int(n), 1), dtype=torch().int32, device="cuda")


def empty_f64(n):
    return torch().empty(max(int(n), 1), dtype=torch().float64, device="cuda")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def host_i64(t, k):
    return t[:k].cpu().numpy().astype(np.int64)


def host_f64(t, k):
    return t[:k].cpu().numpy().astype(np.float64)


FAMILIES = ("separate", "triangulate", "message_passing", "bound", "matching", "forest", "components", "contract",
            "cleanup", "canonicalize")


def profile_enable(on=True):
    call("rama_profile_enable", 1 if on else 0)


def profile_read():
    """{family: (ms, algorithmic_bytes, scopes)} summed since profile_enable."""
    nf = len(FAMILIES)
    ms = (ctypes.c_double * nf)()
    by = (ctypes.c_double * nf)()
    cnt = (ctypes.c_int64 * nf)()
    call("rama_profile_read", ms, by, cnt)
    return {f: (ms[i], by[i], cnt[i]) for i, f in enumerate(FAMILIES)}


def profile_kernels(by_family=False):
    """{kernel: (ms, algorithmic_bytes, launches)} timed since profile_enable;
    by_family: also {family: (kernel ms, bytes, launches)} of the kernels
    launched inside each family scope."""
    import json

    lib = load()
    need = lib.rama_profile_kernels(None, 0)
    buf = ctypes.create_string_buffer(int(need) + 4096)
    lib.rama_profile_kernels(buf, len(buf))
    raw = json.loads(buf.value.decode())
    kern = {k: tuple(v) for k, v in raw.items() if not k.startswith("@")}
    if not by_family:
        return kern
    fam = {FAMILIES[int(k[1:])]: tuple(v) for k, v in raw.items() if k.startswith("@")}
    return kern, fam
