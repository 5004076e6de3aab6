"""ctypes binding of libcurvekit_b200.so (the C-ABI in include/curvekit_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, every entry point raises ``RuntimeError`` (loudly, by design).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# CKB_LIB: tuning / checking variants (a relative path is taken from the repository root, so
# subprocesses with another working directory load the same library)
LIB_PATH = os.environ.get("CKB_LIB") or os.path.join(HERE, "libcurvekit_b200.so")
if not os.path.isabs(LIB_PATH):
    LIB_PATH = os.path.join(os.path.dirname(HERE), LIB_PATH)

# every symbol include/curvekit_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "ckb_abi_version", "ckb_last_error", "ckb_init", "ckb_shutdown", "ckb_launch_count",
    "ckb_biv_resultant", "ckb_reduce", "ckb_uni_resultant_batch", "ckb_interp_plan_points",
    "ckb_interp_geometric", "ckb_crt_lift", "ckb_dev_modular_images", "ckb_dev_crt",
    "ckb_interp_points", "ckb_gcd_mod_batch", "ckb_dev_biv_resultant", "ckb_set_timing",
    "ckb_stage_times", "ckb_measure_peak", "ckb_psc_values", "ckb_host_alloc", "ckb_host_free",
    "ckb_descartes_prepare", "ckb_descartes_variations", "ckb_descartes_release", "ckb_biv_gcd_images",
    "ckb_biv_resultant_batch", "ckb_descartes_variations_batch", "ckb_set_graphs",
    "ckb_init_devices", "ckb_devices", "ckb_biv_resultant_multi", "ckb_subres_profile", "ckb_last_fallback",
    "ckb_last_exchange",
    "ckb_host_times",
)

_P = ctypes.c_void_p
_I = ctypes.c_int
_U32P = ctypes.POINTER(ctypes.c_uint32)

# full C signatures (pointers must never be passed as 32-bit ints)
_SIGS = {
    "ckb_abi_version": (_I, []),
    "ckb_last_error": (ctypes.c_char_p, []),
    "ckb_init": (_I, [_I]),
    "ckb_shutdown": (_I, []),
    "ckb_launch_count": (ctypes.c_ulonglong, []),
    "ckb_biv_resultant": (_I, [_P, _I, _I, _P, _I, _I, _I, _I, _P, _P, _I, _I, _I, _P, _P, _P]),
    "ckb_reduce": (_I, [_P, _I, _I, _P, _I, _P]),
    "ckb_uni_resultant_batch": (_I, [_P, _P, _P, _P, _I, _P, _I, _P, _I, _P]),
    "ckb_interp_plan_points": (_I, [_P, _P, _I, _I, _P]),
    "ckb_interp_geometric": (_I, [_P, _P, _P, _I, _I, _P]),
    "ckb_crt_lift": (_I, [_P, _I, _I, _P, _I, _P]),
    "ckb_gcd_mod_batch": (_I, [_P, _P, _I, _P, _P, _I, _P, _I, _P, _I, _P, _I, _P]),
    "ckb_interp_points": (_I, [_P, _P, _P, _I, _P, _I, _P, _I, _P]),
    "ckb_dev_modular_images": (_I, [_P, _I, _I, _P, _P, _I, _I, _I, _I, _P, _P, _I, _I, _P, _P, _P]),
    "ckb_dev_crt": (_I, [_P, _I, _I, _P, _I, _P, _P]),
    "ckb_dev_biv_resultant": (_I, [_P, _I, _I, _P, _P, _I, _I, _I, _I, _P, _P, _I, _I, _I, _P, _P, _P]),
    "ckb_set_timing": (_I, [_I]),
    "ckb_set_graphs": (_I, [_I]),
    "ckb_stage_times": (_I, [_P, _I]),
    "ckb_measure_peak": (_I, [_P, _I]),
    "ckb_psc_values": (_I, [_P, _P, _I, _I, _P, _P, _I, _I, ctypes.c_uint32, _I, _P, _P]),
    "ckb_host_alloc": (_P, [ctypes.c_ulonglong]),
    "ckb_host_free": (_I, [_P]),
    "ckb_descartes_prepare": (_I, [_P, _I, _I, _P, _P, _I]),
    "ckb_descartes_variations": (_I, [_I, _P, _I, _I, _I, _I, _P]),
    "ckb_descartes_release": (_I, [_I]),
    "ckb_biv_resultant_batch": (_I, [_I] + [_P] * 15),
    "ckb_descartes_variations_batch": (_I, [_I, _P, _I, _P, _I, _I, _I, _P]),
    "ckb_biv_gcd_images": (_I, [_P, _I, _I, _P, _I, _I, _I, _I, _I, _P, _I, _I, _P, _I, _P]),
    "ckb_init_devices": (_I, [_I, _P]),
    "ckb_last_fallback": (_I, [_P, _P]),
    "ckb_last_exchange": (_I, []),
    "ckb_host_times": (_I, [_P, _I]),
    "ckb_subres_profile": (_I, [_P, _P, _I, _I, _P, _P, _I, _I, _P, _I, _I, _I, ctypes.c_uint32, _P]),
    "ckb_devices": (_I, [_P, _P]),
    "ckb_biv_resultant_multi": (_I, [_P, _I, _I, _P, _I, _I, _I, _I, _P, _P, _I, _I, _I, _I, _P, _P, _P]),
}

_lock = threading.Lock()
_lib = None
_ready = False


class CkbError(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the library (no device work).  Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise CkbError(f"{path} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
                       "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name in EXPORTS:
        getattr(lib, name)  # raises AttributeError if not exported
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def _device_index() -> int:
    for var in ("CKB_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(var)
        if v is not None and v != "":
            return int(v)
    return 0


def _device_list():
    """CKB_DEVICES="0,1,2,3" (explicit list; a device may repeat) or CKB_GPUS=N
    (devices 0..N-1): the drop-in then shards every res_y over those GPUs."""
    v = os.environ.get("CKB_DEVICES")
    if v:
        return [int(x) for x in v.split(",") if x.strip() != ""]
    n = int(os.environ.get("CKB_GPUS", "1") or 1)
    return list(range(n)) if n > 1 else None


def lib():
    """The initialised library (lazily binds the CUDA device(s))."""
    global _ready
    lb = load()
    if not _ready:
        with _lock:
            if not _ready:
                devs = _device_list()
                if devs:
                    arr = (ctypes.c_int * len(devs))(*devs)
                    rc = lb.ckb_init_devices(len(devs), ctypes.cast(arr, _P))
                else:
                    rc = lb.ckb_init(_device_index())
                if rc != 0:
                    raise CkbError("ckb_init failed: " + lb.ckb_last_error().decode())
                _ready = True
    return lb


def use_devices(devices) -> int:
    """Shard res_y over these devices from now on (one context per entry; the
    first must be the device already in use, if any).  Returns the count."""
    lb = lib()
    arr = (ctypes.c_int * len(devices))(*devices)
    check(lb.ckb_init_devices(len(devices), ctypes.cast(arr, _P)), "ckb_init_devices")
    return len(devices)


def n_devices() -> int:
    """Device contexts the drop-in shards over (1 = single GPU)."""
    n, nc = ctypes.c_int(0), ctypes.c_int(0)
    lib().ckb_devices(ctypes.byref(n), ctypes.byref(nc))
    return max(1, n.value)


def last_fallback() -> tuple:
    """(images sent to the general warp kernel, all images) of the last res_y call."""
    a, b = ctypes.c_ulonglong(0), ctypes.c_ulonglong(0)
    check(lib().ckb_last_fallback(ctypes.byref(a), ctypes.byref(b)), "ckb_last_fallback")
    return int(a.value), int(b.value)


def last_exchange() -> str:
    """How the last multi-device res_y exchanged residues."""
    return {0: "none", 1: "peer-store", 2: "nccl", 3: "peer-copy"}.get(int(lib().ckb_last_exchange()), "?")


def uses_nccl() -> bool:
    n, nc = ctypes.c_int(0), ctypes.c_int(0)
    lib().ckb_devices(ctypes.byref(n), ctypes.byref(nc))
    return bool(nc.value)


def check(rc: int, what: str) -> int:
    if rc < 0:
        raise CkbError(f"{what} failed: {_lib.ckb_last_error().decode()}")
    return rc


def ptr(a: np.ndarray):
    """ctypes pointer to a C-contiguous numpy array."""
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data_as(_P)


class PinnedPool(threading.local):
    """Per-thread grow-only page-locked uint32 buffers by name (the pipeline
    copies to / from page-locked memory directly).  A view is valid until the
    same thread asks for a larger buffer of that name."""

    def __init__(self):
        self._bufs = {}

    def get(self, name: str, count: int) -> np.ndarray:
        cur = self._bufs.get(name)
        if cur is None or cur[1] < count:
            lb = lib()
            if cur is not None:
                lb.ckb_host_free(cur[0])
            want = max(count, 1024) + count // 4
            p = lb.ckb_host_alloc(4 * want)
            if not p:
                raise CkbError("ckb_host_alloc failed: " + lb.ckb_last_error().decode())
            cur = (p, want)
            self._bufs[name] = cur
        arr = np.ctypeslib.as_array(ctypes.cast(cur[0], _U32P), shape=(cur[1],))
        return arr[:count]


pinned = PinnedPool()


def launch_count() -> int:
    return int(lib().ckb_launch_count())
