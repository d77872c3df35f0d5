"""ctypes binding of libsfw_b200.so (declarations: include/sfw_b200.h).

The CUDA library is the only compute path: if it is missing, or no CUDA
device is visible, every entry point raises DeviceError -- there is no CPU
fallback.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (ConfigError, DeviceError, InstabilityError, NumericalError, ProtocolError)

LIB_PATH = os.environ.get("SFW_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsfw_b200.so")

SFW_ECONFIG, SFW_ENUMERICAL, SFW_EINSTABLE, SFW_EPROTOCOL, SFW_ECUDA = -1, -2, -3, -4, -5

_ERRMAP = {SFW_ECONFIG: ConfigError, SFW_ENUMERICAL: NumericalError,
           SFW_EINSTABLE: InstabilityError, SFW_EPROTOCOL: ProtocolError, SFW_ECUDA: DeviceError}

PD = C.POINTER(C.c_double)
PI = C.POINTER(C.c_int)
PF = C.POINTER(C.c_float)
PL = C.POINTER(C.c_longlong)


class StepDesc(C.Structure):
    _fields_ = [
        ("n_sub", C.c_int), ("m", C.c_int), ("layers", PI), ("neighbors", PI),
        ("gammas", PD), ("gamma_hats", PD), ("scales", PD), ("coef_on_device", C.c_int),
        ("dt", C.c_double),
        ("n_src", C.c_int), ("src_sub", PI), ("src_vec", PD),
        ("n_probe", C.c_int), ("probe_sub", PI), ("probe_w", PD),
    ]


class RomDesc(C.Structure):
    """include/sfw_b200.h sfw_rom_desc."""
    _fields_ = [("n_sub", C.c_int), ("p", C.c_int * 3), ("h", C.c_double * 3), ("m", C.c_int),
                ("n", C.c_int), ("shift", C.c_double), ("c", PD), ("nbr_mask", PI),
                ("n_rows", C.c_int), ("row_sub", PI), ("row_node", PI), ("full_basis", C.c_int),
                ("out_on_device", C.c_int), ("batch", C.c_int)]


class RomOut(C.Structure):
    """include/sfw_b200.h sfw_rom_out."""
    _fields_ = [("layers", PI), ("flags", PI), ("status", PI), ("gammas", PD),
                ("gamma_hats", PD), ("scales", PD), ("tdiag", PD), ("toff", PD),
                ("basis_rows", PD), ("basis", PD), ("stats", PD)]


# name -> (restype, argtypes); every symbol include/sfw_b200.h declares
SIGNATURES = {
    "sfw_rom_build": (C.c_int, [C.POINTER(RomDesc), C.POINTER(RomOut), C.c_char_p, C.c_int]),
    "sfw_subdomain_apply": (C.c_int, [C.c_int, PI, PD, PD, PI, C.c_int, PD, PD, C.c_char_p, C.c_int]),
    "sfw_project_state": (C.c_int, [C.c_int, C.c_int, C.c_int, PD, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_state_to_nodes": (C.c_int, [C.c_int, C.c_int, C.c_int, PD, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_last_error": (C.c_char_p, []),
    "sfw_device_info": (C.c_int, [PI, C.c_char_p, C.c_int]),
    "sfw_step_create": (C.c_int, [C.POINTER(StepDesc), C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "sfw_step_init": (C.c_int, [C.c_void_p, PD, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_step_run": (C.c_int, [C.c_void_p, C.c_int, C.c_int, PD, PD, PD, PD, PI, C.c_char_p, C.c_int]),
    "sfw_step_run_resident": (C.c_int, [C.c_void_p, C.c_int, C.c_int, PD, PF, C.c_char_p, C.c_int]),
    "sfw_step_set_probes": (C.c_int, [C.c_void_p, C.c_int, PI, PD, C.c_char_p, C.c_int]),
    "sfw_step_accel": (C.c_int, [C.c_void_p, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_step_power": (C.c_int, [C.c_void_p, PD, C.c_double, C.c_int, PD, PI, PI, C.c_char_p, C.c_int]),
    "sfw_step_masses": (C.c_int, [C.c_void_p, PI, PD, C.c_char_p, C.c_int]),
    "sfw_step_get_state": (C.c_int, [C.c_void_p, PD, PD]),
    "sfw_step_set_state": (C.c_int, [C.c_void_p, PD, PD, C.c_char_p, C.c_int]),
    "sfw_step_energy": (C.c_int, [C.c_void_p, PD, C.c_char_p, C.c_int]),
    "sfw_step_traffic": (C.c_int, [C.c_void_p, PD, PD, PD]),
    "sfw_pulse_table": (C.c_int, [C.c_int, C.c_double, C.c_double, C.c_longlong, C.c_double, C.c_int, PD]),
    "sfw_step_destroy": (C.c_int, [C.c_void_p]),
    "sfw_shots_setup": (C.c_int, [C.c_void_p, C.c_int, PI, PD, C.c_char_p, C.c_int]),
    "sfw_shots_run": (C.c_int, [C.c_void_p, C.c_int, C.c_int, PD, PD, PD, PD, PF, C.c_char_p, C.c_int]),
    "sfw_shots_state": (C.c_int, [C.c_void_p, C.c_int, PD, PD]),
    "sfw_shots_traffic": (C.c_int, [C.c_void_p, PD, PD, PD]),
    "sfw_wform_setup": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    "sfw_wform_vectors": (C.c_int, [C.c_void_p, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_wform_init": (C.c_int, [C.c_void_p, PD, PD, PD, PD, C.c_char_p, C.c_int]),
    "sfw_wform_run": (C.c_int, [C.c_void_p, C.c_int, C.c_int, PD, PD, PD, PD, PI, PF, C.c_char_p, C.c_int]),
    "sfw_wform_state": (C.c_int, [C.c_void_p, PD, PD, C.c_char_p, C.c_int]),
    "sfw_wform_traffic": (C.c_int, [C.c_void_p, PD, PD]),
    "sfw_wform_destroy": (C.c_int, [C.c_void_p]),
    "sfw_source_vector": (C.c_int, [C.c_int, C.c_int, PD, PD, C.c_double, PD, PD, C.c_char_p, C.c_int]),
    "sfw_probe_weights": (C.c_int, [C.c_int, C.c_int, PD, PD, C.c_double, PD, C.c_char_p, C.c_int]),
    "sfw_fdtd_create": (C.c_int, [C.c_int, C.c_int, C.c_int, PD, PD, C.POINTER(C.c_void_p), C.c_char_p, C.c_int]),
    "sfw_fdtd_apply": (C.c_int, [C.c_void_p, PD, PD, C.c_char_p, C.c_int]),
    "sfw_fdtd_power": (C.c_int, [C.c_void_p, PD, C.c_double, C.c_int, PD, PI, C.c_char_p, C.c_int]),
    "sfw_fdtd_setup": (C.c_int, [C.c_void_p, C.c_int, PL, PD, C.c_int, PL, PD, C.c_char_p, C.c_int]),
    "sfw_fdtd_init": (C.c_int, [C.c_void_p, C.c_double, PD, PD, C.c_double, C.c_char_p, C.c_int]),
    "sfw_fdtd_run": (C.c_int, [C.c_void_p, C.c_double, C.c_int, PD, C.c_int, PD, PD, PF, C.c_char_p, C.c_int]),
    "sfw_fdtd_state": (C.c_int, [C.c_void_p, PD, PD, C.c_char_p, C.c_int]),
    "sfw_fdtd_destroy": (C.c_int, [C.c_void_p]),
    "sfw_ntd_batch": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, PD, PD, PD, C.c_int, PI, PD, PD, PI, C.c_char_p,
                                C.c_int]),
    "sfw_ntd_operator": (C.c_int, [C.c_int, PI, PI, PD, C.c_int, PD, C.c_int, PD, PD, PD, PI, C.c_char_p,
                                   C.c_int]),
    "sfw_face_inputs": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, PD, C.c_char_p, C.c_int]),
}

_lib = None


def load(require_device: bool = True):
    """Load the shared library (and, by default, insist on a CUDA device)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"{LIB_PATH} is missing; build it with `make` (no CPU fallback exists)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    if require_device:
        n_sm = C.c_int(0)
        name = C.create_string_buffer(128)
        cc = _lib.sfw_device_info(C.byref(n_sm), name, 128)
        if cc < 0:
            raise DeviceError("no CUDA device visible; the sm_100a path has no CPU fallback")
        if cc < 100:
            raise DeviceError(f"device {name.value.decode()} (cc {cc}) is not sm_100a")
    return _lib


def device_info():
    lib = load(require_device=False)
    n_sm = C.c_int(0)
    name = C.create_string_buffer(128)
    cc = lib.sfw_device_info(C.byref(n_sm), name, 128)
    return cc, n_sm.value, name.value.decode()


def check(rc: int, errbuf, what: str = ""):
    if rc == 0:
        return
    msg = errbuf.value.decode(errors="replace") if errbuf is not None else ""
    exc = _ERRMAP.get(rc, DeviceError)
    raise exc(f"{what}: {msg}" if what and not msg.startswith(what) else msg or what)


def errbuf():
    return C.create_string_buffer(1024)


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(PD)


def lptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(PL)


def iptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(PI)
