"""ctypes binding to ``libesp_b200.so`` (C ABI declared in include/esp_b200.h).

The library is the product: there is no CPU fallback.  Importing the
binding when the library is missing raises immediately, and every entry point
checks the status code and re-raises the reference's exception classes
(PlanningError / MeshError / ParameterError) or :class:`EspCudaError`.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import EspCudaError, InputError, MeshError, ParameterError, PlanningError

_HERE = os.path.dirname(os.path.abspath(__file__))
# ESP_LIB overrides the library path (experiments with variant builds)
LIB_PATH = os.environ.get("ESP_LIB") or os.path.join(_HERE, "libesp_b200.so")

ESP_OK = 0
ESP_ERR_PLANNING = 1
ESP_ERR_MESH = 2
ESP_ERR_PARAM = 3
ESP_ERR_CUDA = 4
ESP_ERR_CUFFT = 5
ESP_ERR_OOM = 6
ESP_ERR_CAPACITY = 7
ESP_ERR_INPUT = 8

ESP_FP64 = 0
ESP_FP32 = 1

ESP_WANT_ENERGY_PRESSURE = 1
ESP_WANT_FORCES = 2
ESP_FORCES_ANALYTIC = 4

ESP_NEAR_ACCUMULATE = 1

_dp = C.POINTER(C.c_double)


class SlabDesc(C.Structure):
    """esp_slab_desc (include/esp_b200.h)."""
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("z_start", C.c_int32 * 9),
                ("fwd_peers", C.c_void_p * 8), ("back_peers", C.c_void_p * 8)]


class PlanDesc(C.Structure):
    _fields_ = [
        ("M", C.c_int32 * 3),
        ("P", C.c_int32),
        ("precision", C.c_int32),
        ("deterministic", C.c_int32),
        ("max_particles", C.c_int64),
        ("n_pieces", C.c_int32),
        ("degree", C.c_int32),
        ("h_window_coef", _dp),
        ("h_window_deriv_coef", _dp),
        ("h_window_breaks", _dp),
        ("n_legendre", C.c_int32),
        ("h_legendre", _dp),
        ("n_legendre_deriv", C.c_int32),
        ("h_legendre_deriv", _dp),
        ("split_c", C.c_double),
        ("split_lambda0", C.c_double),
        ("split_C0", C.c_double),
        ("r_c", C.c_double),
        ("kmax", C.c_double),
        ("tile", C.c_int32 * 3),
        ("slab_mz_global", C.c_int32),
        ("slab_z0", C.c_int32),
    ]


class CellDesc(C.Structure):
    _fields_ = [
        ("h", C.c_double * 9),
        ("hinv", C.c_double * 9),
        ("orthorhombic", C.c_int32),
        ("spacing", C.c_double * 3),
        ("volume", C.c_double),
        ("volume_element", C.c_double),
        ("h_axis_k", _dp * 9),
        ("h_axis_what", _dp * 3),
        ("what_zero", C.c_double),
        ("band", C.c_int32 * 3),
        ("grad_scale", C.c_double * 3),
    ]


class NearDesc(C.Structure):
    """esp_near_desc (include/esp_b200.h)."""
    _fields_ = [
        ("r_c", C.c_double),
        ("reach", C.c_double),
        ("use_table", C.c_int32),
        ("r_in", C.c_double),
        ("poly_order", C.c_int32),
        ("h_smooth_poly", _dp),
        ("h_fn_poly", _dp),
        ("n_knots", C.c_int32),
        ("h_knots", _dp),
        ("h_smooth_spline", _dp),
        ("h_fn_spline", _dp),
        ("n_legendre", C.c_int32),
        ("h_legendre", _dp),
        ("n_cumint", C.c_int32),
        ("h_cumint", _dp),
        ("C0", C.c_double),
        ("max_particles", C.c_int64),
        ("cell_div", C.c_int32),
    ]


_lib = None


def lib():
    """Load the CUDA library (fails loudly if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"ESP CUDA library not found at {LIB_PATH}; run "
            "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback "
            "exists for the k-space path)")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.esp_last_error.restype = C.c_char_p
    L.esp_version.restype = C.c_int
    L.esp_copy_async.argtypes = [vp, vp, C.c_int64, vp]
    L.esp_host_alloc.argtypes = [C.c_int64, C.POINTER(vp)]
    L.esp_host_free.argtypes = [vp]
    L.esp_set_charges_event.argtypes = [vp, vp]
    L.esp_set_host_forces.argtypes = [vp, vp, C.c_int32]
    L.esp_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(vp)]
    L.esp_plan_destroy.argtypes = [vp]
    L.esp_plan_set_cell.argtypes = [vp, C.POINTER(CellDesc), vp]
    L.esp_spread.argtypes = [vp, vp, vp, C.c_int64, vp, vp]
    L.esp_forward.argtypes = [vp, vp, vp]
    L.esp_scale_reduce.argtypes = [vp, vp, C.c_int32, vp]
    L.esp_forces_ik.argtypes = [vp, vp, vp]
    L.esp_forces_analytic.argtypes = [vp, vp, vp]
    L.esp_gather_fields.argtypes = [vp, vp, vp, vp]
    L.esp_local_pressure.argtypes = [vp, vp, vp]
    L.esp_evaluate.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, vp, vp, vp]
    L.esp_counters.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.esp_reset_counters.argtypes = [vp]
    L.esp_add_counters.argtypes = [vp, C.c_int64, C.c_int64]
    L.esp_grid_ptr.argtypes = [vp]
    L.esp_grid_ptr.restype = vp
    L.esp_spectrum_ptr.argtypes = [vp]
    L.esp_spectrum_ptr.restype = vp
    L.esp_fields_ptr.argtypes = [vp]
    L.esp_fields_ptr.restype = vp
    L.esp_fields_layout.argtypes = [vp, C.POINTER(C.c_int64)]
    L.esp_grid_info.argtypes = [vp, C.POINTER(C.c_int64)]
    L.esp_binning_radix.argtypes = [vp, C.c_int64, C.POINTER(C.c_int32)]
    L.esp_fft_path.argtypes = [vp]
    L.esp_slab_layout.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]
    L.esp_slab_forward.argtypes = [vp, C.POINTER(SlabDesc), vp, vp]
    L.esp_slab_reduce.argtypes = [vp, C.POINTER(SlabDesc), vp, C.c_int32, vp, vp]
    L.esp_slab_inverse.argtypes = [vp, C.POINTER(SlabDesc), vp, vp, vp]
    L.esp_set_spectrum.argtypes = [vp, vp, vp]
    L.esp_set_profiling.argtypes = [vp, C.c_int32]
    L.esp_profile_read.argtypes = [vp, C.c_char_p, C.c_int32, C.POINTER(C.c_double), C.c_int32]
    L.esp_probe_fp64.argtypes = [C.POINTER(C.c_double), vp]
    L.esp_near_create.argtypes = [C.POINTER(NearDesc), C.POINTER(vp)]
    L.esp_near_destroy.argtypes = [vp]
    L.esp_near_reserve.argtypes = [vp, C.c_int64, C.c_int64]
    L.esp_near_set_cell.argtypes = [vp, _dp, _dp, C.c_int32, C.c_double]
    L.esp_near_evaluate.argtypes = [vp, vp, vp, C.c_int64, C.c_int32, vp, vp, vp, vp]
    L.esp_near_evaluate_local.argtypes = [vp, vp, vp, C.c_int64, C.c_int64, C.c_int32, vp, vp,
                                          vp, vp]
    L.esp_near_evaluate_pairs.argtypes = [vp, vp, vp, C.c_int64, vp, vp, C.c_int64,
                                          C.c_int32, vp, vp, vp, vp]
    L.esp_near_info.argtypes = [vp, C.POINTER(C.c_int64)]
    L.esp_near_build_pairs.argtypes = [vp, vp, C.c_int64, C.POINTER(C.c_int64), vp]
    L.esp_near_copy_pairs.argtypes = [vp, vp, vp, vp]
    L.esp_particles_read.argtypes = [C.c_char_p, C.POINTER(vp)]
    L.esp_particles_info.argtypes = [vp, C.POINTER(C.c_int64), C.POINTER(C.c_int32), _dp]
    L.esp_particles_copy.argtypes = [vp, _dp, _dp, _dp]
    L.esp_particles_free.argtypes = [vp]
    L.esp_particles_write.argtypes = [C.c_char_p, C.c_int64, _dp, C.c_int32, _dp, _dp, _dp]
    _lib = L
    return L


EXPORTED = [
    "esp_plan_create", "esp_plan_destroy", "esp_plan_set_cell", "esp_last_error",
    "esp_version", "esp_copy_async", "esp_host_alloc", "esp_host_free",
    "esp_set_charges_event", "esp_set_host_forces", "esp_spread", "esp_forward", "esp_scale_reduce", "esp_forces_ik",
    "esp_forces_analytic", "esp_local_pressure", "esp_evaluate", "esp_counters",
    "esp_reset_counters", "esp_add_counters", "esp_grid_ptr", "esp_spectrum_ptr", "esp_grid_info",
    "esp_binning_radix",
    "esp_set_spectrum", "esp_set_profiling", "esp_profile_read", "esp_probe_fp64",
    "esp_gather_fields", "esp_fields_ptr", "esp_fields_layout", "esp_fft_path",
    "esp_slab_layout", "esp_slab_forward", "esp_slab_reduce", "esp_slab_inverse",
    "esp_near_create", "esp_near_destroy", "esp_near_reserve", "esp_near_set_cell",
    "esp_near_evaluate", "esp_near_evaluate_local", "esp_near_evaluate_pairs", "esp_near_info", "esp_near_build_pairs",
    "esp_near_copy_pairs", "esp_particles_read", "esp_particles_info", "esp_particles_copy",
    "esp_particles_free", "esp_particles_write",
]


def check(rc: int, what: str = "") -> None:
    if rc == ESP_OK:
        return
    msg = lib().esp_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == ESP_ERR_PLANNING:
        raise PlanningError(text)
    if rc == ESP_ERR_MESH:
        raise MeshError(text)
    if rc in (ESP_ERR_PARAM, ESP_ERR_CAPACITY):
        raise ParameterError(text)
    if rc == ESP_ERR_INPUT:
        raise InputError(msg)
    raise EspCudaError(f"[{rc}] {text}")


class HostBuffer:
    """Page-locked host memory from ``esp_host_alloc`` viewed as a CPU torch
    tensor (freed with the object)."""

    def __init__(self, shape, dtype=None):
        import numpy as np
        import torch
        dtype = dtype or torch.float64
        n = 1
        for d in shape:
            n *= int(d)
        item = torch.empty(0, dtype=dtype).element_size()
        self._p = C.c_void_p()
        check(lib().esp_host_alloc(n * item, C.byref(self._p)), "esp_host_alloc")
        npd = {torch.float64: np.float64, torch.float32: np.float32,
               torch.int64: np.int64}[dtype]
        buf = (C.c_char * max(n * item, 1)).from_address(self._p.value)
        arr = np.frombuffer(buf, dtype=npd, count=n).reshape(shape)
        self.tensor = torch.from_numpy(arr)

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            if self._p and self._p.value:
                lib().esp_host_free(self._p)
                self._p = None
        except Exception:
            pass
