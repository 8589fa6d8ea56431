"""ctypes binding of the C ABI in include/wssr.h (libwssr.so, built by __graft_entry__.build()).

There is deliberately no fallback: if the shared library is missing or no CUDA device is
present, every entry point raises.  PyTorch is used only to own device memory and to provide
the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
# WSSR_LIB points the binding at another build of the same ABI (A/B runs of kernel variants)
LIB_PATH = os.environ.get("WSSR_LIB") or os.path.join(_HERE, "lib", "libwssr.so")

WSSR_OK = 0
WSSR_FLAG_FINAL_RESIDUAL = 0x1
WSSR_FLAG_CAREFUL = 0x2

_c_double_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_dbl = ctypes.c_double


class OhatF64(ctypes.Structure):
    _fields_ = [
        ("n_params", _i64),
        ("hist", _vp), ("hist_rank", _i64), ("hist_ld", _i64), ("hist_scale", _dbl),
        ("samples", _vp), ("n_samples", _i64), ("samples_ld", _i64), ("mu", _vp),
        ("samples_scale", _dbl), ("samples_fro2", _dbl), ("samples_f32", _i64),
        ("samples_scale_table", _vp), ("samples_fro2_dev", _vp),
    ]


class AssembleOut(ctypes.Structure):
    _fields_ = [
        ("mu", _vp), ("l_vector", _vp), ("gradient", _vp),
        ("loss", _dbl), ("raw_loss", _dbl), ("e_mean", _dbl), ("e_std", _dbl),
        ("fro2", _dbl), ("n_global", _i64), ("scale_table", _vp),
        ("deferred", _vp), ("fro2_dev", _vp),
    ]


class AceSpec(ctypes.Structure):
    _fields_ = [
        ("n_electrons", _i64), ("n_orbitals", _i64), ("n_features", _i64), ("n_nuclei", _i64),
        ("max_tail", _i64), ("nuclei", _vp), ("spins", _vp), ("orb_center", _vp), ("orb_n", _vp),
        ("orb_axis", _vp), ("orb_gate", _vp), ("orb_zeta", _vp), ("heads", _vp), ("tails", _vp),
        ("coef", _vp),
    ]


class SsiOut(ctypes.Structure):
    _fields_ = [
        ("u", _vp), ("ld_u", _i64), ("sigma", _vp), ("v", _vp), ("ld_v", _i64),
        ("k_pos", _i64), ("iterations", _i64), ("residual", _dbl),
    ]


class StepIn(ctypes.Structure):
    _fields_ = [
        ("ohat", ctypes.POINTER(OhatF64)),
        ("lbar", _vp), ("l_vector", _vp), ("gradient", _vp), ("theta", _vp), ("eta", _dbl),
        ("u_init", _vp), ("ld_init", _i64), ("requested", _i64),
        ("u_prev", _vp), ("ld_prev", _i64), ("r_prev", _i64),
        ("delta", _dbl), ("sigma_floor", _dbl), ("r_reg", _dbl), ("eps_grow", _dbl),
        ("sigma_floor_relative", _i64), ("r_max", _i64), ("max_iters", _i64),
        ("residual_tol", _dbl), ("flags", _i64),
        ("ext_u", _vp), ("ext_ld_u", _i64), ("ext_sigma", _vp), ("ext_v", _vp),
        ("ext_ld_v", _i64), ("ext_k_pos", _i64),
    ]


class StepOut(ctypes.Structure):
    _fields_ = [
        ("theta_next", _vp), ("update", _vp), ("u_next", _vp), ("ld_u", _i64),
        ("obar_next_t", _vp), ("ld_obar", _i64), ("lbar_next", _vp), ("sigma", _vp),
        ("r_eff", _i64), ("k_pos", _i64), ("iterations", _i64), ("next_r_max", _i64),
        ("binding", _i64),
        ("residual", _dbl), ("sigma_drift", _dbl), ("projector_drift", _dbl),
        ("drift_host", _vp),
    ]


# (name, restype, argtypes) for every symbol include/wssr.h declares
SIGNATURES = {
    "wssr_version": (ctypes.c_int, []),
    "wssr_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "wssr_ctx_destroy": (None, [_vp]),
    "wssr_last_error": (ctypes.c_char_p, [_vp]),
    "wssr_set_stream": (ctypes.c_int, [_vp, _vp]),
    "wssr_kernel_launches": (_i64, [_vp]),
    "wssr_set_gemm_path": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_set_precision_guard": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_precision_fallbacks": (_i64, [_vp]),
    "wssr_set_timing": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_set_tallskinny": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_set_dense_svd_mode": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_set_fp32_digits": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_ozaki_digit_pairs": (ctypes.c_int, []),
    "wssr_set_tail_shard": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wssr_release_memory": (ctypes.c_int, [_vp]),
    "wssr_dense_svd_sweeps": (ctypes.c_int, [_vp]),
    "wssr_set_aux_stream": (ctypes.c_int, [_vp, _vp]),
    "wssr_grad_theta_f64": (ctypes.c_int, [_vp, ctypes.POINTER(AceSpec), _vp, _i64, _vp, _i64]),
    "wssr_debug_tallskinny": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i64, _vp, _vp, _vp, _vp,
                                             _dbl, _vp]),
    "wssr_phase_stats": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(_dbl),
                                        ctypes.POINTER(_i64), ctypes.POINTER(_dbl),
                                        ctypes.POINTER(_dbl)]),
    "wssr_dmma_peak_probe": (ctypes.c_int, [_vp, ctypes.POINTER(_dbl)]),
    "wssr_nccl_unique_id": (ctypes.c_int, [_vp, ctypes.c_char_p]),
    "wssr_nccl_attach": (ctypes.c_int, [_vp, ctypes.c_char_p, ctypes.c_int, ctypes.c_int]),
    "wssr_allreduce_f64": (ctypes.c_int, [_vp, _vp, ctypes.c_int64]),
    "wssr_emu_group_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_vp)]),
    "wssr_emu_group_abort": (None, [_vp]),
    "wssr_emu_group_destroy": (None, [_vp]),
    "wssr_emu_attach": (ctypes.c_int, [_vp, _vp, ctypes.c_int]),
    "wssr_assemble_f64": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _dbl,
                                         ctypes.POINTER(AssembleOut)]),
    "wssr_assemble_f32": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _vp, _dbl,
                                         ctypes.POINTER(AssembleOut)]),
    "wssr_qr_f64": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _i64]),
    "wssr_ssi_svd_f64": (ctypes.c_int, [_vp, ctypes.POINTER(OhatF64), _i64, _i64, _vp, _i64,
                                        _dbl, _i64, ctypes.POINTER(SsiOut)]),
    "wssr_subspace_drift_f64": (ctypes.c_int, [_vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64, _vp,
                                               _i64, ctypes.POINTER(_dbl),
                                               ctypes.POINTER(_dbl)]),
    "wssr_step_f64": (ctypes.c_int, [_vp, ctypes.POINTER(StepIn), ctypes.POINTER(StepOut)]),
    "wssr_exact_svd_f64": (ctypes.c_int, [_vp, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64]),
    "wssr_materialize_ohat_f64": (ctypes.c_int, [_vp, ctypes.POINTER(OhatF64), _dbl, _vp, _i64]),
    "wssr_implicit_svd_f64": (ctypes.c_int, [_vp, ctypes.POINTER(OhatF64), _dbl, _i64, _i64, _i64,
                                             ctypes.c_uint64, _i64, _dbl, _vp, _i64, _vp, _vp,
                                             _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                             ctypes.POINTER(_dbl)]),
    "wssr_debug_small_f64": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp,
                                            ctypes.POINTER(ctypes.c_int)]),
    "wssr_debug_gemm_f32a": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _vp,
                                            _vp, _i64, _vp, _i64, _dbl]),
    "wssr_debug_ozaki_gemm": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_int64, _vp, ctypes.c_int64, ctypes.c_int,
                                              _vp, _vp, ctypes.c_int64, _vp, ctypes.c_int64,
                                              ctypes.c_double]),
    "wssr_debug_ozaki_trace": (ctypes.c_int, [_vp, _vp, ctypes.c_int64]),
    "wssr_gemm_f64": (ctypes.c_int, [_vp, ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _vp, _vp,
                                     _i64, _vp, _i64, _dbl, ctypes.c_int, ctypes.c_int]),
}

_STATUS = {
    1: ValueError,
    2: errors.RankTooLarge,
    3: errors.DegenerateInput,
    4: errors.ZeroMatrix,
    5: errors.RankCollapse,
    6: errors.DegenerateBatch,
    7: errors.DeviceError,
    8: errors.DeviceError,
    9: errors.Unsupported,
    10: errors.NodeProximity,
}

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libwssr.so and declare every prototype.  Raises if it is missing."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ImportError(
                f"libwssr.so not found at {path}; run __graft_entry__.build() first "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


class Context:
    """One native context per CUDA device (reference: single control thread)."""

    def __init__(self, device: int):
        lib = load_library()
        h = _vp()
        rc = lib.wssr_ctx_create(int(device), ctypes.byref(h))
        if rc != WSSR_OK:
            raise errors.DeviceError(f"wssr_ctx_create(device={device}) failed with status {rc}")
        self.lib = lib
        self.handle = h
        self.device = int(device)
        self.rank = 0
        self.world = 1
        self._aux = None
        self._pinned = None
        self._pinned_next = 0

    def pinned_slot(self, n: int):
        """n float64 of pinned host memory for stream-ordered device->host scalars.  Slots come
        from a context-owned ring (never handed back to torch's host allocator), so a copy still
        in flight can never land in memory that was reused for something else; a slot is
        recycled only 4096 requests later (~2000 steps), long after its copy completed; the
        holders (bundle scalars, drift telemetry) copy their values out on first read, and
        wssr_step reads the bundle's as soon as they have landed."""
        import torch

        if self._pinned is None:
            self._pinned = torch.empty(4096 * 8, dtype=torch.float64, pin_memory=True)
        assert n <= 8
        i = self._pinned_next
        self._pinned_next = (i + 1) % 4096
        return self._pinned[8 * i:8 * i + n]

    def aux_stream(self):
        """Side stream for the step's asynchronous drift telemetry (created on first use)."""
        import torch

        if self._aux is None:
            self._aux = torch.cuda.Stream(device=self.device)
            self.lib.wssr_set_aux_stream(self.handle, _vp(self._aux.cuda_stream))
        return self._aux

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.wssr_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def call(self, name, *args):
        import torch

        lib = self.lib
        stream = torch.cuda.current_stream(self.device).cuda_stream
        lib.wssr_set_stream(self.handle, _vp(stream))
        rc = getattr(lib, name)(self.handle, *args)
        if rc != WSSR_OK:
            msg = lib.wssr_last_error(self.handle)
            msg = msg.decode() if msg else ""
            raise _STATUS.get(rc, errors.DeviceError)(msg or f"{name} failed with status {rc}")
        return rc

    def kernel_launches(self) -> int:
        return int(self.lib.wssr_kernel_launches(self.handle))

    def set_precision_guard(self, enabled: bool) -> None:
        self.lib.wssr_set_precision_guard(self.handle, int(bool(enabled)))

    def precision_fallbacks(self) -> int:
        return int(self.lib.wssr_precision_fallbacks(self.handle))

    def set_timing(self, enabled: bool) -> None:
        self.lib.wssr_set_timing(self.handle, int(bool(enabled)))

    def phase_stats(self, phase: int) -> dict:
        ms, n, fl, by = _dbl(), _i64(), _dbl(), _dbl()
        self.lib.wssr_phase_stats(self.handle, int(phase), ctypes.byref(ms), ctypes.byref(n),
                                  ctypes.byref(fl), ctypes.byref(by))
        return {"ms": ms.value, "launches": n.value, "flops": fl.value, "bytes": by.value}

    def dmma_peak_tflops(self) -> float:
        out = _dbl()
        self.call("wssr_dmma_peak_probe", ctypes.byref(out))
        return float(out.value)


def scale_table_len(n_params: int) -> int:
    """Doubles in the per-parameter scale table of the int8 tensor-core O-passes (4 per slot,
    one slot per parameter rounded up to 32; see csrc/ozaki.cu biased_digits)."""
    return 4 * ((int(n_params) + 31) // 32 * 32)


_contexts: dict = {}
_thread_ctx = threading.local()


def set_thread_context(ctx) -> None:
    """Route this host thread's drop-in calls to `ctx` (None: the per-device default)."""
    _thread_ctx.ctx = ctx


def context(device=None) -> Context:
    import torch

    override = getattr(_thread_ctx, "ctx", None)
    if override is not None:
        return override
    if not torch.cuda.is_available():
        raise errors.DeviceError("the WSSR drop-in needs a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else int(device)
    ctx = _contexts.get(dev)
    if ctx is None:
        ctx = Context(dev)
        _contexts[dev] = ctx
    return ctx


def ptr(t) -> _vp:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return _vp(0)
    return _vp(t.data_ptr())
