"""B200-native SFSeg / SFSeg++ power-iteration hot path (arxiv 2212.08058).

Thin Python binding over the C ABI of ``libsfseg.so`` (include/sfseg.h):
argument marshalling only -- every step of the path runs in the library's
sm_100a kernels.  PyTorch provides device memory and the current CUDA stream.
There is no CPU fallback: if the in-tree ``libsfseg.so`` is missing or fails
to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import torch

__all__ = [
    "SfsegError", "Gauss", "lib", "workspace_bytes", "combine_channels", "power_iterate",
    "power_iterate_backward", "threshold", "solve_host", "Solver", "Profiler", "AdamWState",
    "ACT_IDENTITY", "ACT_SIGMOID", "THR_PER_FRAME_MAX", "THR_GLOBAL_MAX", "THR_ABSOLUTE",
    "ALGO_AUTO", "ALGO_TWO_PASS", "ALGO_TWO_PASS_FP32",
]

ACT_IDENTITY, ACT_SIGMOID = 0, 1
THR_PER_FRAME_MAX, THR_GLOBAL_MAX, THR_ABSOLUTE = 0, 1, 2
STATUS = {0: "ok", 1: "invalid argument", 2: "shape", 3: "workspace", 4: "degenerate",
          5: "non-finite", 6: "cuda", 7: "nccl", 8: "unsupported"}

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsfseg.so")


class SfsegError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = f"{where}: sfseg status {status} ({STATUS.get(status, '?')})"
        if status == 6 and _lib is not None:
            try:
                msg += ": " + _lib.sfseg_last_cuda_error().decode()
            except Exception:  # pragma: no cover
                pass
        super().__init__(msg)
        self.status = status


class Shape(C.Structure):
    _fields_ = [("B", C.c_int64), ("T", C.c_int64), ("H", C.c_int64), ("W", C.c_int64)]


class GaussC(C.Structure):
    _fields_ = [("sigma_t", C.c_double), ("sigma_s", C.c_double),
                ("radius_t", C.c_int32), ("radius_s", C.c_int32)]


class DistC(C.Structure):
    _fields_ = [("comm", C.c_void_p), ("T_global", C.c_int64), ("t_offset", C.c_int64)]


class BinarizeC(C.Structure):
    _fields_ = [("n_cont", C.c_int32), ("kappa0", C.c_float), ("growth", C.c_float)]


class OptionsC(C.Structure):
    _fields_ = [("algo", C.c_int32), ("profiler", C.c_void_p), ("binarize", C.c_void_p),
                ("slab_schedule", C.c_int32)]


class AdamwC(C.Structure):
    _fields_ = [("lr", C.c_double), ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("weight_decay", C.c_double), ("amsgrad", C.c_int32)]


@dataclass(frozen=True)
class Gauss:
    sigma_t: float
    sigma_s: float
    radius_t: int = -1     # < 0 => ceil(3 sigma)
    radius_s: int = -1

    def c(self) -> GaussC:
        return GaussC(self.sigma_t, self.sigma_s, self.radius_t, self.radius_s)


_lib: Optional[C.CDLL] = None

_P = C.c_void_p
_SIGS = {
    "sfseg_status_string": (C.c_char_p, [C.c_int]),
    "sfseg_abi_version": (C.c_int32, []),
    "sfseg_last_cuda_error": (C.c_char_p, []),
    "sfseg_max_radii": (None, [_P, _P]),
    "sfseg_workspace_bytes": (C.c_int, [Shape, C.c_int32, GaussC, C.c_int32, C.c_int32, _P, _P, _P]),
    "sfseg_combine_channels": (C.c_int, [_P, C.c_int32, Shape, _P, C.c_float, C.c_int32, _P, _P]),
    "sfseg_power_iterate": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC, C.c_int32,
                                      _P, _P, _P, _P, C.c_int32, _P, _P, C.c_size_t, _P, _P]),
    "sfseg_power_iterate_ex": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC, C.c_int32,
                                         _P, _P, _P, _P, C.c_int32, _P, _P, C.c_size_t, _P, _P, _P]),
    "sfseg_power_iterate_backward": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC,
                                               C.c_int32, _P, _P, _P, _P, _P, _P, C.c_size_t, _P, _P]),
    "sfseg_power_iterate_backward_ex": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC,
                                                  C.c_int32, _P, _P, _P, _P, _P, _P, C.c_size_t, _P, _P, _P]),
    "sfseg_workspace_reset": (C.c_int, [_P, _P]),
    "sfseg_profiler_create": (C.c_int, [_P]),
    "sfseg_profiler_destroy": (C.c_int, [_P]),
    "sfseg_profiler_read": (C.c_int, [_P, _P, _P]),
    "sfseg_adamw_step": (C.c_int, [_P, _P, _P, C.c_int32, C.c_int64, _P, _P]),
    "sfseg_focal_dice_ws_bytes": (C.c_size_t, [Shape]),
    "sfseg_focal_dice": (C.c_int, [_P, _P, Shape, C.c_double, _P, _P, _P, C.c_size_t, _P]),
    "sfseg_threshold_ws_bytes": (C.c_size_t, [Shape]),
    "sfseg_threshold": (C.c_int, [_P, Shape, C.c_float, C.c_int32, _P, _P, C.c_size_t, _P]),
    "sfseg_sync_status": (C.c_int, [_P, _P]),
    "sfseg_solve_host": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC, C.c_int32,
                                   C.c_float, C.c_int32, _P, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "sfseg_forward_path": (C.c_int, [Shape, GaussC, C.c_int32, C.POINTER(C.c_int32)]),
    "sfseg_solve_host_batch": (C.c_int, [_P, C.c_int32, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC,
                                         C.c_int32, C.c_float, C.c_int32, _P, _P, _P, _P, _P, _P, C.c_size_t,
                                         _P, _P, _P]),
    "sfseg_workspace_bytes_online": (C.c_int, [Shape, C.c_int32, GaussC, C.c_int32, C.c_int32, _P]),
    "sfseg_power_iterate_online": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC, C.c_int32,
                                             C.c_int32, C.c_int32, _P, _P, C.c_size_t, _P]),
    "sfseg_workspace_bytes_full": (C.c_int, [Shape, C.c_int32, C.c_int32, GaussC, C.c_int32, _P]),
    "sfseg_power_iterate_full": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, _P, C.c_int32, _P, C.c_float,
                                           C.c_int32, C.c_double, C.c_double, Shape, GaussC, C.c_int32, _P, _P,
                                           _P, _P, _P, C.c_size_t, _P, _P]),
    "sfseg_slabs_workspace_bytes": (C.c_int, [Shape, C.c_int32, GaussC, C.c_int32, C.c_int32, _P]),
    "sfseg_power_iterate_slabs": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC, C.c_int32,
                                            C.c_int32, _P, _P, _P, C.c_int32, _P, _P, C.c_size_t, _P, _P]),
    "sfseg_slabs_tape_bytes": (C.c_int, [Shape, C.c_int32, GaussC, C.c_int32, C.c_int32, _P]),
    "sfseg_power_iterate_slabs_backward": (C.c_int, [_P, C.c_int32, _P, C.c_float, C.c_int32, Shape, GaussC,
                                                     C.c_int32, C.c_int32, _P, _P, _P, _P, _P, C.c_size_t, _P,
                                                     _P]),
    "sfseg_slabs_sync_status": (C.c_int, [Shape, C.c_int32, GaussC, C.c_int32, C.c_int32, _P, _P]),
    "sfseg_get_unique_id": (C.c_int, [_P]),
    "sfseg_comm_create": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P]),
    "sfseg_comm_destroy": (C.c_int, [_P]),
}


def lib() -> C.CDLL:
    """Load the in-tree libsfseg.so (raises if it is missing: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run `python -m paper_2212_08058_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(status: int, where: str) -> None:
    if status != 0:
        raise SfsegError(status, where)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def _shape(x: torch.Tensor) -> Shape:
    B, T, H, W = x.shape
    return Shape(B, T, H, W)


def _require(t: torch.Tensor, name: str, ndim: int, dtype=torch.float32, shape=None, device=None):
    """Every tensor handed to the library: CUDA, contiguous, the dtype, rank (and, when
    given, exact shape and device) the C call expects -- a wrong buffer would be read or
    written out of bounds by the kernels, so it is rejected here."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype or t.dim() != ndim or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor with {ndim} dims")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
    if device is not None and t.device != torch.device(device):
        raise ValueError(f"{name} is on {t.device}, expected {device}")


def _weights(w, Cn: int):
    w = [float(v) for v in (w.tolist() if hasattr(w, "tolist") else w)]
    if len(w) != Cn:
        raise ValueError("len(w) must equal the channel count")
    return (C.c_float * Cn)(*w)


class Profiler:
    """Caller-owned per-kernel event timing (sfseg_profiler): pass ``profiler=`` to a solver."""

    def __init__(self):
        self._h = C.c_void_p()
        _check(lib().sfseg_profiler_create(C.byref(self._h)), "sfseg_profiler_create")

    @property
    def handle(self):
        return self._h

    def read(self):
        """Sync the recorded events; returns {category: (total_ms, launches)} and resets."""
        ms = (C.c_double * 6)()
        n = (C.c_int64 * 6)()
        _check(lib().sfseg_profiler_read(self._h, ms, n), "sfseg_profiler_read")
        names = ("tpass", "spass", "once", "backward", "f3d", "reserved")
        return {names[i]: (ms[i], n[i]) for i in range(6)}

    def close(self):
        if self._h:
            _check(lib().sfseg_profiler_destroy(self._h), "sfseg_profiler_destroy")
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


ALGO_AUTO = 0
ALGO_TWO_PASS = 1
ALGO_TWO_PASS_FP32 = 3
ALGO_TWO_PASS_MMA_SYNC = 4
ALGO_TWO_PASS_TCGEN05 = 5
ALGO_TWO_PASS_MMA_F16 = 6

PATH_TWO_PASS_FP32 = 0
PATH_TWO_PASS_TC = 1
PATH_FUSED_3D = 2
PATH_TWO_PASS_TCGEN05 = 4
PATH_TWO_PASS_TC_F16 = 5


SLAB_OVERLAP, SLAB_SERIAL = 0, 1


def _options(algo: int = ALGO_AUTO, profiler: Optional[Profiler] = None, binarize=None,
             slab_schedule: int = SLAB_OVERLAP) -> OptionsC:
    """sfseg_options; binarize = (n_cont, kappa0, growth) or None (the BinarizeC is kept alive
    on the returned object for the duration of the call)."""
    o = OptionsC(int(algo), profiler.handle if profiler is not None else None, None, int(slab_schedule))
    if binarize is not None:
        o._bz = BinarizeC(int(binarize[0]), float(binarize[1]), float(binarize[2]))
        o.binarize = C.cast(C.pointer(o._bz), C.c_void_p)
    return o


def forward_path(shape, gauss, algo: int = ALGO_AUTO) -> tuple:
    """(path, compiled r_t, compiled r_s) of the single-GPU forward without a tape for this
    algo: path is one of PATH_* (host-side plan, no device work)."""
    info = (C.c_int32 * 3)()
    _check(lib().sfseg_forward_path(Shape(*shape), gauss.c(), int(algo), info), "sfseg_forward_path")
    return int(info[0]), int(info[1]), int(info[2])


def workspace_bytes(shape, C_: int, gauss: Gauss, K: int, want_tape: bool = False):
    ws, tape = C.c_size_t(0), C.c_size_t(0)
    _check(lib().sfseg_workspace_bytes(Shape(*shape), C_, gauss.c(), K, int(want_tape), None,
                                       C.byref(ws), C.byref(tape)), "sfseg_workspace_bytes")
    return ws.value, tape.value


def _alloc_bytes(n: int, device) -> torch.Tensor:
    # torch's caching allocator returns >= 512-byte aligned blocks
    return torch.empty(max(n, 256), dtype=torch.uint8, device=device)


def _alloc_ws(n: int, device) -> torch.Tensor:
    """A solve workspace: allocated, then its header (sticky error word, counters) zeroed
    once by sfseg_workspace_reset on the current stream."""
    ws = _alloc_bytes(n, device)
    with torch.cuda.device(ws.device):
        _check(lib().sfseg_workspace_reset(_ptr(ws), _stream()), "sfseg_workspace_reset")
    return ws


def combine_channels(ch: torch.Tensor, w, b: float = 0.0, act: int = ACT_IDENTITY, stream=None) -> torch.Tensor:
    """Eq.9: F = act(sum_c w_c ch_c + b).  ch [B][C][T][H][W]."""
    _require(ch, "ch", 5)
    B, Cn, T, H, W = ch.shape
    F = torch.empty((B, T, H, W), dtype=torch.float32, device=ch.device)
    _check(lib().sfseg_combine_channels(_ptr(ch), Cn, Shape(B, T, H, W), _weights(w, Cn), float(b), int(act),
                                        _ptr(F), _stream(stream)), "sfseg_combine_channels")
    return F


class Solver:
    """Holds the workspace (and optional tape) for one problem shape.

    ``forward`` runs sfseg_power_iterate_ex; ``backward`` runs
    sfseg_power_iterate_backward_ex on the tape of the last forward.  ``algo`` and
    ``profiler`` are this solver's sfseg_options (no process-global switch).
    """

    def __init__(self, shape, C_: int, gauss: Gauss, K: int, device="cuda", want_tape: bool = False,
                 algo: int = ALGO_AUTO, profiler: Optional[Profiler] = None, binarize=None):
        self.shape = tuple(int(v) for v in shape)
        self.C, self.gauss, self.K = int(C_), gauss, int(K)
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.want_tape = bool(want_tape)
        self.algo, self.profiler = int(algo), profiler
        self.binarize = None if binarize is None else (int(binarize[0]), float(binarize[1]), float(binarize[2]))
        ws, tape = workspace_bytes(self.shape, self.C, gauss, self.K, want_tape)
        thr = lib().sfseg_threshold_ws_bytes(Shape(*self.shape))
        self.ws_bytes = ws
        self.ws = _alloc_ws(ws + thr, self.device)
        self.thr_ws_bytes = thr
        self.tape = _alloc_bytes(tape, self.device) if want_tape else None
        self.stats = torch.zeros((self.shape[0], self.K, 3), dtype=torch.float64, device=self.device)

    def _opt(self):
        self._o = _options(self.algo, self.profiler, self.binarize)
        return C.byref(self._o)

    def forward(self, ch: torch.Tensor, w, b: float = 0.0, act: int = ACT_IDENTITY, x0=None,
                x_out: Optional[torch.Tensor] = None, want_rayleigh: bool = False, F_out=None,
                stream=None, check: bool = True) -> torch.Tensor:
        B, T, H, W = self.shape
        _require(ch, "ch", 5, shape=(B, self.C, T, H, W), device=self.device)
        if x0 is not None:
            _require(x0, "x0", 4, shape=self.shape, device=self.device)
        if F_out is not None:
            _require(F_out, "F_out", 4, shape=self.shape, device=self.device)
        if x_out is None:
            x_out = torch.empty(self.shape, dtype=torch.float32, device=self.device)
        _require(x_out, "x_out", 4, shape=self.shape, device=self.device)
        st = lib().sfseg_power_iterate_ex(
            _ptr(ch), self.C, _weights(w, self.C), float(b), int(act), Shape(*self.shape), self.gauss.c(), self.K,
            _ptr(x0), _ptr(x_out), _ptr(F_out), _ptr(self.stats), int(want_rayleigh), _ptr(self.tape),
            _ptr(self.ws), self.ws_bytes, None, self._opt(), _stream(stream))
        _check(st, "sfseg_power_iterate")
        if check:
            self.sync(stream)
        return x_out

    def sync(self, stream=None) -> None:
        _check(lib().sfseg_sync_status(_ptr(self.ws), _stream(stream)), "sfseg_power_iterate (device)")

    def backward(self, ch: torch.Tensor, w, dL_dx: torch.Tensor, b: float = 0.0, act: int = ACT_IDENTITY,
                 x0=None, stream=None):
        if self.tape is None:
            raise RuntimeError("Solver was built without want_tape")
        B, T, H, W = self.shape
        _require(ch, "ch", 5, shape=(B, self.C, T, H, W), device=self.device)
        _require(dL_dx, "dL_dx", 4, shape=self.shape, device=self.device)
        if x0 is not None:
            _require(x0, "x0", 4, shape=self.shape, device=self.device)
        dw = (C.c_double * self.C)()
        db = C.c_double(0.0)
        st = lib().sfseg_power_iterate_backward_ex(
            _ptr(ch), self.C, _weights(w, self.C), float(b), int(act), Shape(*self.shape), self.gauss.c(), self.K,
            _ptr(x0), _ptr(self.tape), _ptr(dL_dx), dw, C.byref(db), _ptr(self.ws), self.ws_bytes, None,
            self._opt(), _stream(stream))
        _check(st, "sfseg_power_iterate_backward")
        return [dw[i] for i in range(self.C)], db.value

    def threshold(self, x: torch.Tensor, tau: float, mode: int = THR_PER_FRAME_MAX,
                  mask: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        _require(x, "x", 4, shape=self.shape, device=self.device)
        if mask is None:
            mask = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
        _require(mask, "mask", 4, dtype=torch.uint8, shape=self.shape, device=self.device)
        thr_ws = self.ws.narrow(0, self.ws_bytes + (-self.ws_bytes) % 256, self.thr_ws_bytes) \
            if self.thr_ws_bytes else None
        _check(lib().sfseg_threshold(_ptr(x), _shape(x), float(tau), int(mode), _ptr(mask), _ptr(thr_ws),
                                     self.thr_ws_bytes, _stream(stream)), "sfseg_threshold")
        return mask


def power_iterate(ch: torch.Tensor, w, gauss: Gauss, K: int, b: float = 0.0, act: int = ACT_IDENTITY,
                  x0=None, want_rayleigh: bool = False, algo: int = ALGO_AUTO):
    """One-shot solve; returns (x_K [B][T][H][W], stats float64 [B][K][3])."""
    B, Cn, T, H, W = ch.shape
    s = Solver((B, T, H, W), Cn, gauss, K, device=ch.device, algo=algo)
    x = s.forward(ch, w, b, act, x0=x0, want_rayleigh=want_rayleigh)
    return x, s.stats.clone()


def power_iterate_backward(ch, w, gauss: Gauss, K: int, dL_dx, b: float = 0.0, act: int = ACT_IDENTITY, x0=None,
                           algo: int = ALGO_AUTO):
    B, Cn, T, H, W = ch.shape
    s = Solver((B, T, H, W), Cn, gauss, K, device=ch.device, want_tape=True, algo=algo)
    x = s.forward(ch, w, b, act, x0=x0)
    dw, db = s.backward(ch, w, dL_dx, b, act, x0=x0)
    return x, dw, db


def power_iterate_slabs(ch: torch.Tensor, w, gauss: Gauss, K: int, nslabs: int, b: float = 0.0,
                        act: int = ACT_IDENTITY, x0=None, want_rayleigh: bool = False, stream=None,
                        algo: int = ALGO_AUTO, want_tape: bool = False, slab_schedule: int = SLAB_OVERLAP):
    """Time-slab decomposition of the solve emulated on ONE GPU (sfseg_power_iterate_slabs):
    the per-rank phases of the multi-GPU path with in-process halo copies and reduction, in
    the overlapped schedule (halo copies and the norm reduction on a second stream) or the
    serial one (SLAB_SERIAL: same kernels, one stream).
    Returns (x, stats) or, with want_tape, (x, stats, tape) for power_iterate_slabs_backward."""
    _require(ch, "ch", 5)
    B, Cn, T, H, W = ch.shape
    shp, g = Shape(B, T, H, W), gauss.c()
    n = C.c_size_t(0)
    _check(lib().sfseg_slabs_workspace_bytes(shp, Cn, g, int(K), int(nslabs), C.byref(n)),
           "sfseg_slabs_workspace_bytes")
    ws = torch.zeros(max(n.value, 256), dtype=torch.uint8, device=ch.device)  # every slab header zeroed
    nsl = int(nslabs)
    tape = None
    if want_tape:
        tb = C.c_size_t(0)
        _check(lib().sfseg_slabs_tape_bytes(shp, Cn, g, int(K), nsl, C.byref(tb)), "sfseg_slabs_tape_bytes")
        tape = torch.zeros(max(tb.value, 256), dtype=torch.uint8, device=ch.device)  # padding bytes defined
    x = torch.empty((B, T, H, W), dtype=torch.float32, device=ch.device)
    stats = torch.zeros((B, int(K), 3), dtype=torch.float64, device=ch.device)
    if x0 is not None:
        _require(x0, "x0", 4, shape=(B, T, H, W), device=ch.device)
    _check(lib().sfseg_power_iterate_slabs(_ptr(ch), Cn, _weights(w, Cn), float(b), int(act), shp, g, int(K),
                                           nsl, _ptr(x0), _ptr(x), _ptr(stats), int(want_rayleigh), _ptr(tape),
                                           _ptr(ws), n.value, C.byref(_options(algo, slab_schedule=slab_schedule)),
                                           _stream(stream)),
           "sfseg_power_iterate_slabs")
    _check(lib().sfseg_slabs_sync_status(shp, Cn, g, int(K), nsl, _ptr(ws), _stream(stream)),
           "sfseg_power_iterate_slabs (device)")
    return (x, stats, tape) if want_tape else (x, stats)


def power_iterate_slabs_backward(ch: torch.Tensor, w, gauss: Gauss, K: int, nslabs: int, tape: torch.Tensor,
                                 dL_dx: torch.Tensor, b: float = 0.0, act: int = ACT_IDENTITY, stream=None,
                                 algo: int = ALGO_AUTO):
    """The time-slab backward emulated on ONE GPU (sfseg_power_iterate_slabs_backward) on the tape
    of power_iterate_slabs(want_tape=True).  Returns (dw, db)."""
    _require(ch, "ch", 5)
    B, Cn, T, H, W = ch.shape
    _require(dL_dx, "dL_dx", 4, shape=(B, T, H, W), device=ch.device)
    shp, g = Shape(B, T, H, W), gauss.c()
    n = C.c_size_t(0)
    _check(lib().sfseg_slabs_workspace_bytes(shp, Cn, g, int(K), int(nslabs), C.byref(n)),
           "sfseg_slabs_workspace_bytes")
    ws = torch.zeros(max(n.value, 256), dtype=torch.uint8, device=ch.device)
    dw = (C.c_double * Cn)()
    db = C.c_double(0.0)
    _check(lib().sfseg_power_iterate_slabs_backward(_ptr(ch), Cn, _weights(w, Cn), float(b), int(act), shp, g,
                                                    int(K), int(nslabs), _ptr(tape), _ptr(dL_dx), dw, C.byref(db),
                                                    _ptr(ws), n.value, C.byref(_options(algo)), _stream(stream)),
           "sfseg_power_iterate_slabs_backward")
    return [dw[i] for i in range(Cn)], db.value


def threshold(x: torch.Tensor, tau: float, mode: int = THR_PER_FRAME_MAX) -> torch.Tensor:
    _require(x, "x", 4)
    n = lib().sfseg_threshold_ws_bytes(_shape(x))
    ws = _alloc_bytes(n, x.device)
    mask = torch.empty(x.shape, dtype=torch.uint8, device=x.device)
    _check(lib().sfseg_threshold(_ptr(x), _shape(x), float(tau), int(mode), _ptr(mask), _ptr(ws), n,
                                 _stream()), "sfseg_threshold")
    return mask


def solve_host(ch_host: torch.Tensor, w, gauss: Gauss, K: int, tau: float, solver: Solver,
               d_ch: torch.Tensor, d_x: torch.Tensor, d_mask: torch.Tensor,
               x_out_host: Optional[torch.Tensor], mask_out_host: Optional[torch.Tensor],
               b: float = 0.0, act: int = ACT_IDENTITY, thr_mode: int = THR_PER_FRAME_MAX, stream=None):
    """End-to-end call over HOST buffers (H2D, solve, threshold, D2H, sync) via sfseg_solve_host."""
    B, Cn, T, H, W = ch_host.shape
    if ch_host.is_cuda or ch_host.dtype != torch.float32 or not ch_host.is_contiguous():
        raise ValueError("ch_host must be a contiguous float32 host tensor")
    if (B, T, H, W) != solver.shape or Cn != solver.C:
        raise ValueError("ch_host does not match the solver")
    _require(d_ch, "d_ch", 5, shape=ch_host.shape, device=solver.device)
    _require(d_x, "d_x", 4, shape=solver.shape, device=solver.device)
    _require(d_mask, "d_mask", 4, dtype=torch.uint8, shape=solver.shape, device=solver.device)
    for t, nm, dt in ((x_out_host, "x_out_host", torch.float32), (mask_out_host, "mask_out_host", torch.uint8)):
        if t is not None and (t.is_cuda or t.dtype != dt or tuple(t.shape) != solver.shape or not t.is_contiguous()):
            raise ValueError(f"{nm} must be a contiguous {dt} host tensor of shape {solver.shape}")
    _check(lib().sfseg_solve_host(
        C.c_void_p(ch_host.data_ptr()), Cn, _weights(w, Cn), float(b), int(act), Shape(B, T, H, W), gauss.c(),
        int(K), float(tau), int(thr_mode), _ptr(d_ch), _ptr(d_x), _ptr(d_mask),
        None if x_out_host is None else C.c_void_p(x_out_host.data_ptr()),
        None if mask_out_host is None else C.c_void_p(mask_out_host.data_ptr()),
        _ptr(solver.ws), solver.ws.numel(), _stream(stream)), "sfseg_solve_host")


class HostBatch:
    """End to end over HOST buffers through ONE library call (sfseg_solve_host_batch): the
    library pipelines H2D of volume i+1 and D2H of volume i-1 under the solve of volume i on
    the caller's streams.  Holds the two device slots and the copy streams."""

    def __init__(self, solver: "Solver"):
        self.solver = solver
        dev = solver.device
        B, T, H, W = solver.shape
        self.d_ch = torch.empty((2, B, solver.C, T, H, W), dtype=torch.float32, device=dev)
        self.d_x = torch.empty((2, B, T, H, W), dtype=torch.float32, device=dev)
        self.d_m = torch.empty((2, B, T, H, W), dtype=torch.uint8, device=dev)
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)

    def run(self, ch_hosts, w, tau: float, x_hosts=None, mask_hosts=None, b: float = 0.0, act: int = ACT_IDENTITY,
            thr_mode: int = THR_PER_FRAME_MAX, stream=None) -> None:
        s = self.solver
        B, T, H, W = s.shape
        n = len(ch_hosts)
        for t in ch_hosts:
            if t.is_cuda or t.dtype != torch.float32 or tuple(t.shape) != (B, s.C, T, H, W) or not t.is_contiguous():
                raise ValueError("ch_hosts must be contiguous float32 host tensors of the solver's shape")
        for arr, dt in ((x_hosts, torch.float32), (mask_hosts, torch.uint8)):
            if arr is not None:
                if len(arr) != n:
                    raise ValueError("one output per input volume")
                for t in arr:
                    if t.is_cuda or t.dtype != dt or tuple(t.shape) != s.shape or not t.is_contiguous():
                        raise ValueError(f"outputs must be contiguous {dt} host tensors of shape {s.shape}")
        chp = (C.c_void_p * n)(*[t.data_ptr() for t in ch_hosts])
        xp = None if x_hosts is None else (C.c_void_p * n)(*[t.data_ptr() for t in x_hosts])
        mp = None if mask_hosts is None else (C.c_void_p * n)(*[t.data_ptr() for t in mask_hosts])
        _check(lib().sfseg_solve_host_batch(
            chp, n, s.C, _weights(w, s.C), float(b), int(act), Shape(*s.shape), s.gauss.c(), s.K, float(tau),
            int(thr_mode), _ptr(self.d_ch), _ptr(self.d_x), _ptr(self.d_m), xp, mp, _ptr(s.ws), s.ws.numel(),
            _stream(stream), C.c_void_p(self.s_h2d.cuda_stream), C.c_void_p(self.s_d2h.cuda_stream)),
            "sfseg_solve_host_batch")


class HostStream:
    """End-to-end solves of a sequence of volumes held in (pinned) HOST memory,
    pipelined over three CUDA streams: the host->device copy of volume i+1 and
    the device->host copy of volume i-1 overlap the solve of volume i
    (sfseg_power_iterate + sfseg_threshold on the compute stream).  Two device
    slots (channels, x, mask) alternate; events order the reuse.  All compute
    is the library's kernels; the copies are cudaMemcpyAsync (torch)."""

    def __init__(self, solver: "Solver", device="cuda"):
        self.solver = solver
        self.device = torch.device(device)
        B, T, H, W = solver.shape
        self.slots = []
        for _ in range(2):
            self.slots.append({
                "ch": torch.empty((B, solver.C, T, H, W), dtype=torch.float32, device=self.device),
                "x": torch.empty((B, T, H, W), dtype=torch.float32, device=self.device),
                "m": torch.empty((B, T, H, W), dtype=torch.uint8, device=self.device),
                "ev_in": torch.cuda.Event(), "ev_cmp": torch.cuda.Event(), "ev_out": torch.cuda.Event(),
                "used": False,
            })
        self.s_h2d = torch.cuda.Stream(self.device)
        self.s_d2h = torch.cuda.Stream(self.device)

    def run(self, ch_hosts, w, tau: float, x_hosts, mask_hosts, b: float = 0.0, act: int = ACT_IDENTITY,
            thr_mode: int = THR_PER_FRAME_MAX) -> None:
        """Solve len(ch_hosts) volumes; results land in x_hosts[i] / mask_hosts[i].  Syncs, then
        reports the first device error of ANY volume (the error word is sticky)."""
        s_cmp = torch.cuda.current_stream(self.device)
        for i, chh in enumerate(ch_hosts):
            sl = self.slots[i % 2]
            if sl["used"]:
                self.s_h2d.wait_event(sl["ev_cmp"])   # the solve that read this slot's channels is done
            with torch.cuda.stream(self.s_h2d):
                sl["ch"].copy_(chh, non_blocking=True)
                sl["ev_in"].record(self.s_h2d)
            s_cmp.wait_event(sl["ev_in"])
            if sl["used"]:
                s_cmp.wait_event(sl["ev_out"])       # x / mask of this slot have been copied out
            self.solver.forward(sl["ch"], w, b, act, x_out=sl["x"], stream=s_cmp, check=False)
            self.solver.threshold(sl["x"], tau, thr_mode, mask=sl["m"], stream=s_cmp)
            sl["ev_cmp"].record(s_cmp)
            self.s_d2h.wait_event(sl["ev_cmp"])
            with torch.cuda.stream(self.s_d2h):
                if x_hosts is not None:
                    x_hosts[i].copy_(sl["x"], non_blocking=True)
                if mask_hosts is not None:
                    mask_hosts[i].copy_(sl["m"], non_blocking=True)
                sl["ev_out"].record(self.s_d2h)
            sl["used"] = True
        self.s_d2h.synchronize()
        self.solver.sync(s_cmp)


class FullSolver:
    """The full SFSeg / SFSeg++ operator (Eq.7 / Eq.10 with
    unary exponent p, pairwise map F and alpha) through sfseg_power_iterate_full."""

    def __init__(self, shape, Cs: int, Cf: int, gauss: Gauss, K: int, device="cuda", algo: int = ALGO_AUTO,
                 profiler: Optional[Profiler] = None):
        self.shape = tuple(int(v) for v in shape)
        self.Cs, self.Cf, self.gauss, self.K = int(Cs), int(Cf), gauss, int(K)
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.algo, self.profiler = int(algo), profiler
        n = C.c_size_t(0)
        _check(lib().sfseg_workspace_bytes_full(Shape(*self.shape), self.Cs, self.Cf, gauss.c(), self.K,
                                                C.byref(n)), "sfseg_workspace_bytes_full")
        self.ws_bytes = n.value
        self.ws = _alloc_ws(self.ws_bytes, self.device)
        self.stats = torch.zeros((self.shape[0], self.K, 3), dtype=torch.float64, device=self.device)

    def forward(self, s_ch: torch.Tensor, ws, f_ch: torch.Tensor, wf, p: float, alpha: float,
                bs: float = 0.0, act_s: int = ACT_IDENTITY, bf: float = 0.0, act_f: int = ACT_IDENTITY,
                x0=None, x_out: Optional[torch.Tensor] = None, binarize=None, stream=None,
                check: bool = True) -> torch.Tensor:
        """binarize = (n_cont, kappa0, growth): Alg.1 STEP 3 soft-binarisation (row f2)."""
        B, T, H, W = self.shape
        _require(s_ch, "s_ch", 5, shape=(B, self.Cs, T, H, W), device=self.device)
        _require(f_ch, "f_ch", 5, shape=(B, self.Cf, T, H, W), device=self.device)
        if x0 is not None:
            _require(x0, "x0", 4, shape=self.shape, device=self.device)
        if x_out is None:
            x_out = torch.empty(self.shape, dtype=torch.float32, device=self.device)
        _require(x_out, "x_out", 4, shape=self.shape, device=self.device)
        st = lib().sfseg_power_iterate_full(
            _ptr(s_ch), self.Cs, _weights(ws, self.Cs), float(bs), int(act_s),
            _ptr(f_ch), self.Cf, _weights(wf, self.Cf), float(bf), int(act_f), float(p), float(alpha),
            Shape(*self.shape), self.gauss.c(), self.K, _ptr(x0), _ptr(x_out), _ptr(self.stats),
            None if binarize is None else C.byref(BinarizeC(int(binarize[0]), float(binarize[1]),
                                                            float(binarize[2]))),
            _ptr(self.ws), self.ws_bytes, C.byref(_options(self.algo, self.profiler)), _stream(stream))
        _check(st, "sfseg_power_iterate_full")
        if check:
            self.sync(stream)
        return x_out

    def sync(self, stream=None) -> None:
        _check(lib().sfseg_sync_status(_ptr(self.ws), _stream(stream)), "sfseg_power_iterate_full (device)")


def power_iterate_online(ch: torch.Tensor, w, gauss: Gauss, K: int, q: int, stride: int, b: float = 0.0,
                         act: int = ACT_IDENTITY, stream=None) -> torch.Tensor:
    """Online / sub-window mode via sfseg_power_iterate_online."""
    _require(ch, "ch", 5)
    B, Cn, T, H, W = ch.shape
    shp = Shape(B, T, H, W)
    n = C.c_size_t(0)
    _check(lib().sfseg_workspace_bytes_online(shp, Cn, gauss.c(), int(K), int(q), C.byref(n)),
           "sfseg_workspace_bytes_online")
    ws = _alloc_ws(n.value, ch.device)
    x = torch.empty((B, T, H, W), dtype=torch.float32, device=ch.device)
    _check(lib().sfseg_power_iterate_online(_ptr(ch), Cn, _weights(w, Cn), float(b), int(act), shp, gauss.c(),
                                            int(K), int(q), int(stride), _ptr(x), _ptr(ws), n.value,
                                            _stream(stream)), "sfseg_power_iterate_online")
    _check(lib().sfseg_sync_status(_ptr(ws), _stream(stream)), "sfseg_power_iterate_online (device)")
    return x


class AdamWState:
    """Device state of sfseg_adamw_step (Eq.13 with AMSGrad) for n
    parameters: the parameters and the moments [m | v | v_max] live in device memory and are
    updated by the library's kernel; this class only holds the buffers and the step count."""

    def __init__(self, params, lr: float, betas=(0.9, 0.999), eps: float = 1e-8, weight_decay: float = 0.0,
                 amsgrad: bool = True, device="cuda"):
        self.w = torch.tensor([float(v) for v in params], dtype=torch.float64, device=device)
        self.state = torch.zeros(3 * self.w.numel(), dtype=torch.float64, device=device)
        self.hp = AdamwC(float(lr), float(betas[0]), float(betas[1]), float(eps), float(weight_decay), int(amsgrad))
        self.t = 0

    def step(self, grad: torch.Tensor, stream=None) -> None:
        _require(grad, "grad", 1, dtype=torch.float64, shape=self.w.shape, device=self.w.device)
        self.t += 1
        _check(lib().sfseg_adamw_step(_ptr(self.w), _ptr(grad), _ptr(self.state), self.w.numel(), self.t,
                                      C.byref(self.hp), _stream(stream)), "sfseg_adamw_step")


class FocalDice:
    """Eq.12 Focal-Dice loss and dJ/dx on the device (sfseg_focal_dice) for one shape."""

    def __init__(self, shape, gamma: float = 0.75, device="cuda"):
        self.shape = tuple(int(v) for v in shape)
        self.gamma = float(gamma)
        self.device = torch.device(device)
        n = lib().sfseg_focal_dice_ws_bytes(Shape(*self.shape))
        self.ws_bytes = n
        self.ws = _alloc_bytes(n, self.device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)

    def __call__(self, x: torch.Tensor, mask: torch.Tensor, grad: Optional[torch.Tensor] = None, stream=None):
        """Returns (loss: 1-element float64 device tensor, dJ/dx)."""
        _require(x, "x", 4, shape=self.shape, device=x.device)
        _require(mask, "mask", 4, dtype=torch.uint8, shape=self.shape, device=x.device)
        if grad is None:
            grad = torch.empty(self.shape, dtype=torch.float32, device=x.device)
        _require(grad, "grad", 4, shape=self.shape, device=x.device)
        _check(lib().sfseg_focal_dice(_ptr(x), _ptr(mask), Shape(*self.shape), self.gamma, _ptr(self.loss),
                                      _ptr(grad), _ptr(self.ws), self.ws_bytes, _stream(stream)), "sfseg_focal_dice")
        return self.loss, grad


def train_weights(ch: torch.Tensor, mask: torch.Tensor, w0, b0: float, act: int, gauss: Gauss, K: int, steps: int,
                  lr: float, weight_decay: float = 0.0, loss: str = "mse", binarize=None, gamma: float = 0.75):
    """Learn the Eq.9 weights end to end: each step runs
    sfseg_power_iterate_ex with a tape (and, with ``binarize``, the soft-binarised
    iterations of Alg.1 STEP 3), the loss -- "focal_dice": Eq.12 on the device
    (sfseg_focal_dice); "mse": reading A13 against the unit-normalised mask (harness-side
    elementwise gradient) -- then sfseg_power_iterate_backward_ex for dL/dw, dL/db and
    sfseg_adamw_step.  Returns (w, b, losses)."""
    _require(ch, "ch", 5)
    B, Cn, T, H, W = ch.shape
    solver = Solver((B, T, H, W), Cn, gauss, K, device=ch.device, want_tape=True, binarize=binarize)
    if loss == "focal_dice":
        fd = FocalDice((B, T, H, W), gamma, device=ch.device)
        m8 = mask.to(torch.uint8).contiguous()
    else:
        m = mask.to(torch.float32)
        mn = torch.linalg.vector_norm(m.reshape(B, -1).double(), dim=1).float().clamp_min(1e-30)
        mh = m / mn.view(B, 1, 1, 1)
    opt = AdamWState(list(w0) + [float(b0)], lr, weight_decay=weight_decay, device=ch.device)
    losses = []
    for _ in range(steps):
        p = opt.w.cpu().tolist()
        w, b = [float(v) for v in p[:-1]], float(p[-1])
        x = solver.forward(ch, w, b, act)
        if loss == "focal_dice":
            Lt, g = fd(x, m8)
            losses.append(float(Lt.item()))
        else:
            d = x - mh
            losses.append(float((d.double() ** 2).mean()))
            g = ((2.0 / x.numel()) * d).contiguous()
        dw, db = solver.backward(ch, w, g, b, act)
        opt.step(torch.tensor(list(dw) + [db], dtype=torch.float64, device=ch.device))
    p = opt.w.cpu().tolist()
    return p[:-1], float(p[-1]), losses
