"""Multi-GPU plumbing for the time-slab decomposition.

One process per GPU.  Rank r owns frames ``slab_range(T, n, r)`` of every
volume.  ``torch.distributed`` only carries the 128-byte NCCL unique id from
rank 0 to the others; the solve itself runs in libsfseg.so, which drives NCCL
(halo send/recv with ranks +-1 and an fp64 allreduce of the norm partials)
on the caller's CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import torch

from . import (DistC, Gauss, Shape, _alloc_bytes, _alloc_ws, _check, _options, _ptr, _require, _stream, _weights,
               lib, ACT_IDENTITY)


def slab_range(T: int, n: int, r: int) -> Tuple[int, int]:
    """Frames [t0, t1) of slab r of n (uneven when n does not divide T; same rule as the C library)."""
    if not (0 <= r < n):
        raise ValueError("rank out of range")
    return (T * r) // n, (T * (r + 1)) // n


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """NCCL unique id created on rank 0 (sfseg_get_unique_id) and broadcast to all ranks."""
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        raw = (C.c_uint8 * 128)()
        _check(lib().sfseg_get_unique_id(raw), "sfseg_get_unique_id")
        buf = torch.tensor(list(bytes(raw)), dtype=torch.uint8)
    if not dist.is_initialized():   # one process: nothing to broadcast
        return bytes(buf.tolist())
    backend = dist.get_backend(group)
    dev_buf = buf.cuda() if backend == "nccl" else buf
    dist.broadcast(dev_buf, src=0, group=group)
    return bytes(dev_buf.cpu().tolist())


def slab_launch_ranges(T: int, radius_t: int, has_lo: bool, has_hi: bool):
    """The spatial-pass launches of one iteration of the overlapped time-slab schedule
    (sfseg_slab_launch_ranges, host only): ([(first frame, count), ...] in launch order,
    number of boundary ranges launched before the halo exchange)."""
    buf = (C.c_int32 * 6)()
    n, nb = C.c_int32(0), C.c_int32(0)
    _check(lib().sfseg_slab_launch_ranges(int(T), int(radius_t), int(bool(has_lo)), int(bool(has_hi)), buf,
                                          C.byref(n), C.byref(nb)), "sfseg_slab_launch_ranges")
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)], nb.value


class Comm:
    """sfseg_comm (NCCL communicator created from a broadcast unique id)."""

    def __init__(self, nranks: int, rank: int, device: int, uid: bytes):
        self.nranks, self.rank, self.device = nranks, rank, device
        self._h = C.c_void_p()
        raw = (C.c_uint8 * 128)(*uid)
        _check(lib().sfseg_comm_create(raw, nranks, rank, device, C.byref(self._h)), "sfseg_comm_create")

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def close(self) -> None:
        if self._h:
            _check(lib().sfseg_comm_destroy(self._h), "sfseg_comm_destroy")
            self._h = C.c_void_p()


class SlabSolver:
    """One rank of a time-slab sharded solve (ch / x are this rank's local slab)."""

    def __init__(self, comm: Comm, local_shape, T_global: int, t_offset: int, C_: int, gauss: Gauss, K: int,
                 device="cuda", want_tape: bool = False, serial: bool = False, algo: int = 0):
        self.comm, self.shape = comm, tuple(int(v) for v in local_shape)
        # overlapped schedule (halo exchange under the interior frames, lagged allreduce) unless serial
        self.algo, self.serial = int(algo), bool(serial)
        self.profiler = None   # optional sf.Profiler (per-pass event timing, benchmark instrumentation)
        self.C, self.gauss, self.K = int(C_), gauss, int(K)
        self.dist = DistC(comm.handle, int(T_global), int(t_offset))
        n = C.c_size_t(0)
        tb = C.c_size_t(0)
        _check(lib().sfseg_workspace_bytes(Shape(*self.shape), self.C, gauss.c(), self.K, int(want_tape),
                                           C.byref(self.dist), C.byref(n), C.byref(tb)), "sfseg_workspace_bytes(dist)")
        self.tape = _alloc_bytes(tb.value, device) if want_tape else None
        self.ws_bytes = n.value
        self.ws = _alloc_ws(n.value, device)
        self.device = self.ws.device
        self.stats = torch.zeros((self.shape[0], self.K, 3), dtype=torch.float64, device=device)

    def forward(self, ch: torch.Tensor, w, b: float = 0.0, act: int = ACT_IDENTITY,
                x_out: Optional[torch.Tensor] = None, check: bool = True, stream=None) -> torch.Tensor:
        B, T, H, W = self.shape
        _require(ch, "ch", 5, shape=(B, self.C, T, H, W), device=self.device)
        if x_out is None:
            x_out = torch.empty(self.shape, dtype=torch.float32, device=self.device)
        _require(x_out, "x_out", 4, shape=self.shape, device=self.device)
        opt = _options(self.algo, self.profiler, slab_schedule=1 if self.serial else 0)
        _check(lib().sfseg_power_iterate_ex(
            _ptr(ch), self.C, _weights(w, self.C), float(b), int(act), Shape(*self.shape), self.gauss.c(), self.K,
            None, _ptr(x_out), None, _ptr(self.stats), 0, _ptr(self.tape), _ptr(self.ws), self.ws_bytes,
            C.byref(self.dist), C.byref(opt), _stream(stream)), "sfseg_power_iterate(dist)")
        if check:
            self.sync(stream)
        return x_out

    def backward(self, ch: torch.Tensor, w, dL_dx: torch.Tensor, b: float = 0.0, act: int = ACT_IDENTITY,
                 stream=None):
        """Time-slab backward on this rank's tape (sfseg_power_iterate_backward with the sfseg_dist):
        returns the GLOBAL (dw, db) -- the ranks allreduce them."""
        if self.tape is None:
            raise RuntimeError("SlabSolver was built without want_tape")
        B, T, H, W = self.shape
        _require(ch, "ch", 5, shape=(B, self.C, T, H, W), device=self.device)
        _require(dL_dx, "dL_dx", 4, shape=self.shape, device=self.device)
        dw = (C.c_double * self.C)()
        db = C.c_double(0.0)
        _check(lib().sfseg_power_iterate_backward(
            _ptr(ch), self.C, _weights(w, self.C), float(b), int(act), Shape(*self.shape), self.gauss.c(), self.K,
            None, _ptr(self.tape), _ptr(dL_dx), dw, C.byref(db), _ptr(self.ws), self.ws_bytes, C.byref(self.dist),
            _stream(stream)), "sfseg_power_iterate_backward(dist)")
        return [dw[i] for i in range(self.C)], db.value

    def sync(self, stream=None) -> None:
        _check(lib().sfseg_sync_status(_ptr(self.ws), _stream(stream)), "sfseg_power_iterate(dist, device)")
