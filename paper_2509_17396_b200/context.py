"""Per-(thread, GPU) execution context: one epk_ctx bound to a CUDA stream."""
from __future__ import annotations

import ctypes as C
import threading

import torch

from . import _lib

_local = threading.local()


class Context:
    """Owns an epk_ctx (include/epk/epk.h).  Work is ordered on `stream`
    (default: torch's current stream on `device` at creation time)."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2509_17396_b200 needs a CUDA (sm_100a) device; none is visible")
        self.device = int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        handle = C.c_void_p()
        _lib.call("epk_ctx_create", self.device, C.c_void_p(self.stream.cuda_stream), C.byref(handle))
        self.handle = handle

    def set_stream(self, stream: torch.cuda.Stream) -> None:
        self.stream = stream
        _lib.call("epk_ctx_set_stream", self.handle, C.c_void_p(stream.cuda_stream))

    def reserve(self, nbytes: int) -> None:
        _lib.call("epk_ctx_reserve", self.handle, int(nbytes))

    def synchronize(self) -> None:
        _lib.call("epk_ctx_synchronize", self.handle)

    def poll_error(self) -> None:
        _lib.call("epk_ctx_poll_error", self.handle)

    @property
    def launches(self) -> int:
        return int(_lib.load().epk_ctx_launch_count(self.handle))

    def set_option(self, layer_group: int | None = None, overlap: bool | None = None,
                   pool_kernel: int | None = None) -> None:
        """epk_evict_step tuning: layers per group (0 = auto), compaction
        overlap, and the opt-in max-pool smoothing kernel (1 = off)."""
        if layer_group is not None:
            _lib.call("epk_ctx_set_option", self.handle, 1, int(layer_group))
        if overlap is not None:
            _lib.call("epk_ctx_set_option", self.handle, 2, int(bool(overlap)))
        if pool_kernel is not None:
            _lib.call("epk_ctx_set_option", self.handle, 4, int(pool_kernel))

    def profile(self, enable: bool) -> None:
        """Bracket every kernel launch with CUDA events (live per-kernel timing)."""
        _lib.call("epk_ctx_profile", self.handle, int(enable))

    def profile_records(self) -> list[tuple[str, float]]:
        """[(kernel name, ms)] recorded since profile(True); synchronises."""
        lib = _lib.load()
        n = int(lib.epk_ctx_profile_read(self.handle, -1, None, None))
        out = []
        name = C.create_string_buffer(32)
        ms = C.c_float()
        for i in range(max(n, 0)):
            lib.epk_ctx_profile_read(self.handle, i, name, C.byref(ms))
            out.append((name.value.decode(), float(ms.value)))
        return out

    def profile_timeline(self) -> list[tuple[str, float, float, int]]:
        """[(kernel, start ms from the first record, duration ms, side stream)]."""
        lib = _lib.load()
        n = int(lib.epk_ctx_profile_read(self.handle, -1, None, None))
        out = []
        name = C.create_string_buffer(32)
        t0, d, side = C.c_float(), C.c_float(), C.c_int32()
        for i in range(max(n, 0)):
            lib.epk_ctx_profile_timeline(self.handle, i, name, C.byref(t0), C.byref(d), C.byref(side))
            out.append((name.value.decode(), float(t0.value), float(d.value), int(side.value)))
        return out

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.load().epk_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def default_context(device: int | None = None) -> Context:
    """The calling thread's context for `device` (created on first use),
    re-bound to torch's current stream."""
    if device is None:
        device = torch.cuda.current_device()
    ctxs = getattr(_local, "ctxs", None)
    if ctxs is None:
        ctxs = _local.ctxs = {}
    ctx = ctxs.get(device)
    cur = torch.cuda.current_stream(device)
    if ctx is None:
        ctx = ctxs[device] = Context(device, cur)
    elif ctx.stream.cuda_stream != cur.cuda_stream:
        ctx.set_stream(cur)
    return ctx


def ptr(t: torch.Tensor | None) -> C.c_void_p:
    return C.c_void_p(0 if t is None else t.data_ptr())
