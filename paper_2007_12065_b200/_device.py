"""Device plumbing for the host layer: torch owns device memory and streams.

All compute goes through libopcfe (the C ABI); torch is used only to allocate
buffers, move bytes between host and device, and supply the current CUDA stream.
"""

from __future__ import annotations

import os
import threading
import warnings
import weakref

import numpy as np
import torch

from . import _lib


def require_cuda() -> None:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2007_12065_b200 runs only on a CUDA device (B200, sm_100a); "
            "there is no CPU fallback")
    _lib.lib()


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


def points_pitch(N: int) -> int:
    return (3 * N + 3) // 4 * 4


def fc_pitch(N: int) -> int:
    return (6 * (N - 1) + 3) // 4 * 4


def host_view(arr: np.ndarray) -> torch.Tensor:
    """torch view of a NumPy array that is only ever READ (a read-only caller array is
    fine: torch's non-writable warning does not apply)."""
    with warnings.catch_warnings():
        warnings.filterwarnings("ignore", message="The given NumPy array is not writable")
        return torch.from_numpy(arr)


class HostTransfer:
    """Large host <-> device copies for the NumPy drop-in API.

    D2H: a large result is returned as a NumPy view of a PINNED host block (torch's
    caching host allocator: freed blocks are reused once the array is garbage), so the
    DMA writes straight into the caller's array at the link rate (~54 GB/s on the B200
    box) -- a D2H into a fresh pageable array runs at ~2 GB/s (the driver's pageable
    path page-faults the destination as it copies) and even a staged copy is bound by
    first-touch page faults (~7 GB/s per thread).  Past `PINNED_OUT_MB` of such results
    still alive in callers' hands it falls back to a ring of pinned
    staging chunks DMA'd on a side stream while `SLOTS` threads copy finished chunks into
    a fresh NumPy array (numpy releases the GIL for the copy).
    H2D: an input that already lives in pinned memory (e.g. a previous call's result)
    is DMA'd directly; a pageable one goes through the staging ring (threads fill the
    slots).  Small arrays take the plain path.
    """

    CHUNK = int(os.environ.get("OPCFE_XFER_CHUNK_MB", "8")) << 20
    SLOTS = int(os.environ.get("OPCFE_XFER_SLOTS", "16"))
    MIN_BYTES = 4 << 20
    PINNED_OUT_MB = int(os.environ.get("OPCFE_PINNED_OUT_MB", "4096"))
    _inst = {}

    def __init__(self, device):
        from concurrent.futures import ThreadPoolExecutor
        self.device = device
        self.stage = [torch.empty(self.CHUNK, dtype=torch.uint8, pin_memory=True)
                      for _ in range(self.SLOTS)]
        self.stage_np = [t.numpy() for t in self.stage]
        self.stream = torch.cuda.Stream(device=device)
        self.events = [torch.cuda.Event() for _ in range(self.SLOTS)]
        self.pool = ThreadPoolExecutor(self.SLOTS)
        self.lock = threading.Lock()         # one transfer at a time per device (shared slots)
        self.out_lock = threading.Lock()
        self.out_bytes = 0                   # pinned result blocks alive in callers' arrays

    @classmethod
    def get(cls, device) -> "HostTransfer":
        key = torch.device(device).index or 0
        if key not in cls._inst:
            cls._inst[key] = cls(torch.device("cuda", key))
        return cls._inst[key]

    def to_numpy(self, t: torch.Tensor) -> np.ndarray:
        """Device tensor -> a new NumPy array (synchronous, like t.cpu().numpy())."""
        t = t.contiguous()
        nbytes = t.numel() * t.element_size()
        if nbytes < self.MIN_BYTES:
            return t.cpu().numpy()
        if self._pinned_room(nbytes):
            h = torch.empty(tuple(t.shape), dtype=t.dtype, pin_memory=True)
            h.copy_(t)                  # one DMA into the returned array's own memory
            arr = h.numpy()             # the array (its base) keeps the pinned block alive
            blk = 1 << (nbytes - 1).bit_length()        # the allocator's power-of-2 block
            with self.out_lock:
                self.out_bytes += blk
            weakref.finalize(arr.base, self._released, blk)
            return arr
        out = np.empty(tuple(t.shape), dtype=torch.empty((), dtype=t.dtype).numpy().dtype)
        with self.lock:
            self._d2h(t, out, nbytes)
        return out

    def _pinned_room(self, nbytes: int) -> bool:
        """Results handed out in pinned blocks and still alive stay under the budget."""
        with self.out_lock:
            return self.out_bytes + 2 * nbytes <= self.PINNED_OUT_MB << 20

    def _released(self, blk: int) -> None:
        with self.out_lock:
            self.out_bytes -= blk

    def _d2h(self, t, out, nbytes):
        src = t.reshape(-1).view(torch.uint8)
        dst = out.reshape(-1).view(np.uint8)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        futs = [None] * self.SLOTS
        for i, a in enumerate(range(0, nbytes, self.CHUNK)):
            b = min(nbytes, a + self.CHUNK)
            k = i % self.SLOTS
            if futs[k] is not None:
                futs[k].result()                      # the slot's previous chunk is copied out
            with torch.cuda.stream(self.stream):
                self.stage[k][:b - a].copy_(src[a:b], non_blocking=True)
                self.events[k].record(self.stream)
            ev, stg = self.events[k], self.stage_np[k]
            futs[k] = self.pool.submit(lambda ev=ev, stg=stg, a=a, b=b: (
                ev.synchronize(), np.copyto(dst[a:b], stg[:b - a])))
        for f in futs:
            if f is not None:
                f.result()

    def to_device(self, arr: np.ndarray, dtype=None) -> torch.Tensor:
        """A contiguous NumPy array -> a new device tensor (ordered before later work on
        the current stream)."""
        arr = np.ascontiguousarray(arr)
        t_host = host_view(arr)
        if arr.nbytes < self.MIN_BYTES:
            return t_host.to(self.device)
        if t_host.is_pinned():          # e.g. a result of a previous call: DMA directly
            out = t_host.to(self.device, non_blocking=True)
            torch.cuda.current_stream(self.device).synchronize()   # caller may reuse arr
            return out
        out = torch.empty(tuple(arr.shape), dtype=t_host.dtype, device=self.device)
        with self.lock:
            self._h2d(arr, out)
        return out

    def _h2d(self, arr, out):
        src = arr.reshape(-1).view(np.uint8)
        dst = out.reshape(-1).view(torch.uint8)
        nbytes = arr.nbytes
        chunks = list(range(0, nbytes, self.CHUNK))
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        fill = {}

        def stage_in(i):
            a = chunks[i]
            b = min(nbytes, a + self.CHUNK)
            k = i % self.SLOTS
            np.copyto(self.stage_np[k][:b - a], src[a:b])
            return a, b, k

        for i in range(min(self.SLOTS, len(chunks))):
            fill[i] = self.pool.submit(stage_in, i)
        for i in range(len(chunks)):
            a, b, k = fill.pop(i).result()
            with torch.cuda.stream(self.stream):
                dst[a:b].copy_(self.stage[k][:b - a], non_blocking=True)
                self.events[k].record(self.stream)
            if i + self.SLOTS < len(chunks):
                ev = self.events[k]
                fill[i + self.SLOTS] = self.pool.submit(
                    lambda ev=ev, j=i + self.SLOTS: (ev.synchronize(), stage_in(j))[1])
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        self.stream.synchronize()                      # staging slots reusable by the caller


class Staged:
    """An input array on the device plus how to hand results back to the caller."""

    def __init__(self, x, float_only=True):
        require_cuda()
        self.numpy = isinstance(x, np.ndarray) or not isinstance(x, torch.Tensor)
        if self.numpy:
            arr = np.asarray(x)
            if float_only and arr.dtype not in (np.float32, np.float64):
                arr = arr.astype(np.float64)
            self.out_dtype = torch.float64 if float_only else None
            self.dev = HostTransfer.get(torch.cuda.current_device()).to_device(arr)
        else:
            t = x
            if float_only and t.dtype not in (torch.float32, torch.float64):
                t = t.to(torch.float64)
            self.out_dtype = t.dtype if float_only else None
            self.dev = t.to("cuda").contiguous()
        self.is_f64 = self.dev.dtype == torch.float64

    def give(self, t: torch.Tensor):
        """Return a device result in the caller's world: NumPy callers get host arrays,
        floating point as float64 like the reference (np.asarray(opc, dtype=float64),
        smoothing.py:55); torch callers keep the device tensor."""
        if self.numpy:
            if self.out_dtype is not None and t.is_floating_point():
                t = t.to(self.out_dtype)
            return HostTransfer.get(t.device).to_numpy(t)
        return t


def to_host_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()
