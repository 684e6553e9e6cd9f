"""Device plumbing for the host layer: torch owns device memory and streams.

All compute goes through libopcfe (the C ABI); torch is used only to allocate
buffers, move bytes between host and device, and supply the current CUDA stream.
"""

from __future__ import annotations

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
            t = torch.from_numpy(np.ascontiguousarray(arr))
            self.dev = t.to("cuda", non_blocking=False)
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
            return t.cpu().numpy()
        return t


def to_host_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()
