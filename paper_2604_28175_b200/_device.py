"""Device plumbing for the host mirror: torch owns device memory and streams,
the CUDA library (``_strait.so``) does the arithmetic.  No CPU fallback."""
from __future__ import annotations

import numpy as np
import torch

from ._abi import StraitUnavailable, check, lib


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise StraitUnavailable("no CUDA device: the Strait B200 path has no CPU fallback")
    lib()  # fail loudly if the extension is missing
    return torch.device("cuda", torch.cuda.current_device())


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def dev(array, dtype=torch.float64) -> torch.Tensor:
    """Host array-like -> contiguous device tensor."""
    device = require_cuda()
    if isinstance(array, torch.Tensor):
        return array.to(device=device, dtype=dtype).contiguous()
    a = np.ascontiguousarray(array)
    if not a.flags.writeable:  # torch.from_numpy needs a writable buffer
        a = a.copy()
    return torch.from_numpy(a).to(device=device, dtype=dtype).contiguous()


def empty(shape, dtype=torch.float64) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=require_cuda())


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


__all__ = ["require_cuda", "stream_handle", "dev", "empty", "ptr", "host", "check", "lib"]
