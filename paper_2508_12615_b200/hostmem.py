"""Pinned host buffers for the host<->device path (plumbing, not compute).

`pinned_empty(shape)` returns a CPU float32 tensor whose pages were first
touched by the calling thread and then page-locked in place with
`cudaHostRegister`. On the B200 leases of this pool a buffer from torch's
`pin_memory()` uploaded at 10-21 GB/s on some leases while a buffer pinned this
way uploaded at 53-54 GB/s on the same lease and process
(`tools/h2d_probe.py`, DESIGN.md §5 "End to end"), so the e2e leg of bench.py
and users streaming inputs every step use these. The registration lives as long
as the returned tensor's storage (it is undone when the storage is freed).
"""
from __future__ import annotations

import weakref

import numpy as np
import torch


def _unregister(ptr: int) -> None:
    try:
        torch.cuda.cudart().cudaHostUnregister(ptr)
    except Exception:  # interpreter shutdown
        pass


def pinned_empty(shape, dtype=np.float32) -> torch.Tensor:
    """A page-locked CPU tensor of `shape` (zero-filled: the fill is the
    first touch that places its pages on the calling thread's node)."""
    if not torch.cuda.is_available():
        raise RuntimeError("pinned host buffers need a CUDA device")
    a = np.empty(shape, dtype=dtype)
    a.fill(0)
    t = torch.from_numpy(a)
    nbytes = a.nbytes
    if nbytes:
        err = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
        if int(err) != 0:
            raise RuntimeError(f"cudaHostRegister failed: {err}")
        # the tensor keeps the array alive; numpy runs weakref callbacks before it
        # frees the data, so the pages are unregistered while still mapped
        weakref.finalize(a, _unregister, t.data_ptr())
    return t
