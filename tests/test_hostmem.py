"""hostmem.pinned_empty: the page-locked host buffers of the e2e path."""
import gc

import numpy as np
import pytest
import torch

from paper_2508_12615_b200 import hostmem


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only contract")
def test_pinned_empty_needs_cuda():
    with pytest.raises(RuntimeError):
        hostmem.pinned_empty((4,))


@pytest.mark.gpu
def test_pinned_empty_roundtrip_and_release():
    """Zero-filled, reported pinned, async copies both ways are exact, and the
    registration is dropped (cudaHostUnregister) when the buffer is freed."""
    n = 3 * 1024 * 1024 + 5  # not a page multiple
    h = hostmem.pinned_empty((n,))
    assert h.is_pinned() and h.dtype == torch.float32 and h.shape == (n,)
    assert float(h.abs().sum()) == 0.0
    src = torch.from_numpy(np.random.default_rng(0).standard_normal(n).astype(np.float32))
    h.copy_(src)
    d = torch.empty(n, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        d.copy_(h, non_blocking=True)
        d.mul_(2.0)
        h.copy_(d, non_blocking=True)
    s.synchronize()
    assert torch.equal(h, src * 2.0)
    released = []
    orig = hostmem._unregister

    def record(ptr):
        released.append(ptr)
        orig(ptr)

    hostmem._unregister = record
    try:
        t = hostmem.pinned_empty((1 << 20,))
        ptr = t.data_ptr()
        del t
        gc.collect()
    finally:
        hostmem._unregister = orig
    assert released == [ptr]  # unregistered when the buffer went away
