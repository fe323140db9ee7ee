"""Device allocations of the pipeline, with an optional self-check mode.

compute-sanitizer is not available on the GPU pool, so the library's memory
discipline is checked by the allocator instead (``checking()``):

* every buffer the host hands to a kernel -- outputs and workspaces -- is
  poisoned before the call (0xFF bytes: NaN for floats, -1 for integers), so
  a kernel that reads a byte it never wrote propagates NaN / -1 into results
  that the test then compares bit for bit with an unpoisoned run
  (initcheck's question);
* each buffer sits between two 4 KiB guard regions filled with a canary;
  ``verify()`` (after a run) raises if any canary changed -- a kernel wrote
  outside the buffer it was given (memcheck's question for writes).

Off by default: plain ``torch.empty``.
"""

from __future__ import annotations

import contextlib

import torch

GUARD = 4096  # bytes on each side; keeps the 256-B alignment of the buffer
CANARY = 0xA5
POISON = 0xFF

_state = {"on": False, "live": []}


def empty(shape, dtype, device) -> torch.Tensor:
    if not _state["on"]:
        return torch.empty(shape, dtype=dtype, device=device)
    shape = (shape,) if isinstance(shape, int) else tuple(shape)
    n = 1
    for d in shape:
        n *= int(d)
    nbytes = max(n, 1) * torch.empty((), dtype=dtype).element_size()
    raw = torch.full((nbytes + 2 * GUARD,), CANARY, dtype=torch.uint8, device=device)
    body = raw[GUARD:GUARD + nbytes]
    body.fill_(POISON)
    _state["live"].append(raw)
    return body.view(dtype)[:n].view(shape) if n else body.view(dtype)[:0]


def verify() -> int:
    """Raise if a guard region changed; returns the number of buffers checked."""
    torch.cuda.synchronize()
    live, _state["live"] = _state["live"], []
    for raw in live:
        lo, hi = raw[:GUARD], raw[-GUARD:]
        if not (bool((lo == CANARY).all()) and bool((hi == CANARY).all())):
            raise AssertionError(f"out-of-bounds write next to a {raw.numel() - 2 * GUARD}-byte "
                                 "device buffer")
    return len(live)


@contextlib.contextmanager
def checking():
    """Poison + guard every pipeline allocation inside the block."""
    prev = _state["on"]
    _state["on"] = True
    try:
        yield
    finally:
        _state["on"] = prev
