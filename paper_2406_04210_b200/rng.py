"""Counter-based random streams on the device (reference rng.py:40-66).

Every number is addressed by ``(seed, stream, step, word)``: Philox4x64-10 keyed
``(seed, 0)`` at counter ``(block + 1, 0, stream, step)``, uniforms
``((raw >> 11) + 0.5) * 2**-53``, normals through the inverse normal CDF (Cephes
``ndtri`` in fp64).  Raw words and uniforms are bit-identical to the reference's;
normals agree to the last few ulp (device ``log``)."""
from __future__ import annotations

import numpy as np

from . import _lib

STREAM_THERMOSTAT = 0
STREAM_INIT_VELOCITIES = 1
_TWO64 = 1 << 64


def _words(seed, stream, step, count, word_offset, want, device=0):
    import torch
    if count < 0:
        raise ValueError("count must be non-negative")
    dev = torch.device("cuda", device)
    _lib.load()
    raw = torch.empty(count, dtype=torch.int64, device=dev) if want == "raw" else None
    uni = torch.empty(count, dtype=torch.float64, device=dev) if want == "uniform" else None
    nrm = torch.empty(count, dtype=torch.float64, device=dev) if want == "normal" else None
    ptr = lambda t: None if t is None else t.data_ptr()
    _lib.call("b2md_stream_words", int(seed) % _TWO64, int(stream) % _TWO64, int(step) % _TWO64,
              int(word_offset), int(count), ptr(raw), ptr(uni), ptr(nrm),
              int(torch.cuda.current_stream(dev).cuda_stream))
    out = raw if raw is not None else (uni if uni is not None else nrm)
    return out.cpu().numpy()


def raw_words(seed: int, stream: int, step: int, count: int):
    """First ``count`` raw 64-bit words of the (seed, stream, step) block."""
    return _words(seed, stream, step, count, 0, "raw").view(np.uint64)


def uniforms(seed: int, stream: int, step: int, count: int, word_offset: int = 0):
    """Open-interval (0, 1) uniforms from words [offset, offset + count)."""
    return _words(seed, stream, step, count, word_offset, "uniform")


def normals(seed: int, stream: int, step: int, count: int, word_offset: int = 0):
    """Standard normals, one word per variate, via the inverse normal CDF."""
    return _words(seed, stream, step, count, word_offset, "normal")
