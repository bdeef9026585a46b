"""Execution backend selector (reference backend.py:35-73).

The reference dispatches numba chunk kernels to a loop or a thread pool and
accepts the kinds "sequential" / "parallel".  Here there is exactly one kind,
"b200": every operator enqueues hand-written sm_100a kernels from libb2md.so on
the current CUDA stream of ``device``.  There is no other backend and no CPU
fallback; asking for one is a ConfigError, like an unknown kind in the reference
(test_backend.py:25-30).
"""
from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

B200 = "b200"


@dataclass
class BackendSelector:
    kind: str = B200
    device: int = 0
    #: kept for signature compatibility with the reference; ignored
    worker_count: int = 1
    chunk_size: int = 256

    def __post_init__(self):
        if self.kind != B200:
            raise ConfigError(
                f"unknown backend kind {self.kind!r}; this package only runs on 'b200'")
        if int(self.device) < 0:
            raise ConfigError("device must be >= 0")
        self.device = int(self.device)

    def stream_ptr(self) -> int:
        """cudaStream_t of torch's current stream on the device, as an int."""
        import torch
        return int(torch.cuda.current_stream(self.device).cuda_stream)
