"""Periodic box, version-tracked particle storage with a DEVICE compute side, and
the signal-driven step loop -- the B200 counterpart of reference core.py.

Reference semantics kept (core.py:25-279): ``SimBox`` (read-only fp64 edges and
inverse edges), ``minimum_image`` / ``wrap_position`` (host helpers, same
formulas), ``TrackedBuffer`` (two sides, ``version``, ``valid_on``,
``copy_count``, ``acquire_read/write/update``), ``ParticleState`` (the seven
per-particle buffers) and ``SignalEngine`` (integrate -> force -> finalize ->
sample).

What changes: the COMPUTE side is no longer a second numpy array but the packed
HBM layout described in include/b2md.h (double-single positions, float4 rows),
owned by PyTorch tensors.  Switching sides is therefore a format conversion done
by libb2md kernels (fp64 <-> packed), not ``np.copyto`` (core.py:131-137).  The
HOST side keeps the reference's dtypes and shapes, always in *logical* particle
order; the device may hold rows in Hilbert order, tracked by per-row ids.
"""
from __future__ import annotations

import ctypes

import weakref

import numpy as np

from . import _lib
from .errors import ConfigError

HOST = "host"
COMPUTE = "compute"
_SIDES = (HOST, COMPUTE)


# --------------------------------------------------------------------- box
class SimBox:
    """Orthorhombic periodic box (reference core.py:25-57)."""

    __slots__ = ("edge_lengths", "inverse_edges", "_cbox")

    def __init__(self, edge_lengths):
        edges = np.array(edge_lengths, dtype=np.float64).reshape(-1)
        if edges.shape != (3,):
            raise ValueError("edge_lengths must have exactly three components")
        if not np.all(np.isfinite(edges)) or np.any(edges <= 0.0):
            raise ValueError("edge_lengths must be finite and positive")
        edges.setflags(write=False)
        inv = 1.0 / edges
        inv.setflags(write=False)
        self.edge_lengths = edges
        self.inverse_edges = inv
        self._cbox = _lib.make_box(edges)

    @classmethod
    def cubic(cls, edge: float) -> "SimBox":
        return cls((edge, edge, edge))

    @property
    def volume(self) -> float:
        return float(np.prod(self.edge_lengths))

    def c_box(self):
        """ctypes view passed to libb2md (b2md_box)."""
        return ctypes.byref(self._cbox)

    def __repr__(self):
        lx, ly, lz = self.edge_lengths
        return f"SimBox(({lx:g}, {ly:g}, {lz:g}))"


def minimum_image(dr, box: SimBox):
    """``dr - L * rint(dr * (1/L))``, ties to even (reference core.py:60-69)."""
    dr = np.asarray(dr, dtype=np.float64)
    return dr - box.edge_lengths * np.rint(dr * box.inverse_edges)


def wrap_position(r, image, box: SimBox):
    """Wrap into [0, L), absorbing the shift into image counts (core.py:72-93)."""
    r = np.asarray(r, dtype=np.float64)
    image = np.asarray(image, dtype=np.int64)
    L = box.edge_lengths
    k = np.floor(r * box.inverse_edges)
    w = r - k * L
    low = w < 0.0
    w = np.where(low, w + L, w)
    k = np.where(low, k - 1.0, k)
    high = w >= L
    w = np.where(high, w - L, w)
    k = np.where(high, k + 1.0, k)
    return w, image + k.astype(np.int64)


# ------------------------------------------------------------ device side
def _torch():
    import torch
    return torch


def _require_cuda(device: int):
    torch = _torch()
    if not torch.cuda.is_available():
        raise _lib.B2mdError(
            "the COMPUTE side lives in B200 HBM; no CUDA device is available and this "
            "package has no CPU fallback")
    _lib.load()
    return torch.device("cuda", device)


class DeviceState:
    """Packed per-particle arrays in HBM (layout: include/b2md.h)."""

    ROW16 = ("pos_hi", "pos_lo", "vel", "force", "image")

    def __init__(self, n: int, device: int = 0, capacity: int | None = None):
        torch = _torch()
        self.device_index = int(device)
        self.device = _require_cuda(self.device_index)
        self.n = int(n)
        # rows are addressed up to the list pitch (n rounded up to a multiple of 32)
        self.capacity = (int(capacity if capacity is not None else n) + 31) // 32 * 32
        cap = self.capacity
        with torch.cuda.device(self.device):
            self.pos_hi = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
            self.pos_lo = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
            self.vel = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
            self.force = torch.zeros((cap, 4), dtype=torch.float32, device=self.device)
            self.image = torch.zeros((cap, 4), dtype=torch.int32, device=self.device)
            self.virial = torch.zeros((cap,), dtype=torch.float32, device=self.device)
            # masses default to 1 so that padded rows never divide by zero
            self.vel[:, 3] = 1.0
            self.status = torch.zeros(16, dtype=torch.int32, device=self.device)
        self.identity_order = True
        _lib.call("b2md_set_ids", self.pos_lo.data_ptr(), self.capacity, self.stream)
        self.reset_status()

    @property
    def stream(self) -> int:
        return int(_torch().cuda.current_stream(self.device).cuda_stream)

    def ids_ptr(self):
        """pos_lo pointer when rows are permuted, NULL for identity order."""
        return None if self.identity_order else self.pos_lo.data_ptr()

    def reset_status(self):
        _lib.call("b2md_status_reset", self.status.data_ptr(), self.stream)

    def read_status(self) -> _lib.Status:
        """Synchronising read of the 64-byte status block."""
        raw = self.status.cpu().numpy().tobytes()
        return _lib.Status.from_buffer_copy(raw)

    def particle_ids(self) -> np.ndarray:
        torch = _torch()
        out = torch.empty(self.n, dtype=torch.int32, device=self.device)
        _lib.call("b2md_get_ids", self.pos_lo.data_ptr(), self.n, out.data_ptr(), self.stream)
        return out.cpu().numpy()


class DeviceView:
    """What ``acquire_*(COMPUTE)`` hands out: the packed tensors holding this
    logical buffer.  Operators use ``.state``; ``.to_numpy()`` decodes it into
    the reference's host format (a fresh copy, for inspection)."""

    __slots__ = ("buffer", "state", "writable")

    def __init__(self, buffer, state, writable):
        self.buffer, self.state, self.writable = buffer, state, writable

    def to_numpy(self):
        return self.buffer._download()


#: bytes moved across the host<->device boundary by side switches (process-wide)
TRANSFER_BYTES = {"h2d": 0, "d2h": 0}

_KINDS = {
    # kind: (host dtype, trailing shape, pack entry, unpack entry, device tensor(s))
    "positions": (np.float64, (3,), "b2md_pack_positions", "b2md_unpack_positions", ("pos_hi", "pos_lo")),
    "velocities": (np.float64, (3,), "b2md_pack_vec3", "b2md_unpack_vec3", ("vel",)),
    "forces": (np.float64, (3,), "b2md_pack_vec3", "b2md_unpack_vec3", ("force",)),
    "masses": (np.float64, (), "b2md_pack_w_f64", "b2md_unpack_w_f64", ("vel",)),
    "per_particle_potential": (np.float64, (), "b2md_pack_w_f64", "b2md_unpack_w_f64", ("force",)),
    "species": (np.int32, (), "b2md_pack_w_i32", "b2md_unpack_w_i32", ("pos_hi",)),
    "images": (np.int64, (3,), "b2md_pack_images", "b2md_unpack_images", ("image",)),
    "virial": (np.float64, (), "b2md_pack_scalar_f32", "b2md_unpack_scalar_f32", ("virial",)),
}


def _host_array(values, copy: bool):
    """HOST-side storage of a buffer.  ``copy=False`` adopts the caller's array
    (zero-copy; e.g. page-locked memory the caller allocated once) when it already
    has the right layout; otherwise a private contiguous copy is made, as the
    reference does (core.py:110-112)."""
    arr = np.asarray(values)
    if not copy and isinstance(values, np.ndarray) and arr.flags.c_contiguous \
            and arr.flags.writeable and arr.flags.aligned:
        return arr
    return np.array(arr, order="C")


class LazyDefault:
    """HOST side of a buffer that still holds its default (all zeros / all ones): the numpy
    array is only materialised when somebody looks at it.  (Filling a million-row array the
    device never reads cost 2.3 ms of page faults per ParticleState.)"""

    __slots__ = ("shape", "dtype", "fill")

    def __init__(self, shape, dtype, fill):
        self.shape, self.dtype, self.fill = tuple(shape), np.dtype(dtype), fill

    def materialise(self):
        if self.fill == 0:
            return np.zeros(self.shape, dtype=self.dtype)
        return np.full(self.shape, self.fill, dtype=self.dtype)


class TrackedBuffer:
    """Double buffer with explicit ownership and a version counter
    (reference core.py:96-153), HOST = numpy, COMPUTE = packed HBM rows."""

    __slots__ = ("_host_data", "_lazy", "_owner", "kind", "version", "valid_on", "copy_count")

    @property
    def _host(self):
        if self._host_data is None:
            self._host_data = self._lazy.materialise()
        return self._host_data

    def __init__(self, array, owner=None, kind: str | None = None, copy: bool = True):
        if isinstance(array, LazyDefault):
            self._host_data, self._lazy = None, array
        else:
            self._host_data, self._lazy = _host_array(array, copy), None
        # weak: the state owns its buffers, not the other way round (a strong back reference
        # makes every ParticleState a reference cycle, and its HBM is then only returned by
        # the cycle collector -- 1 GB per abandoned Simulation at N = 1 M)
        self._owner = weakref.ref(owner) if owner is not None else None
        self.kind = kind
        self.version = 0
        # the device copy is materialised on first COMPUTE acquisition
        self.valid_on = HOST
        self.copy_count = 0

    @property
    def shape(self):
        return self._lazy.shape if self._host_data is None else self._host_data.shape

    @property
    def dtype(self):
        return self._lazy.dtype if self._host_data is None else self._host_data.dtype

    def _require_side(self, side):
        if side not in _SIDES:
            raise ValueError(f"unknown buffer side {side!r}")

    # -- conversions -------------------------------------------------------
    def _device(self) -> DeviceState:
        owner = self._owner() if self._owner is not None else None
        if owner is None or self.kind is None:
            raise _lib.B2mdError("this TrackedBuffer is not attached to a ParticleState")
        return owner.device_state()

    def _upload(self):
        torch = _torch()
        dev = self._device()
        _, _, pack, _, targets = _KINDS[self.kind]
        stage = torch.from_numpy(self._host).to(dev.device, non_blocking=True)
        TRANSFER_BYTES["h2d"] += self._host.nbytes
        ptrs = [getattr(dev, t).data_ptr() for t in targets]
        _lib.call(pack, stage.data_ptr(), dev.n, dev.ids_ptr(), *ptrs, dev.stream)

    def _download(self, into=None) -> np.ndarray:
        """Decode the device rows into the reference's host format.  With ``into``
        the result is copied straight into that array (a direct DMA when it is
        page-locked)."""
        torch = _torch()
        dev = self._device()
        dtype, _, _, unpack, targets = _KINDS[self.kind]
        tdtype = {np.float64: torch.float64, np.int32: torch.int32, np.int64: torch.int64}[dtype]
        stage = torch.empty(self._host.shape, dtype=tdtype, device=dev.device)
        ptrs = [getattr(dev, t).data_ptr() for t in targets]
        _lib.call(unpack, *ptrs, dev.n, dev.ids_ptr(), stage.data_ptr(), dev.stream)
        TRANSFER_BYTES["d2h"] += self._host.nbytes
        if into is not None:
            torch.from_numpy(into).copy_(stage)
            return into
        return stage.cpu().numpy()

    # -- acquisition -------------------------------------------------------
    def acquire_read(self, side):
        """Read access to ``side``, converting from the other side if stale."""
        self._require_side(side)
        if self.valid_on not in (side, "both"):
            if side == COMPUTE:
                self._upload()
            else:
                self._download(into=self._host)
            self.copy_count += 1
            self.valid_on = "both"
        if side == HOST:
            view = self._host.view()
            view.flags.writeable = False
            return view
        return DeviceView(self, self._device(), False)

    def acquire_write(self, side):
        """Write access to ``side``; whatever the other side holds is discarded."""
        self._require_side(side)
        self.version += 1
        self.valid_on = side
        if side == HOST:
            return self._host
        return DeviceView(self, self._device(), True)

    def acquire_update(self, side):
        """Read-modify-write: sync ``side`` if stale, then make it the only valid one."""
        self.acquire_read(side)
        return self.acquire_write(side)


# ---------------------------------------------------------- particle state
class ParticleState:
    """Structure-of-arrays particle data (reference core.py:156-226).

    HOST arrays: positions (n,3) f64 wrapped into [0,L); images (n,3) i64;
    velocities, forces (n,3) f64; masses (n,) f64 > 0; species (n,) i32;
    per_particle_potential (n,) f64; plus ``virial`` (n,) f64 (extension:
    per-particle half-share of sum r.f).
    """

    def __init__(self, positions, velocities=None, masses=None, images=None,
                 species=None, device: int = 0, copy: bool = True):
        """``copy=False`` adopts the caller's fp64 arrays as the HOST side (they are
        then updated in place by HOST acquisitions); the reference always copies."""
        pos = np.array(positions, dtype=np.float64) if copy else \
            np.asarray(positions, dtype=np.float64)
        if pos.ndim != 2 or pos.shape[1] != 3:
            raise ValueError("positions must have shape (n, 3)")
        n = pos.shape[0]
        if n < 1:
            raise ValueError("at least one particle is required")

        def take(arr, shape, dtype, fill):
            if arr is None:
                return LazyDefault(shape, dtype, fill)
            out = np.array(arr, dtype=dtype) if copy else np.asarray(arr, dtype=dtype)
            if out.shape != shape:
                raise ValueError(f"expected shape {shape}, got {out.shape}")
            return out

        # (defaults need no validation: a pass over a fresh zero-filled array only
        # faults its pages in -- 15 ms per million particles)
        masses_arr = take(masses, (n,), np.float64, 1.0)
        if masses is not None and np.any(masses_arr <= 0.0):
            raise ValueError("masses must be strictly positive")
        img = take(images, (n, 3), np.int64, 0)
        if images is not None and np.any(np.abs(img) > 2**31 - 1):
            raise ValueError("image counters must fit in int32 on the device")

        self._n = n
        self._device_index = int(device)
        self._dev: DeviceState | None = None
        # the arrays built above are already private (or deliberately adopted): no second copy
        self.positions = TrackedBuffer(pos, self, "positions", copy=False)
        self.images = TrackedBuffer(img, self, "images", copy=False)
        self.velocities = TrackedBuffer(take(velocities, (n, 3), np.float64, 0.0), self,
                                        "velocities", copy=False)
        self.forces = TrackedBuffer(LazyDefault((n, 3), np.float64, 0), self, "forces", copy=False)
        self.masses = TrackedBuffer(masses_arr, self, "masses", copy=False)
        self.species = TrackedBuffer(take(species, (n,), np.int32, 0), self, "species", copy=False)
        self.per_particle_potential = TrackedBuffer(LazyDefault((n,), np.float64, 0), self,
                                                    "per_particle_potential", copy=False)
        self.virial = TrackedBuffer(LazyDefault((n,), np.float64, 0), self, "virial", copy=False)
        # buffers that still hold their defaults match what DeviceState allocates
        # (zeros, unit masses): no upload is needed for them
        self._defaults = {"images": images is None, "forces": True, "masses": masses is None,
                          "species": species is None, "per_particle_potential": True,
                          "virial": True, "velocities": velocities is None}

    @property
    def n(self) -> int:
        return self._n

    def device_state(self) -> DeviceState:
        """Packed HBM arrays, allocated on first use (raises without CUDA)."""
        if self._dev is None:
            self._dev = DeviceState(self._n, self._device_index)
            # freshly allocated rows already equal the untouched default buffers
            for name, is_default in self._defaults.items():
                buf = getattr(self, name)
                if is_default and buf.version == 0 and buf.valid_on == HOST:
                    buf.valid_on = "both"
        return self._dev

    def buffers(self):
        """All per-particle buffers keyed by name (used for reordering)."""
        return {
            "positions": self.positions,
            "images": self.images,
            "velocities": self.velocities,
            "forces": self.forces,
            "masses": self.masses,
            "species": self.species,
            "per_particle_potential": self.per_particle_potential,
            "virial": self.virial,
        }

    def sync_to_compute(self):
        """Make every buffer valid on the device (one conversion per stale buffer)."""
        for buf in self.buffers().values():
            buf.acquire_read(COMPUTE)
        return self.device_state()

    def mark_compute_written(self, *names):
        """Operators call this after a kernel overwrote the named buffers."""
        for name in names:
            getattr(self, name).acquire_write(COMPUTE)

    def unwrapped_positions(self, box: SimBox, side=HOST):
        """pos + image * L in fp64 (reference core.py:216-219).  Always returns a
        host array; ``side`` only selects which copy must be current."""
        if side == COMPUTE:
            pos = self.positions.acquire_read(COMPUTE).to_numpy()
            img = self.images.acquire_read(COMPUTE).to_numpy()
        else:
            pos = self.positions.acquire_read(HOST)
            img = self.images.acquire_read(HOST)
        return pos + img * box.edge_lengths

    def particle_ids(self) -> np.ndarray:
        """Logical id of every physical device row (identity unless the engine
        reordered rows internally for locality)."""
        if self._dev is None:
            return np.arange(self._n, dtype=np.int32)
        return self._dev.particle_ids()

    def validate(self, box: SimBox):
        pos = self.positions.acquire_read(HOST)
        if np.any(pos < 0.0) or np.any(pos >= box.edge_lengths):
            raise ValueError("positions must be wrapped into [0, L) per axis")
        if np.any(self.masses.acquire_read(HOST) <= 0.0):
            raise ValueError("masses must be strictly positive")


# ------------------------------------------------------------- step loop
class SignalEngine:
    """Fires ``integrate``, ``force``, ``finalize`` every step and ``sample``
    whenever the post-step counter hits a multiple of ``sample_interval``
    (reference core.py:229-279)."""

    SIGNALS = ("integrate", "force", "finalize", "sample")
    MANDATORY = ("integrate", "force", "finalize")

    def __init__(self, sample_interval: int = 1, sample_initial: bool = False):
        if int(sample_interval) < 1:
            raise ConfigError("sample_interval must be >= 1")
        self.sample_interval = int(sample_interval)
        self.sample_initial = bool(sample_initial)
        self.step_count = 0
        self._slots = {name: [] for name in self.SIGNALS}
        self._initial_sample_done = False

    def connect(self, signal: str, slot):
        if signal not in self._slots:
            raise ConfigError(f"unknown signal {signal!r}")
        if not callable(slot):
            raise ConfigError("slot must be callable")
        self._slots[signal].append(slot)

    def emit(self, signal: str):
        for slot in self._slots[signal]:
            slot()

    def _check_ready(self, n_steps):
        if n_steps < 0:
            raise ValueError("n_steps must be non-negative")
        for name in self.MANDATORY:
            if not self._slots[name]:
                raise ConfigError(f"no slot attached to mandatory signal {name!r}")

    def emit_initial_sample(self):
        if self.sample_initial and not self._initial_sample_done:
            self._initial_sample_done = True
            self.emit("sample")

    def run_steps(self, n_steps: int):
        self._check_ready(n_steps)
        if n_steps == 0:
            return
        self.emit_initial_sample()
        for _ in range(n_steps):
            self.emit("integrate")
            self.emit("force")
            self.emit("finalize")
            self.step_count += 1
            if self.step_count % self.sample_interval == 0:
                self.emit("sample")
