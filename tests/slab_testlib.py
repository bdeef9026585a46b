"""Test double for the slab protocol: the `ops` interface of
paper_2406_04210_b200.decomp.SlabSimulation implemented with numpy + the CPU
oracle (fp64), so the decomposition protocol (migration, ghost selection, halo
exchange, collective rebuild decision, stride growth, reductions) can run over
gloo on CPU ranks.  TEST INFRASTRUCTURE ONLY -- the product path is CudaSlabOps."""
import numpy as np
import torch

from oracle import oracle as orc


class NumpySlabOps:
    device = torch.device("cpu")

    GATE_WORDS = (5, 12)

    def __init__(self, pos, vel, ids, edges, stride=32, advance=False):
        # one-launch steps (SlabSimulation._run_advance): the 16 status words of the
        # device block, a second position buffer with its own ghost rows
        self.can_advance = bool(advance)
        self.status = torch.zeros(16, dtype=torch.int32)
        self.gate_in = 5
        self.pos_alt = None
        self.ghost_pos_alt = np.zeros((0, 3))
        self.noop_launches = 0
        self.pos = np.array(pos, dtype=np.float64)
        self.vel = np.array(vel, dtype=np.float64)
        self.img = np.zeros(self.pos.shape, dtype=np.int64)
        self.ids = np.array(ids, dtype=np.int64)
        self.edges = np.array(edges, dtype=np.float64)
        self.n_own = self.pos.shape[0]
        self.ghost_pos = np.zeros((0, 3))
        self.stride = stride
        self.forces = np.zeros_like(self.pos)
        self.pe = np.zeros(self.n_own)
        self.virial = np.zeros(self.n_own)
        self.flag = 0
        self.kernel_launches = 0
        self._ghosts_dirty = False

    # -- plumbing ------------------------------------------------------------
    def attach(self, geo, lj, dt, skin):
        self.geo, self.lj, self.dt, self.skin = geo, lj, dt, skin
        self.r_list = lj.max_r_cut + skin
        self.table = lj.table()

    def scalar_pair(self, a, b):
        return torch.tensor([a, b], dtype=torch.int64)

    # records are fp64 here: pos(3) vel(3) image(3) id(1) / pos(3)
    def migrant_buffer(self, rows):
        return torch.zeros((rows, 10), dtype=torch.float64)

    def ghost_buffer(self, rows):
        return torch.zeros((rows, 3), dtype=torch.float64)

    def grow_stride(self, max_count):
        self.stride = max(self.stride + 1, ((int(max_count * 1.125) + 1) + 7) // 8 * 8)

    def _offset(self):
        """d = x - centre wrapped into [-L/2, L/2) exactly like k_slab_classify."""
        L = self.edges[0]
        d = self.pos[:self.n_own, 0] - self.geo.centre
        return d - L * np.floor(d / L + 0.5)

    # -- migration -------------------------------------------------------------
    def select_migrants(self):
        if self.geo.world == 1:
            self.sel = (np.zeros(0, int), np.zeros(0, int))
            return 0, 0
        half = 0.5 * self.geo.width
        d = self._offset()
        self.sel = (np.flatnonzero(d < -half), np.flatnonzero(d >= half))
        self.stay = np.flatnonzero((d >= -half) & (d < half))
        return len(self.sel[0]), len(self.sel[1])

    def pack_migrants(self):
        out = []
        for idx in self.sel:
            buf = np.zeros((len(idx), 10), dtype=np.float64)
            buf[:, 0:3], buf[:, 3:6] = self.pos[idx], self.vel[idx]
            buf[:, 6:9], buf[:, 9] = self.img[idx], self.ids[idx]
            out.append(torch.from_numpy(buf))
        return out

    def apply_migration(self, in_l, in_r):
        if self.geo.world == 1:
            return
        keep = self.stay
        pos, vel, img, ids = [self.pos[keep]], [self.vel[keep]], [self.img[keep]], [self.ids[keep]]
        for buf in (in_l, in_r):
            b = buf.numpy()
            pos.append(b[:, 0:3].copy())
            vel.append(b[:, 3:6].copy())
            img.append(b[:, 6:9].astype(np.int64))
            ids.append(b[:, 9].astype(np.int64))
        self.pos, self.vel = np.concatenate(pos), np.concatenate(vel)
        self.img, self.ids = np.concatenate(img), np.concatenate(ids)
        self.n_own = self.pos.shape[0]
        self.forces = np.zeros_like(self.pos)

    def reorder_owned(self):
        perm, _ = orc.hilbert_permutation(self.pos, self.edges, self.r_list)
        self.pos, self.vel = self.pos[perm], self.vel[perm]
        self.img, self.ids, self.forces = self.img[perm], self.ids[perm], self.forces[perm]

    # -- ghosts -----------------------------------------------------------------
    def select_ghosts(self, r_ghost):
        if self.geo.world == 1:
            self.sel = (np.zeros(0, int), np.zeros(0, int))
            return 0, 0
        half = 0.5 * self.geo.width
        d = self._offset()
        self.sel = (np.flatnonzero(d < -half + r_ghost), np.flatnonzero(d >= half - r_ghost))
        return len(self.sel[0]), len(self.sel[1])

    def pack_ghost_records(self):
        return [torch.from_numpy(self.pos[idx].copy()) for idx in self.sel]

    def set_ghosts(self, in_l, in_r):
        parts = [in_l.numpy().copy(), in_r.numpy().copy()]
        self.ghost_counts = (len(parts[0]), len(parts[1]))
        self.ghost_pos = np.concatenate(parts)
        self.ghost_recv = [torch.zeros((c, 3), dtype=torch.float64) for c in self.ghost_counts]
        self._ghosts_dirty = False

    def pack_ghost_positions(self):
        return [torch.from_numpy(self.pos[idx].copy()) for idx in self.sel]

    def ghost_position_views(self):
        self._ghosts_dirty = True
        return self.ghost_recv[0], self.ghost_recv[1]

    def _all_pos(self):
        if self._ghosts_dirty:
            self.ghost_pos = np.concatenate([t.numpy() for t in self.ghost_recv])
            self._ghosts_dirty = False
        return np.concatenate([self.pos, self.ghost_pos]) if len(self.ghost_pos) else self.pos

    # -- hot path ------------------------------------------------------------------
    def build_list(self):
        allpos = self._all_pos()
        grid = orc.bin_particles(allpos, self.edges, self.r_list)
        nl = orc.build_neighbor_list(allpos, np.zeros(allpos.shape, np.int64), grid,
                                     self.r_list, self.stride, r_cut=self.lj.max_r_cut)
        over = bool(nl.row_overflow[:self.n_own].any())
        # rows of ghost particles are never used
        nl.counts[self.n_own:] = 0
        nl.overflow = False
        self.nlist = nl
        self.at_build = self.pos + self.img * self.edges
        self.flag = 0
        self.status.zero_()
        # true wanted length is not exposed by the oracle: on overflow ask for double
        return over, (2 * self.stride if over else int(nl.counts[:self.n_own].max()))

    def integrate(self, fused):
        if fused:
            self.vel = orc.vv_finalize(self.vel, self.forces, np.ones(self.n_own), self.dt)
        self.pos, self.img, self.vel = orc.vv_integrate(
            self.pos, self.img, self.vel, self.forces, np.ones(self.n_own), self.edges, self.dt)
        disp = (self.pos + self.img * self.edges) - self.at_build
        half = 0.5 * self.skin
        self.flag = int(np.max((disp * disp).sum(axis=1)) > half * half)
        if self.flag:
            self.status[5] = 1

    def rebuild_flag(self):
        return torch.tensor([self.flag], dtype=torch.int64)

    def force(self, thermo):
        allpos = self._all_pos()
        f, pe, w = orc.forces_truncated(allpos, self.edges, self.table, self.nlist)
        self.forces, self.pe, self.virial = f[:self.n_own], pe[:self.n_own], w[:self.n_own]

    # -- one-launch steps: same contract as CudaSlabOps -----------------------------
    @property
    def gate_out(self):
        return self.GATE_WORDS[1] if self.gate_in == self.GATE_WORDS[0] else self.GATE_WORDS[0]

    def gate_word_in(self):
        return self.status[self.gate_in:self.gate_in + 1]

    def gate_word_out(self):
        return self.status[self.gate_out:self.gate_out + 1]

    def gate_toggle(self):
        self.gate_in = self.gate_out

    def gate_reset_to_integrate(self):
        self.gate_in = self.GATE_WORDS[0]

    def advance(self):
        """force(s) + finalize(s) + integrate(s+1) + displacement check; gated."""
        self.kernel_launches += 1
        if int(self.status[self.gate_in]):
            self.status[self.gate_out] = 1          # hand the flag on, do nothing
            self.noop_launches += 1
            if self.pos_alt is None or self.pos_alt.shape != self.pos.shape:
                self.pos_alt = np.full_like(self.pos, np.nan)     # never-written buffer
            return
        self.force(thermo=False)
        ones = np.ones(self.n_own)
        vel = orc.vv_finalize(self.vel, self.forces, ones, self.dt)
        self.pos_alt, self.img, self.vel = orc.vv_integrate(
            self.pos, self.img, vel, self.forces, ones, self.edges, self.dt)
        disp = (self.pos_alt + self.img * self.edges) - self.at_build
        half = 0.5 * self.skin
        if np.max((disp * disp).sum(axis=1)) > half * half:
            self.status[self.gate_out] = 1

    def swap_positions(self):
        self._all_pos()                             # received ghosts belong to this buffer
        self.pos, self.pos_alt = self.pos_alt, self.pos
        self.ghost_pos, self.ghost_pos_alt = self.ghost_pos_alt, self.ghost_pos

    def snapshot_status(self):
        self._snap = self.status.clone()
        return self.gate_in

    def snapshot_gate_in(self, word):
        return int(self._snap[word]) != 0

    def read_gate_in(self):
        return int(self.status[self.gate_in]) != 0

    def finalize(self):
        self.vel = orc.vv_finalize(self.vel, self.forces, np.ones(self.n_own), self.dt)

    def thermo_sums(self):
        t = orc.thermo(self.vel, np.ones(self.n_own), self.pe, self.virial)
        return torch.tensor([t["pe"], t["ke"], *t["momentum"], t["virial"], t["mass"],
                             float(self.n_own)], dtype=torch.float64)

    def owned_state(self):
        return self.ids.copy(), self.pos.copy(), self.vel.copy()
