"""GPU parity at the BENCHMARKED sizes (run on the B200 with `-m gpu`).

The production path -- Hilbert reorder, ballot list kernel with its 26-bit staged
index, pair rows, packed fp32x2 pair kernel, one-launch ADVANCE step, int32 row
offsets at 39^3 cells -- against the CPU oracle on the configurations bench.py and
BASELINE.json quote numbers on:

* config 3: N = 1 000 000 LJ fluid (fcc k = 63 with 188 vacancies + jitter, rho 0.75):
  cells, CSR arrays and neighbour rows bit-exact (in the caller's order and after the
  Hilbert reorder the step loop applies), forces / energies / virial of both force
  kernels within the stated 1e-5, and three MD steps of the native loop (integrate,
  one-launch force+finalize+integrate, force+finalize) against the oracle's loop;
* config 4: Kob-Andersen N = 262 144 (rho 1.2, per-pair-type tables): forces of both
  kernels vs the oracle.

The measured M1 / M2 / M3 figures are printed (`pytest -s`) and written to
``gpurun_out/parity_bench_sizes.json`` so that they can be quoted.

Matches /root/reference/pkg/tests/test_acceptance.py:32-79 (force oracle and list
exactness), scaled to the benchmark's sizes.
"""
import json
import os

import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from conftest import ROOT
from helpers import backward_error, fluid_state, force_error_metrics, quantize_f32
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

FORCE_TOL = 1e-5          # stated fp32 tolerance (BASELINE.json north_star)
N_MILLION = 1_000_000
R_CUT, SKIN = 2.5, 0.3
R_LIST = R_CUT + SKIN

_REPORT = {}


def _record(key, value):
    _REPORT[key] = value
    out = os.path.join(ROOT, "gpurun_out")
    try:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, "parity_bench_sizes.json"), "w") as fh:
            json.dump(_REPORT, fh, indent=1, sort_keys=True)
    except OSError:          # read-only checkout: the printed values remain
        pass
    print(f"[parity] {key}: {value}")


def assert_rows_equal(nl, onl):
    assert nl.overflow == onl.overflow
    cnt = nl.counts
    assert np.array_equal(cnt, onl.counts)
    width = onl.indices.shape[1]
    mask = np.arange(width)[None, :] < cnt[:, None]
    got = nl.indices[:, :width]
    # compare in slices: a (1 M, 96) boolean temporary is enough, not three of them
    for lo in range(0, cnt.size, 200_000):
        hi = min(lo + 200_000, cnt.size)
        assert np.array_equal(np.where(mask[lo:hi], got[lo:hi], 0),
                              np.where(mask[lo:hi], onl.indices[lo:hi], 0))


@pytest.fixture(scope="module")
def million():
    pos, vel, edge = fluid_state(N_MILLION, seed=2026)
    pos = quantize_f32(pos)
    pos = np.where(pos >= edge, 0.0, pos)            # fl32 may round up onto the face
    vel = quantize_f32(vel)
    return pos, vel, edge


@pytest.fixture(scope="module")
def million_oracle(million):
    pos, _, edge = million
    th = orc.host_threads()
    edges = [edge] * 3
    grid = orc.bin_particles(pos, edges, R_LIST)
    nl = orc.build_neighbor_list(pos, np.zeros((pos.shape[0], 3), np.int64), grid, R_LIST, 96,
                                 r_cut=R_CUT, threads=th)
    assert not nl.overflow
    table = orc.pair_table(1.0, 1.0, R_CUT)
    f, pe, w = orc.forces_truncated(pos, edges, table, nl, threads=th)
    fs, us, ws = orc.pair_scales(pos, edges, table, nl, threads=th)
    return dict(grid=grid, nl=nl, f=f, pe=pe, w=w, fs=fs, us=us, ws=ws)


def test_million_cells_and_rows_bit_exact_in_caller_order(million, million_oracle):
    pos, _, edge = million
    box = b2.SimBox.cubic(edge)
    st = b2.ParticleState(pos)
    grid = b2.bin_particles(st, box, R_LIST)
    og = million_oracle["grid"]
    assert np.array_equal(grid.cells_per_axis, og.cells_per_axis)       # 39^3
    assert int(np.prod(grid.cells_per_axis)) == 59319
    assert np.array_equal(grid.cell_of_particle, og.cell_of_particle)
    assert np.array_equal(grid.cell_start, og.cell_start)
    assert np.array_equal(grid.cell_particles, og.cell_particles)
    nl = b2.build_neighbor_list(st, grid, R_LIST, 96, r_cut=R_CUT)
    assert_rows_equal(nl, million_oracle["nl"])
    assert np.array_equal(nl.positions_at_build, million_oracle["nl"].positions_at_build)
    _record("million.rows_identical_caller_order", True)
    _record("million.mean_listed", float(nl.counts.mean()))


def test_million_rows_bit_exact_after_the_hilbert_reorder(million):
    """What the step loop does at every rebuild: Hilbert reorder, bin, ballot list kernel on
    cell-contiguous rows (rows born ascending), pair rows.  The oracle runs on the permuted
    coordinates, so rows are compared index for index."""
    pos, _, edge = million
    box = b2.SimBox.cubic(edge)
    st = b2.ParticleState(pos)
    perm = b2.reorder_hilbert(st, box, R_LIST)
    want_perm, _ = orc.hilbert_permutation(pos, [edge] * 3, R_LIST)
    assert np.array_equal(perm, want_perm)
    ppos = pos[perm]
    grid = b2.bin_particles(st, box, R_LIST)
    og = orc.bin_particles(ppos, [edge] * 3, R_LIST)
    assert np.array_equal(grid.cell_of_particle, og.cell_of_particle)
    assert np.array_equal(grid.cell_particles, og.cell_particles)
    # after the reorder every cell is a contiguous, ascending range of rows (cells follow
    # the curve, so consecutive flat cell numbers are not neighbours in memory)
    cp, cs = grid.cell_particles, grid.cell_start
    inside = np.ones(cp.size, dtype=bool)
    inside[cs[:-1][cs[:-1] < cp.size]] = False           # first occupant of every cell
    assert np.all(np.diff(cp)[inside[1:]] == 1)
    nl = b2.build_neighbor_list(st, grid, R_LIST, 96, r_cut=R_CUT)
    onl = orc.build_neighbor_list(ppos, np.zeros((pos.shape[0], 3), np.int64), og, R_LIST, 96,
                                  r_cut=R_CUT, threads=orc.host_threads())
    assert_rows_equal(nl, onl)
    # pair rows derived from them: union of the two rows, ascending, with ownership flags
    d_pair, d_cnt, pair_pitch = nl.pair_rows()
    counts = d_cnt.cpu().numpy()
    idx, cnt = onl.indices, onl.counts
    sample = list(range(0, 64)) + list(range(250_000, 250_064)) + list(range(499_936, 500_000))
    # (tiles, pitch, 4) -> entry k of pair t, for the sampled pairs only
    rows = {t: d_pair[:, t, :].reshape(-1).cpu().numpy() for t in sample}
    for t in sample:
        a = set(idx[2 * t, :cnt[2 * t]].tolist())
        b = set(idx[2 * t + 1, :cnt[2 * t + 1]].tolist())
        union = sorted(a | b)
        assert counts[t] == len(union)
        got = rows[t][:counts[t]]
        assert np.array_equal(got >> 2, union)
        assert np.array_equal(got & 1, [j in a for j in union])
        assert np.array_equal((got >> 1) & 1, [j in b for j in union])
    _record("million.rows_identical_hilbert_order", True)


def cutoff_band_particles(pos, edge, onl, rows, rel_band=4e-7):
    """Of the particles `rows`, those with a listed pair whose fp64 r^2 lies within
    `rel_band` (a few fp32 roundings of the squared distance) of r_c^2.  The truncated LJ
    force is DISCONTINUOUS at r_c (|F(r_c)| = 0.039 for epsilon = sigma = 1, r_c = 2.5; the
    energy is shifted, the force is not: potential.py:42-66), so for such a pair an fp32
    kernel may legitimately land on the other side of `r2 >= rc2` (forces.py:92) than the
    fp64 reference; the stated tolerance cannot apply to it.  At N = 10^6 about 15 such
    pairs exist (4 pi r_c^2 rho * r_c * rel_band * N / 2)."""
    out = []
    rc2 = R_CUT * R_CUT
    for i in rows:
        j = onl.indices[i, :onl.counts[i]]
        d = pos[i] - pos[j]
        d -= edge * np.rint(d / edge)
        r2 = (d * d).sum(axis=1)
        if np.any(np.abs(r2 - rc2) <= rel_band * rc2):
            out.append(int(i))
    return out


def test_million_forces_of_both_kernels_vs_oracle(million, million_oracle):
    pos, _, edge = million
    o = million_oracle
    box = b2.SimBox.cubic(edge)
    lj = b2.make_shifted(1.0, 1.0, R_CUT)
    st = b2.ParticleState(pos)
    grid = b2.bin_particles(st, box, R_LIST)
    nl = b2.build_neighbor_list(st, grid, R_LIST, 96, r_cut=R_CUT)
    for pair_rows, name in ((True, "pair_kernel"), (False, "row_kernel")):
        b2.compute_forces_truncated(st, lj, box, nl, pair_rows=pair_rows)
        f = st.forces.acquire_read(b2.HOST)
        pe = st.per_particle_potential.acquire_read(b2.HOST)
        w = st.virial.acquire_read(b2.HOST)
        # particles whose error exceeds the tolerance must all have a pair inside the fp32
        # guard band of the cutoff sphere (see cutoff_band_particles); they are then set
        # aside, counted, and their error is bounded by the force discontinuity itself
        err = np.max(np.abs(f - o["f"]), axis=1)
        suspects = np.nonzero(err > 0.5 * FORCE_TOL * o["fs"])[0]
        banded = cutoff_band_particles(pos, edge, o["nl"], suspects)
        assert sorted(banded) == sorted(suspects.tolist()), (len(banded), len(suspects))
        assert len(banded) <= 200
        if len(banded):
            assert err[banded].max() <= 1.05 * 0.039 * 2      # at most two flipped pairs each
        keep = np.ones(pos.shape[0], dtype=bool)
        keep[banded] = False
        m = force_error_metrics(f[keep], o["f"][keep], o["fs"][keep])
        m["particles_with_a_pair_in_the_cutoff_band"] = len(banded)
        m["max_error_of_those"] = float(err[banded].max()) if len(banded) else 0.0
        m["L2"] = float(np.linalg.norm(f - o["f"]) / np.linalg.norm(o["f"]))       # everyone
        m["pe_backward"] = backward_error(pe, o["pe"], o["us"])                    # everyone
        m["virial_backward"] = backward_error(w[keep], o["w"][keep], o["ws"][keep])
        m["pe_total_rel"] = float(abs(pe.sum() - o["pe"].sum()) / np.abs(o["pe"]).sum())
        _record(f"million.{name}", m)
        assert m["M2"] <= FORCE_TOL, m           # error / sum_j |f_ij|: the stated metric
        assert m["L2"] <= FORCE_TOL, m
        # (M3 = error / rms force is recorded only: this jittered lattice has particles whose
        # pair terms are 100x the rms force, so an absolute scale says nothing here)
        # error against the NET force of the particle (cancellation-sensitive):
        # measured value is recorded above; the bound documents what fp32 pair terms give
        assert m["M1"] <= 1e-4, m
        assert m["pe_backward"] <= FORCE_TOL and m["virial_backward"] <= FORCE_TOL, m
        assert m["pe_total_rel"] <= 1e-6, m


def oracle_loop_forces_from_high_words(pos, vel, edge, table, dt, skin, steps, stride=96):
    """The oracle's step loop (sim.py:114-129, integrate.py:58-79) with ONE documented change:
    forces are evaluated at the fp32 high words of the positions, as the device kernels do
    (double-single positions for the drift, fp32 pair arithmetic on the high
    words -- the paper's dsfloat scheme).  Everything else is fp64."""
    th = orc.host_threads()
    edges = np.array([edge] * 3)
    n = pos.shape[0]
    img = np.zeros((n, 3), np.int64)
    masses = np.ones(n)

    def hi(p):
        q = p.astype(np.float32).astype(np.float64)
        return np.where(q >= edge, q - edge, q)

    grid = orc.bin_particles(pos, edges, R_CUT + skin)
    nl = orc.build_neighbor_list(pos, img, grid, R_CUT + skin, stride, r_cut=R_CUT, threads=th)
    evaluated_at = [hi(pos)]
    f, pe, w = orc.forces_truncated(evaluated_at[-1], edges, table, nl, threads=th)
    for _ in range(steps):
        pos, img, vel = orc.vv_integrate(pos, img, vel, f, masses, edges, dt)
        assert not orc.needs_rebuild(pos, img, edges, nl)
        evaluated_at.append(hi(pos))
        f, pe, w = orc.forces_truncated(evaluated_at[-1], edges, table, nl, threads=th)
        vel = orc.vv_finalize(vel, f, masses, dt)
    return pos, img, vel, pe, nl, evaluated_at


def test_million_three_native_steps_vs_oracle_loop():
    """run(3) of the native loop = integrate | force+finalize+integrate (ONE launch, the
    ADVANCE kernel) x 2 | force + finalize, from an fp32-representable state, against the
    oracle's fp64 loop evaluating forces at the fp32 high words (the device's documented
    scheme), and -- recorded, looser -- against the pure fp64 loop."""
    pos, vel, edge = fluid_state(N_MILLION, seed=3033, jitter=0.03)
    pos = quantize_f32(pos)
    pos = np.where(pos >= edge, 0.0, pos)
    vel = quantize_f32(vel)
    box = b2.SimBox.cubic(edge)
    lj = b2.make_shifted(1.0, 1.0, R_CUT)
    dt = 0.001
    st = b2.ParticleState(pos, velocities=vel)
    sim = b2.Simulation(st, box, lj, dt, force_mode=b2.TRUNCATED, skin=SKIN,
                        sample_interval=1000, reorder="hilbert")
    assert sim.native and sim.pair_rows and sim.advance
    launches0, rebuilds0 = sim.kernel_launches, sim.rebuild_count
    sim.run(3)
    steps_launches = sim.kernel_launches - launches0
    assert sim.rebuild_count == rebuilds0              # no rebuild inside these three steps
    # integrate, 2 x one-launch step, force, finalize
    assert steps_launches == 5, steps_launches
    got_u = st.unwrapped_positions(box)
    got_v = np.array(st.velocities.acquire_read(b2.HOST))
    got_img = np.array(st.images.acquire_read(b2.HOST))
    s = sim.measure()
    sim.close()

    opos, oimg, ovel, ope, onl, evaluated_at = oracle_loop_forces_from_high_words(
        pos, vel, edge, lj.table(), dt, SKIN, 3)
    want_u = opos + oimg * edge
    vscale = float(np.abs(ovel).max())
    vel_tol = 6 * 2e-7 * max(vscale, 1.0)               # 2e-7 per half-kick
    # a pair inside the fp32 guard band of the cutoff sphere at one of the four force
    # evaluations may be cut on the other side than in fp64 (cutoff_band_particles): its
    # particles are kicked by up to |F(r_c)| dt/2 = 2e-5 differently -- set aside, counted
    verr = np.max(np.abs(got_v - ovel), axis=1)
    suspects = np.nonzero(verr > 0.5 * vel_tol)[0]
    banded = set()
    for at in evaluated_at:
        banded |= set(cutoff_band_particles(at, edge, onl, suspects, rel_band=1e-6))
    assert banded == set(suspects.tolist()), (len(banded), len(suspects))
    assert len(banded) <= 400
    keep = np.ones(pos.shape[0], dtype=bool)
    keep[sorted(banded)] = False
    pos_err = float(np.max(np.abs(got_u - want_u)[keep]))
    vel_err = float(verr[keep].max())
    # pure fp64 loop (positions never rounded): what the high-word scheme itself costs
    osim = orc.Sim(pos, vel, [edge] * 3, lj.table(), dt, SKIN, stride=96,
                   threads=orc.host_threads())
    osim.run(3)
    pure_u = osim.pos + osim.images * osim.edges
    _record("million.three_steps", {
        "unwrapped_position_abs": pos_err, "velocity_abs": vel_err, "velocity_scale": vscale,
        "particles_with_a_pair_in_the_cutoff_band": len(banded),
        "max_velocity_error_of_those": float(verr[sorted(banded)].max()) if banded else 0.0,
        "vs_pure_fp64_loop": {"unwrapped_position_abs": float(np.max(np.abs(got_u - pure_u))),
                              "velocity_abs": float(np.max(np.abs(got_v - osim.vel)))}})
    assert pos_err <= 3e-9                              # 1e-9 per step
    assert vel_err <= vel_tol
    assert np.array_equal(got_img, oimg)
    assert abs(s.potential_energy - ope.sum()) <= 2e-6 * abs(ope.sum())


def test_kob_andersen_262144_forces_vs_oracle():
    """BASELINE.json configs[3]: two species 80:20, per-pair-type epsilon / sigma / r_c
    tables, rho = 1.2 (stride 256: the fcc start lists 134 neighbours)."""
    n = 262_144
    pos, _, edge = fluid_state(n, density=1.2, seed=262, jitter=0.03)
    pos = quantize_f32(pos)
    pos = np.where(pos >= edge, 0.0, pos)
    species = (np.random.default_rng(42).permutation(n) < n // 5).astype(np.int32)
    ka = b2.PairTable.kob_andersen()
    r_list = ka.max_r_cut + SKIN
    th = orc.host_threads()
    box = b2.SimBox.cubic(edge)
    st = b2.ParticleState(pos, species=species)
    grid = b2.bin_particles(st, box, r_list)
    nl = b2.build_neighbor_list(st, grid, r_list, 256, r_cut=ka.max_r_cut)
    og = orc.bin_particles(pos, [edge] * 3, r_list)
    onl = orc.build_neighbor_list(pos, np.zeros((n, 3), np.int64), og, r_list, 256,
                                  r_cut=ka.max_r_cut, threads=th)
    assert_rows_equal(nl, onl)
    table = ka.table()
    rf, rpe, rw = orc.forces_truncated(pos, [edge] * 3, table, onl, species=species, threads=th)
    fs, us, ws = orc.pair_scales(pos, [edge] * 3, table, onl, species=species, threads=th)
    for pair_rows, name in ((True, "pair_kernel"), (False, "row_kernel")):
        b2.compute_forces_truncated(st, ka, box, nl, pair_rows=pair_rows)
        f = st.forces.acquire_read(b2.HOST)
        pe = st.per_particle_potential.acquire_read(b2.HOST)
        w = st.virial.acquire_read(b2.HOST)
        m = force_error_metrics(f, rf, fs)
        m["L2"] = float(np.linalg.norm(f - rf) / np.linalg.norm(rf))
        m["pe_backward"] = backward_error(pe, rpe, us)
        m["virial_backward"] = backward_error(w, rw, ws)
        _record(f"kob_andersen_262144.{name}", m)
        assert m["M2"] <= FORCE_TOL and m["L2"] <= FORCE_TOL and m["M3"] <= FORCE_TOL, m
        assert m["M1"] <= 1e-4, m
        assert m["pe_backward"] <= FORCE_TOL and m["virial_backward"] <= FORCE_TOL, m
