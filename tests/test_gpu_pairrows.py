"""Pair rows (b2md_pair_rows) and the two-particles-per-thread force kernel
(b2md_force_lj_pairs): the merged rows are exactly the ascending union of the two
per-particle rows with the right ownership flags, and everything computed from
them is bit-identical to the thread-per-particle path (forces, energies, virial,
whole trajectories, error reporting)."""
import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from helpers import fluid_state, quantize_f32

pytestmark = pytest.mark.gpu


def build(pos, edge, r_list=2.8, stride=128, species=None):
    box = b2.SimBox.cubic(edge)
    st = b2.ParticleState(pos, species=species)
    grid = b2.bin_particles(st, box, r_list)
    nl = b2.build_neighbor_list(st, grid, r_list, stride, r_cut=2.5)
    assert not nl.overflow
    return st, box, nl


@pytest.mark.parametrize("n", [1, 2, 63, 500, 4097])
def test_pair_rows_are_the_flagged_union_of_both_rows(n):
    gen = np.random.default_rng(n)
    edge = max((n / 0.75) ** (1.0 / 3.0), 9.0)
    pos = quantize_f32(gen.uniform(0, edge, size=(n, 3)))
    st, box, nl = build(pos, edge)
    idx, cnt = nl.indices, nl.counts
    d_pair, d_cnt, pair_pitch = nl.pair_rows()
    tiles = d_pair.shape[0]
    # (tiles, pitch, 4) -> (pitch, 4 * tiles): entry k of pair t
    rows = d_pair.permute(1, 0, 2).reshape(pair_pitch, 4 * tiles).cpu().numpy()
    counts = d_cnt.cpu().numpy()
    n_pairs = (n + 1) // 2
    assert pair_pitch % 32 == 0 and pair_pitch >= n_pairs
    assert np.all(counts[n_pairs:] == 0)
    for t in range(n_pairs):
        a = set(idx[2 * t, :cnt[2 * t]].tolist())
        b = set(idx[2 * t + 1, :cnt[2 * t + 1]].tolist()) if 2 * t + 1 < n else set()
        union = sorted(a | b)
        assert counts[t] == len(union)
        got = rows[t, :counts[t]]
        assert np.array_equal(got >> 2, union)
        assert np.array_equal(got & 1, [j in a for j in union])
        assert np.array_equal((got >> 1) & 1, [j in b for j in union])
    # padding up to the longest row of each warp carries no flags
    for w in range(0, pair_pitch, 32):
        longest = (int(counts[w:w + 32].max()) + 3) // 4 * 4
        for t in range(w, min(w + 32, pair_pitch)):
            assert np.all(rows[t, counts[t]:longest] & 3 == 0)


@pytest.mark.parametrize("n,density", [(1001, 0.75), (20_000, 0.75), (8192, 1.2),
                                       (262_144, 0.75), (262_145, 1.2)])
def test_pair_kernel_matches_the_row_kernel(n, density):
    """Same pair terms in the same ascending-j order: bit-identical to the
    thread-per-particle kernel (n >= 200 000); small systems run the row kernel with
    four lanes per particle, whose partial sums are combined in another order."""
    pos, _, edge = fluid_state(n, density=density, seed=n)
    pos = quantize_f32(pos)
    species = None
    params = b2.make_shifted(1.0, 1.0, 2.5)
    if density > 1.0:                      # Kob-Andersen tables
        species = (np.random.default_rng(1).permutation(n) < n // 5).astype(np.int32)
        params = b2.PairTable.kob_andersen()
    st, box, nl = build(pos, edge, stride=256, species=species)
    out = []
    for pr in (False, True):
        b2.compute_forces_truncated(st, params, box, nl, pair_rows=pr)
        out.append([np.array(getattr(st, name).acquire_read(b2.HOST))
                    for name in ("forces", "per_particle_potential", "virial")])
    assert np.abs(out[0][0]).max() > 0.0
    for x, y in zip(*out):
        if n >= 200_000:
            assert np.array_equal(x, y)
        else:
            assert np.max(np.abs(x - y)) <= 2e-6 * np.abs(x).max()


def test_pair_kernel_reports_singular_pairs_like_the_reference():
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    box = b2.SimBox.cubic(10.0)
    pos = np.array([[1.0, 1.0, 1.0], [3.0, 3.0, 3.0], [1.0, 1.0, 1.0], [5.0, 5.0, 5.0],
                    [9.75, 2.0, 2.0], [-0.25 + 10.0, 2.0, 2.0]])
    pos[5] = pos[4]                         # second coincident pair, higher i
    st = b2.ParticleState(pos)
    grid = b2.bin_particles(st, box, 3.0)
    nl = b2.build_neighbor_list(st, grid, 3.0, 8, r_cut=2.5)
    with pytest.raises(b2.SingularPairError) as exc:
        b2.compute_forces_truncated(st, lj, box, nl, pair_rows=True)
    assert (exc.value.i, exc.value.j) == (0, 2)


def test_trajectory_with_and_without_pair_rows():
    n = 4096
    series = []
    for pr in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=50,
                            sample_initial=True, pair_rows=pr)
        assert sim.pair_rows == pr
        sim.run(300)
        series.append((np.array([s.total_energy for s in sim.samples]),
                       np.array([s.potential_energy for s in sim.samples]),
                       sim.rebuild_count))
    # (the small-system row kernel sums four partial rows: not bitwise the same)
    assert series[0][2] >= 5 and abs(series[0][2] - series[1][2]) <= 1
    assert np.max(np.abs(series[0][0] - series[1][0])) <= 2e-6 * abs(series[0][0][0])
    assert np.max(np.abs(series[0][1] - series[1][1])) <= 1e-4 * abs(series[0][1][0])


def test_large_trajectory_is_bit_identical_with_and_without_pair_rows():
    n = 262_144
    series = []
    for pr in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=40,
                            sample_initial=True, pair_rows=pr)
        assert sim.pair_rows == pr
        sim.run(120)
        series.append((np.array([s.total_energy for s in sim.samples]),
                       np.array(st.positions.acquire_read(b2.HOST)), sim.rebuild_count))
    assert series[0][2] == series[1][2] and series[0][2] >= 2
    assert np.array_equal(series[0][0], series[1][0])
    assert np.array_equal(series[0][1], series[1][1])


def test_stride_growth_reallocates_pair_rows():
    # fcc start at stride 64 overflows once (78 listed neighbours): the runner grows
    # both the list and its pair rows and the run continues
    n = 4096
    st, box = b2.init_lattice_any(n, 0.75)
    b2.init_velocities(st, 1.2, 42)
    sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                        force_mode=b2.TRUNCATED, skin=0.3, stride=64, pair_rows=True)
    assert sim.overflow_events >= 1
    sim.run(20)
    e0 = sim.measure().total_energy
    sim.run(50)
    assert abs(sim.measure().total_energy - e0) <= 1e-4 * abs(e0)


@pytest.mark.parametrize("n,steps", [(4096, 400), (262_144, 150)])
def test_one_launch_steps_are_bit_identical_to_separate_launches(n, steps):
    """b2md_force_lj_pairs_advance applies the same kicks / drift / wrap to the same fp32
    forces as the separate integrate launch would: identical trajectories, energies,
    image counters and rebuild schedule."""
    out = []
    for advance in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=37,
                            sample_initial=True, pair_rows=True, advance=advance)
        sim.run(steps)
        sim.run(3)                       # a short call: first / last step handling
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST)),
                    np.array(st.images.acquire_read(b2.HOST)),
                    np.array(st.forces.acquire_read(b2.HOST)), sim.rebuild_count,
                    sim.kernel_launches))
    assert out[0][5] == out[1][5] and out[0][5] >= 3
    for k in range(5):
        assert np.array_equal(out[0][k], out[1][k]), k
    assert out[1][6] < 0.8 * out[0][6]          # one launch per intermediate step instead of two


def test_one_launch_steps_survive_stride_growth_and_wraps():
    # stride 64 overflows on the fcc start; dt large enough that particles cross faces
    n = 8192
    out = []
    for advance in (False, True):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 2.0, 7)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.004,
                            force_mode=b2.TRUNCATED, skin=0.3, stride=64, sample_interval=50,
                            pair_rows=True, advance=advance)
        sim.run(500)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.images.acquire_read(b2.HOST)), sim.rebuild_count))
    assert np.abs(out[0][2]).max() >= 1                       # some particle wrapped
    assert out[0][3] == out[1][3]
    for k in range(3):
        assert np.array_equal(out[0][k], out[1][k]), k


def test_one_launch_steps_with_pair_tables():
    n = 16_384
    species = (np.random.default_rng(42).permutation(n) < n // 5).astype(np.int32)
    out = []
    for advance in (False, True):
        st, box = b2.init_lattice_any(n, 1.2)
        st = b2.ParticleState(st.positions.acquire_read(b2.HOST), species=species)
        b2.init_velocities(st, 1.0, 42)
        sim = b2.Simulation(st, box, b2.PairTable.kob_andersen(), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=40,
                            sample_initial=True, pair_rows=True, advance=advance)
        sim.run(200)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)), sim.rebuild_count))
    assert out[0][2] == out[1][2] and out[0][2] >= 2
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])
    assert abs(out[1][0][-1] - out[1][0][0]) <= 5e-5 * abs(out[1][0][0])


@pytest.mark.parametrize("n,depth", [(4096, 8), (4096, 3), (32_768, 16)])
def test_queued_one_launch_steps_are_bit_identical(n, depth):
    """Several gated launches per status read-back: a due rebuild turns the launches queued
    behind it into no-ops, the device counts the steps taken -- same trajectory as one
    read-back per step."""
    out = []
    for queue_depth in (1, depth):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=53,
                            sample_initial=True, pair_rows=True, advance=True,
                            queue_depth=queue_depth)
        sim.run(500)
        sim.run(2)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST)),
                    np.array(st.images.acquire_read(b2.HOST)), sim.rebuild_count))
    assert out[0][4] == out[1][4] and out[0][4] >= 5
    for k in range(4):
        assert np.array_equal(out[0][k], out[1][k]), k


@pytest.mark.parametrize("n,depth", [(4096, 1), (4096, 8), (20_000, 5)])
def test_row_kernel_one_launch_steps_are_bit_identical(n, depth):
    """The thread-per-particle kernel with the ADVANCE epilogue (small systems), one or
    several launches per status read-back, against separate integrate / force launches."""
    out = []
    for kw in (dict(advance=False), dict(advance=True, queue_depth=depth)):
        st, box = b2.init_lattice_any(n, 0.75)
        b2.init_velocities(st, 1.2, 42)
        sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0, 2.5), 0.001,
                            force_mode=b2.TRUNCATED, skin=0.3, sample_interval=41,
                            sample_initial=True, pair_rows=False, **kw)
        sim.run(400)
        sim.run(2)
        out.append((np.array([s.total_energy for s in sim.samples]),
                    np.array(st.positions.acquire_read(b2.HOST)),
                    np.array(st.velocities.acquire_read(b2.HOST)),
                    np.array(st.images.acquire_read(b2.HOST)),
                    np.array(st.forces.acquire_read(b2.HOST)), sim.rebuild_count))
    assert out[0][5] == out[1][5] and out[0][5] >= 5
    for k in range(5):
        assert np.array_equal(out[0][k], out[1][k]), k
