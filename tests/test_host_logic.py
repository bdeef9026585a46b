"""CPU-only checks: the C-ABI library loads and exports every declared symbol,
and the host-side mirror of the reference API behaves like the reference
(error behaviour, residency bookkeeping, signal order).  No kernels run here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2406_04210_b200 as b2
from paper_2406_04210_b200 import _lib
from conftest import GOLDEN, ROOT, load_golden


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    assert lib.b2md_version() == 108
    header = open(os.path.join(ROOT, "include", "b2md.h")).read()
    declared = set(re.findall(r"\b(b2md_[a-z0-9_]+)\(", header))
    declared -= {"b2md_box", "b2md_grid", "b2md_status"}
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(lib, name), f"{name} declared in b2md.h but not exported"
    # and the binding table covers the header
    assert declared <= set(_lib.exported_symbols()) | {"b2md_runner"}


def test_struct_layouts_match_the_header():
    assert ctypes.sizeof(_lib.Status) == 64
    assert ctypes.sizeof(_lib.Box) == 24
    assert ctypes.sizeof(_lib.Grid) == 48


def test_grid_shape_host_arithmetic():
    # test_neighbor.py:30-45 : box (10,8,6), r_list 2 -> 5x4x3 cells
    from paper_2406_04210_b200.neighbor import grid_shape
    g = grid_shape(b2.SimBox((10.0, 8.0, 6.0)), 2.0)
    assert list(g.ncell) == [5, 4, 3] and g.fallback == 0 and g.n_cells == 60
    assert list(g.cell_edge) == [2.0, 2.0, 2.0]
    assert grid_shape(b2.SimBox.cubic(5.0), 2.0).fallback == 1
    NB = load_golden("neighbor")
    for name in [str(x) for x in NB["names"]]:
        g = grid_shape(b2.SimBox(NB[f"{name}.edges"]), float(NB[f"{name}.r_list"]))
        assert list(g.ncell) == list(NB[f"{name}.ncells"])
        assert np.array_equal(np.array(list(g.cell_edge)), NB[f"{name}.cell_edge"])
        assert bool(g.fallback) == bool(NB[f"{name}.fallback"])
    with pytest.raises(b2.ConfigError):
        grid_shape(b2.SimBox((4.0, 10.0, 10.0)), 4.5)     # test_neighbor.py:76-82
    with pytest.raises(ValueError):
        grid_shape(b2.SimBox.cubic(10.0), -1.0)


def test_box_validation_and_helpers():
    with pytest.raises(ValueError):
        b2.SimBox((1.0, 2.0))
    with pytest.raises(ValueError):
        b2.SimBox((1.0, -2.0, 3.0))
    box = b2.SimBox.cubic(10.0)
    assert box.volume == 1000.0
    G = load_golden("integrate")
    w, k = b2.wrap_position(G["wrap_in"], G["wrap_img"], box)
    assert np.array_equal(w, G["wrap_out"]) and np.array_equal(k, G["wrap_img_out"])
    assert np.array_equal(b2.minimum_image(G["mi_in"], box), G["mi_out"])


def test_particle_state_validation_and_host_residency():
    with pytest.raises(ValueError):
        b2.ParticleState(np.zeros((3, 2)))
    with pytest.raises(ValueError):
        b2.ParticleState(np.zeros((2, 3)), masses=[1.0, 0.0])
    st = b2.ParticleState(np.array([[1.0, 2.0, 3.0]]))
    assert st.n == 1 and set(st.buffers()) >= {
        "positions", "images", "velocities", "forces", "masses", "species",
        "per_particle_potential"}
    buf = st.positions
    assert buf.valid_on == b2.HOST and buf.version == 0 and buf.copy_count == 0
    view = buf.acquire_read(b2.HOST)
    assert not view.flags.writeable
    buf.acquire_write(b2.HOST)[0, 0] = 4.0
    assert buf.version == 1 and buf.acquire_read(b2.HOST)[0, 0] == 4.0
    with pytest.raises(ValueError):
        buf.acquire_read("gpu")
    with pytest.raises(ValueError):
        st.validate(b2.SimBox.cubic(3.5))   # x=4.0 outside [0, 3.5)


def test_compute_side_fails_loudly_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    st = b2.ParticleState(np.zeros((4, 3)))
    with pytest.raises(_lib.B2mdError):
        st.positions.acquire_read(b2.COMPUTE)
    with pytest.raises(_lib.B2mdError):
        b2.bin_particles(st, b2.SimBox.cubic(10.0), 2.5)


def test_backend_selector_rejects_other_kinds():
    # the reference pins that unknown kinds raise ConfigError (test_backend.py:25-30)
    assert b2.BackendSelector().kind == "b200"
    for kind in ("sequential", "parallel", "gpu", "cpu"):
        with pytest.raises(b2.ConfigError):
            b2.BackendSelector(kind=kind)


def test_potential_shift_and_tables():
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    assert lj.energy_shift == pytest.approx(0.016316891136, abs=1e-12)   # test_potential.py:19-23
    assert lj.energy_shift == float(load_golden("forces")["shift_2p5"])
    e, f = b2.lj_eval(np.array([1.0, 6.25, 9.0]), lj)
    assert e[1] == 0.0 and f[2] == 0.0 and e[0] == pytest.approx(lj.energy_shift)
    with pytest.raises(ValueError):
        b2.make_shifted(1.0, 1.0, 0.9)
    ka = b2.PairTable.kob_andersen()
    tab = ka.table()
    assert tab.shape == (4, 4) and ka.max_r_cut == 2.5
    assert np.array_equal(tab[1], tab[2])                      # AB == BA
    assert tab[1, 0] == 1.5 and tab[3, 1] == pytest.approx(0.88 ** 2)
    assert np.array_equal(lj.table()[0], b2.PairTable([[1.0]], [[1.0]], [[2.5]]).table()[0])
    with pytest.raises(ValueError):
        b2.PairTable([[1.0, 2.0], [3.0, 1.0]], np.ones((2, 2)), 2.5 * np.ones((2, 2)))


def test_signal_engine_order_and_sampling():
    eng = b2.SignalEngine(sample_interval=2, sample_initial=True)
    trace = []
    for sig in b2.SignalEngine.SIGNALS:
        eng.connect(sig, lambda s=sig: trace.append(s))
    eng.run_steps(3)
    assert trace == ["sample", "integrate", "force", "finalize",
                     "integrate", "force", "finalize", "sample",
                     "integrate", "force", "finalize"]
    with pytest.raises(b2.ConfigError):
        b2.SignalEngine(sample_interval=0)
    with pytest.raises(b2.ConfigError):
        b2.SignalEngine().run_steps(1)          # no mandatory slots
    with pytest.raises(b2.ConfigError):
        eng.connect("nope", lambda: None)


def test_initial_conditions_match_reference_generators():
    G = load_golden("trajectory")
    st, box = b2.init_lattice_any(int(G["n"]), float(G["density"]))
    b2.init_velocities(st, 1.2, 42)
    assert np.array_equal(st.positions.acquire_read(b2.HOST), G["pos0"])
    assert np.array_equal(st.velocities.acquire_read(b2.HOST), G["vel0"])
    assert np.array_equal(box.edge_lengths, G["edges"])
    st, _ = b2.init_lattice_any(256, 0.8)
    assert np.array_equal(st.positions.acquire_read(b2.HOST), G["lat256"])
    with pytest.raises(ValueError):
        b2.init_lattice(100, 0.8)


def test_simulation_argument_validation():
    st, box = b2.init_lattice_any(32, 0.5)
    lj = b2.make_shifted(1.0, 1.0, 2.5)
    with pytest.raises(b2.ConfigError):
        b2.Simulation(st, box, lj, 0.001, force_mode="nope")
    with pytest.raises(b2.ConfigError):
        b2.Simulation(st, box, b2.make_shifted(1.0, 1.0), 0.001, force_mode=b2.TRUNCATED)
    with pytest.raises(b2.ConfigError):
        b2.Simulation(st, box, lj, 0.001, force_mode=b2.TRUNCATED, skin=-0.1)


def test_bench_config_files_and_records_round_trip(tmp_path):
    # reference bench.py:126-142, 207-263 (test_bench.py analogues)
    cfg_path = tmp_path / "run.cfg"
    cfg_path.write_text("# quick run\nn_particles = 864\ndensity=0.75\nsteps = 50  # short\n"
                        "deterministic = no\nforce_mode = truncated\n")
    cfg = b2.parse_config_file(cfg_path)
    assert (cfg.n_particles, cfg.density, cfg.steps, cfg.deterministic) == (864, 0.75, 50, False)
    assert cfg.backend == "b200"
    (tmp_path / "bad.cfg").write_text("n_particles = 10\nbogus = 1\n")
    with pytest.raises(b2.ConfigError, match=r"bad.cfg:2"):
        b2.parse_config_file(tmp_path / "bad.cfg")
    with pytest.raises(b2.ConfigError):
        b2.BenchConfig(backend="sequential").validate()
    with pytest.raises(b2.ConfigError):
        b2.BenchConfig(r_cut=float("inf")).validate()       # truncated needs a finite cutoff
    assert set(b2.PRESETS) == {"all2all-2k", "all2all-2k-long", "trunc-10k", "smoke-256"}
    assert b2.preset_config("trunc-10k").thermostat_rate == 5.0
    with pytest.raises(b2.ConfigError):
        b2.preset_config("nope")
    rec = b2.BenchRecord(cfg, 0.1234567890123456789, 405.0, 0.6, 0.3, 7, 1, 1.25e-06)
    path = tmp_path / "records.csv"
    b2.write_records_csv(path, [rec])
    b2.write_records_csv(path, [rec], append=True)
    back = b2.read_records_csv(path)
    assert back == [rec, rec]                                  # 17 significant digits round-trip
    header = path.read_text().splitlines()[0].split(",")
    assert header[:3] == ["n_particles", "density", "temperature"] and header[-1] == "engine_version"
    s = b2.Sample(10, 0.02, -1.5, 0.5, -1.0, 1.1, (1e-3, -2e-3, 0.0), 2)
    b2.write_samples_csv(tmp_path / "samples.csv", [s])
    lines = (tmp_path / "samples.csv").read_text().splitlines()
    assert lines[0] == "step,time,potential_energy,kinetic_energy,total_energy,temperature,px,py,pz,rebuild_count"
    assert lines[1].startswith("10,0.02") and lines[1].endswith(",2")


def test_reference_written_csv_files_round_trip_byte_for_byte(tmp_path):
    """tests/golden/reference_records.csv / reference_samples.csv were written by the
    REFERENCE's writers from a sweep it ran itself (make_golden.py harness_csv_case;
    bench.py:222-285, 372-383): the harness reads them and writes the same bytes back."""
    src = os.path.join(GOLDEN, "reference_records.csv")
    records = b2.read_records_csv(src)
    assert [r.config.backend for r in records] == ["sequential", "parallel", "parallel", "parallel"]
    assert [r.config.worker_count for r in records] == [1, 1, 2, 3]
    assert records[0].engine_version == "0.1.0" and records[0].config.n_particles == 108
    out = tmp_path / "records.csv"
    b2.write_records_csv(out, records)
    assert out.read_bytes() == open(src, "rb").read()
    src = os.path.join(GOLDEN, "reference_samples.csv")
    samples = b2.read_samples_csv(src)
    assert [s.step for s in samples] == [20, 30, 40, 50]
    out = tmp_path / "samples.csv"
    b2.write_samples_csv(out, samples)
    assert out.read_bytes() == open(src, "rb").read()
    # same file format as pkg/frontend/test/data/sweep6.csv (header checked verbatim)
    with pytest.raises(b2.ConfigError):
        b2.read_records_csv(os.path.join(GOLDEN, "reference_samples.csv"))


def test_speedup_efficiency_rows_match_the_reference(tmp_path):
    """compute_speedup_efficiency on the reference's own records reproduces its rows
    (bench.py:393-442) for both baselines; B200 records join the same summary."""
    import dataclasses
    records = b2.read_records_csv(os.path.join(GOLDEN, "reference_records.csv"))
    want = np.load(os.path.join(GOLDEN, "harness.npz"))
    for base in ("sequential", "single"):
        rows = b2.compute_speedup_efficiency(records, baseline=base)
        got = np.array([[r.worker_count, r.wall_time_s, r.speedup, r.efficiency] for r in rows])
        assert np.array_equal(got, want[f"speedup_{base}"]), base
        assert all(r.backend == "parallel" for r in rows)
    # a B200 record of the same physics is summarised against the sequential CPU record
    gpu = dataclasses.replace(records[0], wall_time_s=records[0].wall_time_s / 500.0,
                              config=dataclasses.replace(records[0].config, backend="b200"))
    rows = b2.compute_speedup_efficiency(records + [gpu])
    assert rows[-1].backend == "b200" and rows[-1].speedup == pytest.approx(500.0)
    assert rows[-1].efficiency == pytest.approx(1.0)
    with pytest.raises(b2.ConfigError):
        b2.compute_speedup_efficiency([])
    with pytest.raises(b2.ConfigError):
        b2.compute_speedup_efficiency(records, baseline="nope")
    with pytest.raises(b2.ConfigError):                       # no sequential record
        b2.compute_speedup_efficiency(records[1:])
    other = dataclasses.replace(records[1], config=dataclasses.replace(records[1].config, dt=0.004))
    with pytest.raises(b2.ConfigError, match="dt"):
        b2.compute_speedup_efficiency([records[0], other])
    with pytest.raises(b2.ConfigError):
        b2.run_sweep(b2.preset_config("smoke-256"), [0])
