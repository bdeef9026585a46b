"""Workload for the compute-sanitizer job (profiles/sanitize.sh): every kernel family of the
hot path on small systems -- operator path (bin, list, pair rows, both force kernels,
integrate, finalize, reductions, reorder), native loop with rebuilds (row kernel, pair rows +
one-launch steps, queue depth 8, CUDA-graph steps), thermostat in the native loop, Kob-Andersen
tables, all-pairs kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_04210_b200 as b2

def lattice(n, rho=0.75, t=1.2):
    st, box = b2.init_lattice_any(n, rho)
    b2.init_velocities(st, t, 42)
    return st, box

lj = b2.make_shifted(1.0, 1.0, 2.5)
steps = int(os.environ.get("SAN_STEPS", "200"))
# operator path
st, box = lattice(4096)
grid = b2.bin_particles(st, box, 2.8)
nl = b2.build_neighbor_list(st, grid, 2.8, 96, r_cut=2.5)
for pr in (False, True):
    b2.compute_forces_truncated(st, lj, box, nl, pair_rows=pr)
b2.vv_integrate(st, b2.IntegratorParams(0.001), box, nlist=nl)
b2.vv_finalize(st, b2.IntegratorParams(0.001))
print("needs_rebuild", b2.needs_rebuild(st, box, nl))
b2.reorder_hilbert(st, box, 2.8)
print("KE", b2.kinetic_energy_and_temperature(st))
# native loops
variants = [dict(pair_rows=False), dict(pair_rows=True, advance=True),
            dict(pair_rows=True, advance=True, queue_depth=8),
            dict(pair_rows=True, advance=True, prune_delta=0.1),      # pruned pair rows
            dict(thermostat=b2.ThermostatParams(1.2, 20.0, 7))]
if os.environ.get("SAN_GRAPH") == "1":      # CUDA-graph steps (conditional IF nodes) only
    variants = [dict(graph=4)]
for kw in variants:
    st, box = lattice(4096)
    sim = b2.Simulation(st, box, lj, 0.002, force_mode=b2.TRUNCATED, skin=0.3, sample_interval=50,
                        **kw)
    sim.run(steps)
    print(kw, "rebuilds", sim.rebuild_count, "E", sim.measure().total_energy)
    sim.close()
if os.environ.get("SAN_GRAPH") == "1":
    print("SANITIZE_WORKLOAD_DONE")
    sys.exit(0)
# Kob-Andersen tables through pair rows, all-pairs kernel
n = 2048
st, box = lattice(n, rho=1.2)
sp = (np.random.default_rng(1).permutation(n) < n // 5).astype(np.int32)
st2 = b2.ParticleState(np.array(st.positions.acquire_read(b2.HOST)),
                       velocities=np.array(st.velocities.acquire_read(b2.HOST)), species=sp)
sim = b2.Simulation(st2, box, b2.PairTable.kob_andersen(), 0.002, force_mode=b2.TRUNCATED, skin=0.3,
                    pair_rows=True, advance=True)
sim.run(60); print("KA E", sim.measure().total_energy); sim.close()
st, box = lattice(500, rho=0.8)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0), 0.002, force_mode=b2.ALL_TO_ALL)
sim.run(20); print("all-pairs E", sim.measure().total_energy); sim.close()
# ... its thermostatted loop (finalize + thermostat + integrate in one pass), the table variant,
# and the 4-warp / one-thread-per-particle shapes of the all-pairs kernel (one evaluation each)
st, box = lattice(500, rho=0.8)
sim = b2.Simulation(st, box, b2.make_shifted(1.0, 1.0), 0.002,
                    thermostat=b2.ThermostatParams(1.0, 20.0, 3))
sim.run(20); print("all-pairs NVT E", sim.measure().total_energy); sim.close()
st, box = lattice(600, rho=1.2)
sp = (np.random.default_rng(2).permutation(600) < 120).astype(np.int32)
st2 = b2.ParticleState(np.array(st.positions.acquire_read(b2.HOST)),
                       velocities=np.array(st.velocities.acquire_read(b2.HOST)), species=sp)
sim = b2.Simulation(st2, box, b2.PairTable.kob_andersen(), 0.002)
sim.run(10); print("all-pairs KA E", sim.measure().total_energy); sim.close()
if os.environ.get("SAN_BIG_ALL_PAIRS", "1") == "1":
    st, box = lattice(12500, rho=0.8)
    b2.compute_forces_all_to_all(st, b2.make_shifted(1.0, 1.0), box)
    print("all-pairs 12500 PE", b2.potential_energy_total(st))
print("SANITIZE_WORKLOAD_DONE")
