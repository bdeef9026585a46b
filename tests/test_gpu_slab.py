"""Slab decomposition with the real CUDA backend (`-m gpu`).  The box has one
GPU, so two ranks share cuda:0 and talk over gloo (SlabComm stages device
buffers through the host for that backend; production uses NCCL send/recv on
device buffers with the same protocol code)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

pytestmark = pytest.mark.gpu

N_PER_RANK, DENSITY, T0, DT, SKIN, STEPS = 4000, 0.75, 2.0, 0.002, 0.3, 100


def global_system(world):
    from oracle import oracle as orc
    block, edge = orc.fcc_lattice(N_PER_RANK, DENSITY)
    pos = np.concatenate([block + np.array([r * edge, 0.0, 0.0]) for r in range(world)])
    vel = orc.maxwell_velocities(N_PER_RANK * world, T0, 7)
    q32 = lambda a: a.astype(np.float32).astype(np.float64)
    return q32(pos), q32(vel), (edge * world, edge, edge)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2406_04210_b200 as b2
        from paper_2406_04210_b200.decomp import CudaSlabOps, SlabComm, SlabGeometry, SlabSimulation
        pos, vel, edges = global_system(world)
        geo = SlabGeometry(rank, world, edges)
        mine = np.flatnonzero((pos[:, 0] >= geo.x_lo) & (pos[:, 0] < geo.x_lo + geo.width))
        ops = CudaSlabOps(pos[mine], vel[mine], mine, edges, device_index=0, stride=32)
        sim = SlabSimulation(ops, SlabComm(geo), b2.make_shifted(1.0, 1.0, 2.5), DT, SKIN,
                             sample_interval=25)
        first = sim.measure()
        sim.run(STEPS)
        ids, p, v = ops.owned_state()
        out[rank] = dict(ids=ids, pos=p, vel=v, samples=[first] + sim.samples,
                         rebuilds=sim.rebuilds, stride=ops.stride, halo=sim.halo_rows,
                         left_home=int(np.count_nonzero(~np.isin(ids, mine))),
                         launches=ops.kernel_launches)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2])
def test_cuda_slab_run_tracks_single_domain_oracle(world):
    from oracle import oracle as orc
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]

    pos, vel, edges = global_system(world)
    ref = orc.Sim(pos, vel, edges, orc.pair_table(1.0, 1.0, 2.5), DT, SKIN, stride=128,
                  sample_interval=25, threads=orc.host_threads())
    ref.samples.append(ref.measure())
    ref.run(STEPS)

    n = N_PER_RANK * world
    ids = np.concatenate([r["ids"] for r in res])
    assert sorted(ids.tolist()) == list(range(n))
    if world > 1:
        assert sum(r["left_home"] for r in res) > 0           # migration happened
        assert all(min(r["halo"]) > 0 for r in res)
    assert all(r["rebuilds"] >= 3 and r["launches"] > 2 * STEPS for r in res)
    order = np.argsort(ids)
    got_pos = np.concatenate([r["pos"] for r in res])[order]
    d = got_pos - ref.pos
    d -= np.array(edges) * np.rint(d / np.array(edges))
    assert np.max(np.abs(d)) <= 2e-3          # fp32 forces vs fp64 over 100 hot steps
    for r in res:
        for a, b in zip(r["samples"], ref.samples):
            assert a["step"] == b["step"] and a["n"] == n
            assert a["pe"] == pytest.approx(b["pe"], rel=2e-5)
            assert a["ke"] == pytest.approx(b["ke"], rel=2e-5)
            assert a["virial"] == pytest.approx(b["virial"], rel=5e-4)
    e = np.array([s["total_energy"] for s in res[0]["samples"]])
    assert np.max(np.abs(e - e[0])) <= 2e-4 * abs(e[0])
