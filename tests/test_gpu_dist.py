"""The multi-GPU path (VERDICT r1 "next" 2) with the REAL kernels: two processes
(gloo, world size 2) on the one B200 of a gpurun box, each running fiber_intersect_nearest on
its ray shard in chunk launches and gathering the per-ray records (ShardedNearest).  The
gathered records and the per-pair records must be bit-identical to one process doing all
rays.  The two ranks' kernels never wait on one another (only the host-side gloo gather
synchronises), so sharing one GPU is safe.  Needs a B200."""
import os
import socket

import numpy as np
import pytest

from workloads import gen

pytestmark = pytest.mark.gpu
N_RAYS, N_STRANDS, DEPTH, K = 1 << 13, 1 << 12, 6, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, rank, out_dir):
    import torch

    import paper_1811_03374_b200 as fx
    from paper_1811_03374_b200 import dist as fxd

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    perm = fxd.ray_permutation(N_RAYS, seed=5)
    all_owned = [perm[slice(*fxd.shard_bounds(N_RAYS, world, r))] for r in range(world)]
    owned = all_owned[rank]
    w = gen.config5(n_rays=N_RAYS, n_strands=N_STRANDS, depth=DEPTH, ray_ids=owned)
    pairs, bounds, blocks = fxd.chunk_by_ray(w.pairs, owned, N_RAYS, K, local=True)
    rays = torch.from_numpy(w.rays[owned]).to(dev)  # the rank's own rays, in shard order
    segs = fx.build_segments(torch.from_numpy(w.ctrl).to(dev), torch.from_numpy(w.radii).to(dev))
    sn = fxd.ShardedNearest(fx, rays, segs, pairs, bounds, blocks, DEPTH, dev)
    sn.step()
    sn.step()  # a second pass gives the same records (nearest is re-initialised)
    torch.cuda.synchronize()
    rec = sn.records_by_ray(N_RAYS, all_owned).cpu().numpy()
    np.save(os.path.join(out_dir, f"rec_{world}_{rank}.npy"), rec)
    np.save(os.path.join(out_dir, f"hits_{world}_{rank}.npy"), sn.hits.cpu().numpy())
    gp = pairs.copy()
    gp[:, 0] = owned[pairs[:, 0].astype(np.int64)]  # back to global ray ids
    np.save(os.path.join(out_dir, f"pairs_{world}_{rank}.npy"), gp)


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _run(world, rank, out_dir)
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_one(tmp_path):
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp

    out = str(tmp_path)
    _run(1, 0, out)
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0
    ref = np.load(os.path.join(out, "rec_1_0.npy"))
    assert np.isfinite(ref[:, 0]).mean() > 0.3  # most targeted rays hit
    for r in range(2):
        got = np.load(os.path.join(out, f"rec_2_{r}.npy"))
        assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))  # bit-identical records
    # per-pair records of each rank == the single-process records of the same (ray, seg) pairs
    p1, h1 = np.load(os.path.join(out, "pairs_1_0.npy")), np.load(os.path.join(out, "hits_1_0.npy"))
    key1 = p1[:, 0].astype(np.int64) << 32 | p1[:, 1].astype(np.int64)
    o1 = np.argsort(key1)
    n = 0
    for r in range(2):
        p2, h2 = np.load(os.path.join(out, f"pairs_2_{r}.npy")), np.load(os.path.join(out, f"hits_2_{r}.npy"))
        key2 = p2[:, 0].astype(np.int64) << 32 | p2[:, 1].astype(np.int64)
        j = o1[np.searchsorted(key1[o1], key2)]
        assert np.array_equal(key1[j], key2)
        assert np.array_equal(h1[j].view(np.uint32), h2.view(np.uint32))
        n += p2.shape[0]
    assert n == p1.shape[0]
