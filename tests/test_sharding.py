"""CPU, world_size 2 over gloo: the multi-GPU path shards streams with no data-path
collective; sharded outputs (oracle on each shard) equal the unsharded run, and the bench's
max-over-ranks timing reduction works.  (The GPU kernels themselves are per-device.)"""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2204_07064_b200.shard import strong_range, weak_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from oracle import pyoracle as po
    from paper_2204_07064_b200 import configs
    from paper_2204_07064_b200.shard import max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    m = configs.build(3, seed=4)
    total = 5
    rng_ = strong_range(total, world, rank)
    x = configs.batch_input(3, rng_, 16, 512, seed=4)
    y = po.run(m, x, [256, 256], "stream", threads=1)
    # gather variable-size shards (pad to the max shard)
    mx = -(-total // world)
    buf = np.zeros((mx,) + y.shape[1:], np.float32)
    buf[:y.shape[0]] = y
    out = [torch.zeros_like(torch.from_numpy(buf)) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(buf))
    t = max_over_ranks(float(rank + 1))
    if rank == 0:
        parts = [out[r][:len(strong_range(total, world, r))].numpy() for r in range(world)]
        q.put((np.concatenate(parts), t))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_equals_unsharded_gloo():
    from oracle import pyoracle as po
    from paper_2204_07064_b200 import configs
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    y_sharded, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = configs.build(3, seed=4)
    x = configs.batch_input(3, range(5), 16, 512, seed=4)
    y_ref = po.run(m, x, [256, 256], "stream")
    assert np.array_equal(y_sharded, y_ref)
    assert tmax == 2.0


def test_ranges():
    assert list(weak_range(4, 2)) == [8, 9, 10, 11]
    parts = [strong_range(16384, 8, r) for r in range(8)]
    assert sum(len(p) for p in parts) == 16384 and parts[-1].stop == 16384
    parts = [strong_range(10, 4, r) for r in range(4)]
    assert [len(p) for p in parts] == [3, 3, 2, 2] and parts[1].start == 3


import pytest  # noqa: E402


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,total,world,parts", [(3, 37, 4, [512, 512]), (5, 13, 8, [2048, 2048]), (2, 9, 2, [256, 256])])
def test_product_shards_equal_unsharded_gpu(cfg, total, world, parts):
    """The PRODUCT on every rank's shard (ranks run one after another on the one GPU a test box
    has: shards never exchange data, so their order is immaterial) equals the unsharded batch
    bit for bit — the strong-scaling split of bench.py --total-streams."""
    from paper_2204_07064_b200 import configs
    from test_gpu_parity import run_gpu
    m = configs.build(cfg, seed=9)
    x = configs.batch_input(cfg, range(total), m.in_channels, sum(parts), seed=9)
    y_full, plan, _ = run_gpu(m, x, parts)
    ys = []
    for r in range(world):
        rg = strong_range(total, world, r)
        if len(rg) == 0:
            continue
        xr = configs.batch_input(cfg, rg, m.in_channels, sum(parts), seed=9)
        assert np.array_equal(xr, x[rg.start:rg.stop])  # inputs are seeded by global stream index
        y, _, _ = run_gpu(m, xr, parts, plan=plan)
        ys.append(y)
    assert np.array_equal(np.concatenate(ys), y_full)
