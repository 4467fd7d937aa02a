"""Data-parallel host logic on CPU: world_size 2 over gloo (no GPU needed).

Each rank takes its image shard (trainer.shard), computes its summed gradient
with the oracle (standing in for the per-rank engine), packs it into the flat
bucket (trainer.flatten), and runs the trainer's all-reduce (SUM).  The
all-reduced bucket must equal the single-process gradient sum over all images
(unweighted-sum semantics, reference backward.py:190-191) -- SURVEY.md 8(e).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

SPEC = ("input channels=2\n"
        "conv out=3 in=2 k=3 stride=1 weights=seed:7\n"
        "pool kind=max k=2 stride=2\nnonlin kind=relu\n"
        "conv out=2 in=3 k=2 stride=1 weights=seed:8\n")
N_IMAGES, SIDE = 5, 9


def _data():
    rng = np.random.default_rng(11)
    imgs = rng.uniform(-0.5, 0.5, (N_IMAGES, 2, SIDE, SIDE))
    deltas = rng.uniform(-1, 1, (N_IMAGES, 2, SIDE, SIDE))
    masks = rng.random((N_IMAGES, SIDE, SIDE)) < 0.3
    return imgs, deltas, masks


def _grads_for(indices):
    from oracle import engine_np
    from oracle.netdesc import read_spec

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    net = read_spec(SPEC)
    spec = dp.parse_spec(SPEC)
    imgs, deltas, masks = _data()
    total = np.zeros(trainer.bucket_layout(spec)[1])
    for i in indices:
        cache = engine_np.dense_forward(net, imgs[i])
        kg, bg, _ = engine_np.dense_backward(net, cache, deltas[i], masks[i])
        total += trainer.flatten(spec, kg, bg)
    return total


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1412_4526_b200 import trainer
    mine = trainer.shard(N_IMAGES, rank, world)
    bucket = torch.from_numpy(_grads_for(mine))
    trainer.allreduce_sum(bucket)
    if rank == 0:
        np.save(out_path, bucket.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_allreduced_bucket_equals_single_process_sum(tmp_path):
    out = str(tmp_path / "bucket.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    got = np.load(out)
    want = _grads_for(range(N_IMAGES))
    assert np.max(np.abs(got - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))


def test_shards_partition_images():
    from paper_1412_4526_b200 import trainer
    for world in (1, 2, 3, 8):
        seen = [i for r in range(world) for i in trainer.shard(N_IMAGES, r, world)]
        assert seen == list(range(N_IMAGES))


def test_allreduce_is_noop_without_process_group():
    from paper_1412_4526_b200 import trainer
    t = torch.arange(4.0)
    assert torch.equal(trainer.allreduce_sum(t.clone()), t)
