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


# ---------------------------------------------------------------- band sharding
# SURVEY.md 8(e) fallback: fewer images than ranks -> each rank takes an output-row band
# of one image plus its (patch - 1)-row halo of padded input.

BAND_IMAGES, BAND_SIDE = 1, 13


def _band_data():
    rng = np.random.default_rng(5)
    imgs = rng.uniform(-0.5, 0.5, (BAND_IMAGES, 2, BAND_SIDE, BAND_SIDE))
    deltas = rng.uniform(-1, 1, (BAND_IMAGES, 2, BAND_SIDE, BAND_SIDE))
    masks = rng.random((BAND_IMAGES, BAND_SIDE, BAND_SIDE)) < 0.4
    return imgs, deltas, masks


def _band_grads(rank, world):
    """This rank's band: oracle forward on the padded band rows, masked backward with the
    band's rows of delta and mask; returns (flat bucket, band output or None)."""
    from oracle import engine_np
    from oracle.netdesc import read_spec

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    net = read_spec(SPEC)
    spec = dp.parse_spec(SPEC)
    imgs, deltas, masks = _band_data()
    a = trainer.band_assignment(BAND_IMAGES, BAND_SIDE, rank, world)
    if a is None:
        return np.zeros(trainer.bucket_layout(spec)[1]), None
    img, r0, r1 = a
    rin, rout = trainer.band_rows(r0, r1, dp.patch_size(spec))
    x0 = engine_np.pad_image(net, imgs[img])
    cache = engine_np.dense_forward(net, x0[:, rin], padded=True)
    kg, bg, _ = engine_np.dense_backward(net, cache, deltas[img][:, rout], masks[img][rout])
    return trainer.flatten(spec, kg, bg), cache.output


def _band_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1412_4526_b200 import trainer
    flat, _ = _band_grads(rank, world)
    bucket = torch.from_numpy(flat)
    trainer.allreduce_sum(bucket)
    if rank == 0:
        np.save(out_path, bucket.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_band_sharded_gradients_equal_full_image(tmp_path, world):
    from oracle import engine_np
    from oracle.netdesc import read_spec

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    out = str(tmp_path / "bucket.npy")
    mp.spawn(_band_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    net = read_spec(SPEC)
    imgs, deltas, masks = _band_data()
    cache = engine_np.dense_forward(net, imgs[0])
    kg, bg, _ = engine_np.dense_backward(net, cache, deltas[0], masks[0])
    want = trainer.flatten(dp.parse_spec(SPEC), kg, bg)
    assert np.max(np.abs(got - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))


def test_band_outputs_tile_the_full_map():
    from oracle import engine_np
    from oracle.netdesc import read_spec
    net = read_spec(SPEC)
    imgs, _, _ = _band_data()
    full = engine_np.dense_forward(net, imgs[0]).output
    for world in (2, 3, 4):
        parts = [_band_grads(r, world)[1] for r in range(world)]
        got = np.concatenate([p for p in parts if p is not None], axis=1)
        assert np.array_equal(got, full)


def test_band_assignment_partitions_rows():
    from paper_1412_4526_b200 import trainer
    for n_img, world, h in ((1, 2, 13), (1, 8, 100), (2, 8, 64), (3, 8, 50)):
        rows = {}
        for r in range(world):
            a = trainer.band_assignment(n_img, h, r, world)
            if a is None:
                continue
            img, r0, r1 = a
            rows.setdefault(img, []).extend(range(r0, r1))
        assert sorted(rows) == list(range(n_img))
        for img in rows:
            assert rows[img] == list(range(h))
    with pytest.raises(ValueError):
        trainer.band_assignment(4, 10, 0, 2)


def test_band_assignment_more_ranks_than_rows():
    """bands never empty when height < world // n_images."""
    from paper_1412_4526_b200 import trainer
    for n_img, world, h in ((1, 8, 3), (2, 8, 1), (1, 5, 4)):
        got = [trainer.band_assignment(n_img, h, r, world) for r in range(world)]
        live = [a for a in got if a is not None]
        assert all(r1 > r0 for _, r0, r1 in live)
        for img in range(n_img):
            rows = sorted(y for i, r0, r1 in live if i == img for y in range(r0, r1))
            assert rows == list(range(h))


def _subgroup_worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1412_4526_b200 import trainer
    group = dist.new_group([1, 2])           # a subgroup without global rank 0
    t = torch.full((4,), float(rank + 10))
    if rank in (1, 2):
        assert trainer.group_root(group) == 1
        trainer.broadcast_params(t, group)
        trainer.allreduce_sum(t, group)
        np.save(f"{out_path}.{rank}.npy", t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_subgroup_broadcast_uses_group_first_member(tmp_path):
    """the initial-weight broadcast on a subgroup comes from the group's first
    member (global rank 1 here), not global rank 0, and does not raise."""
    out = str(tmp_path / "t")
    mp.spawn(_subgroup_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    for r in (1, 2):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), np.full(4, 22.0))
