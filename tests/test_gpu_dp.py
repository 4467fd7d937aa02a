"""DataParallelTrainer at world size 2 on the REAL engine (GPU).

Two processes share the one GPU of the box and talk over gloo (which all-reduces CUDA
tensors); each runs `DataParallelTrainer.step()` -- fused fast-tier engine, CUDA-graph
replay, bucket all-reduce(SUM), SGD -- on its image shard (`trainer.shard`).  The
all-reduced bucket must equal the single-process engine's gradient bucket over all images
(unweighted-sum semantics, reference backward.py:190-191), and after the
SGD update both ranks hold identical parameters.  NCCL refuses two ranks on one device, so
the collective here is gloo; the NCCL path is the same `allreduce_sum` call.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SPEC = ("input channels=3\n"
        "conv out=16 in=3 k=6 stride=1 weights=seed:1\n"
        "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
        "conv out=32 in=16 k=5 stride=1 weights=seed:2\n"
        "pool kind=max k=2 stride=2\nnonlin kind=tanh\n"
        "conv out=10 in=32 k=4 stride=1 weights=seed:3\n")
N_IMAGES, SIDE, LR = 4, 96, 1e-3


def _data():
    rng = np.random.default_rng(21)
    imgs = rng.uniform(-0.5, 0.5, (N_IMAGES, 3, SIDE, SIDE)).astype(np.float32)
    tgts = rng.uniform(-1, 1, (N_IMAGES, 10, SIDE, SIDE)).astype(np.float32)
    masks = (rng.random((N_IMAGES, SIDE, SIDE)) < 0.05).astype(np.uint8)
    return imgs, tgts, masks


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    plan = dp.compile_plan(dp.parse_spec(SPEC))
    mine = trainer.shard(N_IMAGES, rank, world)
    imgs, tgts, masks = _data()
    tr = trainer.DataParallelTrainer(plan, len(mine), SIDE, SIDE, lr=LR)
    sl = slice(mine.start, mine.stop)
    tr.load_batch(torch.from_numpy(imgs[sl]).cuda(), torch.from_numpy(tgts[sl]).cuda(),
                  torch.from_numpy(masks[sl]).cuda())
    tr.step()
    torch.cuda.synchronize()
    np.save(f"{out}.grad{rank}.npy", tr.net.grad_flat.double().cpu().numpy())
    np.save(f"{out}.param{rank}.npy", tr.net.param_flat.double().cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_trainer_step_equals_single_process(tmp_path):
    import torch
    import torch.multiprocessing as mp

    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200.engine import DenseNet
    out = str(tmp_path / "dp")
    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    g0, g1 = np.load(f"{out}.grad0.npy"), np.load(f"{out}.grad1.npy")
    p0, p1 = np.load(f"{out}.param0.npy"), np.load(f"{out}.param1.npy")
    assert np.array_equal(g0, g1) and np.array_equal(p0, p1)

    imgs, tgts, masks = _data()
    plan = dp.compile_plan(dp.parse_spec(SPEC))
    net = DenseNet(plan, N_IMAGES, SIDE, SIDE, train=True)
    p_init = net.param_flat.double().cpu().numpy()
    net.set_input(torch.from_numpy(imgs).cuda())
    net.target.copy_(torch.from_numpy(tgts))
    net.mask.copy_(torch.from_numpy(masks))
    net.forward()
    net.loss_delta()
    net.backward()
    torch.cuda.synchronize()
    want = net.grad_flat.double().cpu().numpy()
    scale = np.max(np.abs(want))
    assert np.max(np.abs(g0 - want)) <= 1e-5 * scale
    # fp32 rounding of the updated parameters (|p| reaches ~1e2 here: summed gradients ~1e5)
    assert np.max(np.abs(p0 - (p_init - LR * g0))) <= 1e-6 * max(1.0, np.max(np.abs(p0)))


def _nccl_worker(out, port):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), DP_FORCE_ALLREDUCE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import paper_1412_4526_b200 as dp
    from paper_1412_4526_b200 import trainer
    plan = dp.compile_plan(dp.parse_spec(SPEC))
    imgs, tgts, masks = (torch.from_numpy(a).cuda() for a in _data())
    res = {}
    for mode in ("graph", "eager"):
        tr = trainer.DataParallelTrainer(plan, N_IMAGES, SIDE, SIDE, lr=LR,
                                         use_graph=(mode == "graph"))
        assert tr.in_graph == (mode == "graph") and tr.nccl
        tr.load_batch(imgs, tgts, masks)
        tr.step()
        tr.step()  # second step starts from the first step's update
        torch.cuda.synchronize()
        res[mode] = (tr.net.grad_flat.double().cpu().numpy(),
                     tr.net.param_flat.double().cpu().numpy())
    np.savez(out, gg=res["graph"][0], pg=res["graph"][1], ge=res["eager"][0],
             pe=res["eager"][1])
    dist.destroy_process_group()


def test_nccl_allreduce_and_sgd_captured_in_graph(tmp_path):
    """The NCCL path captures the all-reduce and the SGD update inside the step's CUDA graph
    (one graph launch per step).  World size 1 (one GPU per box) with the collective forced
    on: two graph-replayed steps give the same gradients and parameters as two eager steps
    (the capture's warm-up updates are rolled back)."""
    import torch.multiprocessing as mp
    out = str(tmp_path / "nccl.npz")
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_nccl_worker, args=(out, _free_port()))
    p.start()
    p.join(600)
    assert p.exitcode == 0
    r = np.load(out)
    assert np.array_equal(r["gg"], r["ge"])
    assert np.array_equal(r["pg"], r["pe"])
