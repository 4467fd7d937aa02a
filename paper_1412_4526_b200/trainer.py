"""Image-sharded data-parallel trainer (NCCL all-reduce over NVLink / NVSwitch).

Images are independent units: each rank runs the fused dense
engine on its shard, sums its GradientSet locally (the engine's flat gradient
bucket), then ONE `all_reduce(SUM)` of that bucket per step.  SUM keeps the
reference's unweighted-sum gradient semantics (backward.py:190-191,
SPEC.md:446), so the all-reduced bucket equals the single-process GradientSet
of all images.  Forward-only inference shards images with no collective.

The bucket layout is the conv layers in plan order, weights then bias each,
flattened -- `bucket_layout()` / `flatten()` / `unflatten()` below, shared by
the engine (engine.DenseNet.grad_flat) and the CPU gloo tests.
"""

from __future__ import annotations

import numpy as np

from .netspec import ConvLayerSpec, NetworkSpec
from .plan import DensePlan


def bucket_layout(spec: NetworkSpec):
    """[(layer_index, w_shape, b_shape, offset)] for the flat gradient bucket."""
    out, off = [], 0
    for k, layer in enumerate(spec.layers):
        if isinstance(layer, ConvLayerSpec):
            out.append((k, tuple(layer.weights.shape), tuple(layer.bias.shape), off))
            off += layer.weights.size + layer.bias.size
    return out, off


def flatten(spec: NetworkSpec, kernels, biases, dtype=np.float64) -> np.ndarray:
    layout, total = bucket_layout(spec)
    flat = np.zeros(total, dtype=dtype)
    for k, ws, bs, off in layout:
        nw = int(np.prod(ws))
        flat[off:off + nw] = np.asarray(kernels[k]).ravel()
        flat[off + nw:off + nw + int(np.prod(bs))] = np.asarray(biases[k]).ravel()
    return flat


def unflatten(spec: NetworkSpec, flat):
    """flat bucket -> (kernel list, bias list) aligned with spec.layers (None elsewhere)."""
    flat = np.asarray(flat)
    layout, _ = bucket_layout(spec)
    ks = [None] * len(spec.layers)
    bs = [None] * len(spec.layers)
    for k, wshape, bshape, off in layout:
        nw, nb = int(np.prod(wshape)), int(np.prod(bshape))
        ks[k] = flat[off:off + nw].reshape(wshape).copy()
        bs[k] = flat[off + nw:off + nw + nb].reshape(bshape).copy()
    return ks, bs


def shard(n_images: int, rank: int, world: int) -> range:
    """Contiguous image shard of this rank (balanced, deterministic)."""
    base, extra = divmod(n_images, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def band_assignment(n_images: int, height: int, rank: int, world: int):
    """Fallback when images < ranks: spatial band sharding.

    Ranks are split into n_images groups of `per = world // n_images`; rank r takes image
    r // per and the balanced band (r % per) of its output rows.  Returns
    (image, r0, r1) -- output rows [r0, r1) -- or None for the ranks left over (world %
    n_images, plus any beyond `height` bands per image), which contribute an all-zero
    bucket.  An output row depends on the padded
    input rows [row, row + patch - 1] only (valid convolutions on the padded image,
    forward.py:96-98), so a band is computed exactly from padded rows [r0, r1 + patch - 1)
    (the (patch - 1)-row halo) and band gradients, with the mask restricted to the band,
    sum to the full image's (unweighted-sum semantics, backward.py:190-191)."""
    if n_images >= world:
        raise ValueError("band sharding is the fallback for fewer images than ranks")
    per = min(world // n_images, height)  # every band keeps >= 1 output row
    if rank >= per * n_images:
        return None
    img, band = divmod(rank, per)
    r0 = band * height // per
    r1 = (band + 1) * height // per
    return img, r0, r1


def band_rows(r0: int, r1: int, patch: int):
    """(padded-input rows, output rows) of a band as slices."""
    return slice(r0, r1 + patch - 1), slice(r0, r1)


def group_root(group=None) -> int:
    """Global rank of the first member of `group` (the broadcast source of the initial
    weights); 0 for the default group.  dist.broadcast's `src` is a GLOBAL rank."""
    import torch.distributed as dist
    if group is None or group is dist.group.WORLD:
        return 0
    return dist.get_global_rank(group, 0)


def broadcast_params(tensor, group=None):
    """Every member of `group` starts from the group's first member's weights."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if tensor.is_cuda and dist.get_backend(group) != "nccl":
            # gloo: through a host copy, so no device write lands after later kernels
            host = tensor.cpu()
            dist.broadcast(host, src=group_root(group), group=group)
            tensor.copy_(host)
        else:
            dist.broadcast(tensor, src=group_root(group), group=group)
    return tensor


def allreduce_sum(tensor, group=None):
    """In-place SUM all-reduce of the gradient bucket (no-op when not distributed).

    NCCL is stream-ordered on the tensor's device.  Other backends (gloo: the CPU tests, and
    ranks sharing one GPU) reduce a host copy, so the result is in place before the next
    kernel on the current stream (the SGD update) reads it."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        if tensor.is_cuda and dist.get_backend(group) != "nccl":
            host = tensor.cpu()
            dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
            tensor.copy_(host)
        else:
            dist.all_reduce(tensor, op=dist.ReduceOp.SUM, group=group)
    return tensor


class DataParallelTrainer:
    """One DenseNet per rank + bucket all-reduce + SGD, optionally as one CUDA graph.

    With NCCL the all-reduce (and the SGD update) are captured INSIDE the step's CUDA graph:
    one graph launch per step runs forward, masked backward, the NCCL all-reduce of the
    gradient bucket and the update, with no host round trip between them (the communicator
    is brought up by a warm-up all-reduce before capture).  Other backends (gloo: CPU tests,
    ranks sharing a GPU) cannot be captured: the all-reduce then follows the graph replay on
    the same stream (`allreduce_sum`).  DP_ALLREDUCE_OUTSIDE=1 forces that order with NCCL
    too; DP_FORCE_ALLREDUCE=1 runs the collective even at world size 1 (single-GPU tests of
    the captured NCCL path).
    """

    def __init__(self, plan: DensePlan, batch_per_rank: int, height: int, width: int,
                 lr: float = 0.0, group=None, dtype=None, use_graph: bool = True,
                 precision: str = "fast"):
        import os

        import torch
        import torch.distributed as dist

        from .engine import DenseNet
        self.net = DenseNet(plan, batch_per_rank, height, width, dtype=dtype, train=True,
                            precision=precision)
        self.group = group
        self.lr = lr
        self.distributed = dist.is_available() and dist.is_initialized()
        # every rank starts from the group's first member's weights (seeded specs agree)
        broadcast_params(self.net.param_flat, group)
        force = bool(os.environ.get("DP_FORCE_ALLREDUCE"))
        self.collective = self.distributed and (dist.get_world_size(group) > 1 or force)
        self.nccl = self.collective and dist.get_backend(group) == "nccl"
        self.in_graph = (use_graph and self.nccl and
                         not os.environ.get("DP_ALLREDUCE_OUTSIDE"))
        self._graph = None
        self._use_graph = use_graph
        self._torch = torch

    def load_batch(self, images, targets, masks):
        n = self.net
        n.set_input(images)
        n.target.copy_(targets)
        n.mask.copy_(masks)

    def _compute(self):
        n = self.net
        n.forward(prepare_backward=True)
        n.loss_delta()
        n.backward()

    def _reduce(self):
        import torch.distributed as dist
        if self.nccl:
            dist.all_reduce(self.net.grad_flat, op=dist.ReduceOp.SUM, group=self.group)
        elif self.collective:
            allreduce_sum(self.net.grad_flat, self.group)

    def _compute_reduce_update(self):
        self._compute()
        self._reduce()
        if self.lr:
            self.net.sgd_step(self.lr)

    def step(self):
        """forward + masked loss + backward [+ all-reduce] [+ SGD] on the loaded batch."""
        if self._use_graph and self.in_graph:
            if self._graph is None:
                self._reduce()  # communicator up (and warm) before capture
                # capture() runs the step eagerly to warm up: keep the parameters it updates
                keep = self.net.param_flat.clone()
                self._graph = self.net.capture(self._compute_reduce_update)
                self.net.param_flat.copy_(keep)
            self._graph.replay()
            return
        if self._use_graph:
            if self._graph is None:
                self._graph = self.net.capture(self._compute)
            self._graph.replay()
        else:
            self._compute()
        self._reduce()
        if self.lr:
            self.net.sgd_step(self.lr)

    @property
    def graph_kernel_count(self) -> int:
        return getattr(self.net, "graph_kernels", 0)

    def forward_only(self):
        self.net.forward()
        return self.net.output


class H2DPipeline:
    """Double-buffered host -> device input pipeline for `DataParallelTrainer`.

    `submit(images, targets, masks)` copies a batch from pinned host memory into one of
    two device staging slots on a dedicated copy stream; `step()` makes the compute
    stream wait for the oldest submitted batch, loads it into the engine and runs one
    training step.  Submitting batch s+1 before stepping batch s overlaps the H2D
    transfer with the step's kernels.  A slot is reused only after the step that read
    it has finished (event), so no batch is overwritten in flight.
    """

    def __init__(self, trainer, images_like, targets_like, masks_like):
        import torch
        self._torch = torch
        self.tr = trainer
        dev = trainer.net.device
        self.slots = [tuple(torch.empty(t.shape, dtype=t.dtype, device=dev)
                            for t in (images_like, targets_like, masks_like)) for _ in range(2)]
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        self._free_recorded = [False, False]
        self._submitted = 0
        self._consumed = 0

    def submit(self, images, targets, masks):
        torch = self._torch
        k = self._submitted % 2
        if self._submitted - self._consumed >= 2:
            raise RuntimeError("H2DPipeline: both slots hold unconsumed batches")
        with torch.cuda.stream(self.copy_stream):
            if self._free_recorded[k]:
                self.copy_stream.wait_event(self.free[k])
            for dst, src in zip(self.slots[k], (images, targets, masks)):
                dst.copy_(src, non_blocking=True)
            self.ready[k].record(self.copy_stream)
        self._submitted += 1

    def step(self):
        torch = self._torch
        if self._consumed >= self._submitted:
            raise RuntimeError("H2DPipeline: step() without a submitted batch")
        k = self._consumed % 2
        cur = torch.cuda.current_stream()
        cur.wait_event(self.ready[k])
        self.tr.load_batch(*self.slots[k])
        self.free[k].record(cur)
        self._free_recorded[k] = True
        self.tr.step()
        self._consumed += 1


class BandParallelTrainer:
    """Fewer images than ranks: each rank runs the engine on one (image, output-row band)
    with its (patch - 1)-row halo of padded input (band_assignment), then the same SUM
    all-reduce of the gradient bucket as DataParallelTrainer.  Forward-only inference
    needs no collective: each rank's band output is a disjoint slice of the image's map."""

    def __init__(self, plan: DensePlan, n_images: int, height: int, width: int,
                 rank: int = 0, world: int = 1, lr: float = 0.0, group=None, dtype=None,
                 precision: str = "fast"):
        from .engine import DenseNet
        from .netspec import patch_size
        self.patch = patch_size(plan.source)
        self.assign = band_assignment(n_images, height, rank, world)
        self.height, self.width = height, width
        self.group = group
        self.lr = lr
        rows = (self.assign[2] - self.assign[1]) if self.assign else 1
        self.net = DenseNet(plan, 1, rows, width, dtype=dtype, train=True, precision=precision)
        broadcast_params(self.net.param_flat, group)

    def load(self, padded_images, targets, masks):
        """padded_images: (N, C, h + patch - 1, w + patch - 1) device tensor (the engine's
        x0 layout for the whole batch); targets (N, Q, h, w); masks (N, h, w)."""
        n = self.net
        if self.assign is None:
            n.x0.zero_()
            n.mask.zero_()
            return
        img, r0, r1 = self.assign
        rin, rout = band_rows(r0, r1, self.patch)
        n.set_padded_input(padded_images[img:img + 1, :, rin])
        n.target.copy_(targets[img:img + 1, :, rout])
        n.mask.copy_(masks[img:img + 1, rout])

    def step(self):
        n = self.net
        n.forward()
        n.loss_delta()
        n.backward()
        allreduce_sum(n.grad_flat, self.group)
        if self.lr:
            n.sgd_step(self.lr)

    def forward_only(self):
        self.net.forward()
        return self.net.output
