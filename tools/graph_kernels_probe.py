"""Kernel nodes of the captured c3 training-step graph (ours vs all): python tools/graph_kernels_probe.py"""
import sys, torch
sys.path.insert(0, '.')
import bench
import paper_1412_4526_b200 as dp
from paper_1412_4526_b200.engine import DenseNet, graph_kernel_nodes, ops
from paper_1412_4526_b200.trainer import DataParallelTrainer
text, side, B, mf, _ = bench.CONFIGS["c3"]
plan = dp.compile_plan(dp.parse_spec(text))
tr = DataParallelTrainer(plan, 2, side, side, lr=1e-12, use_graph=True)
imgs, tgts, masks = [t.cuda() for t in bench._synthetic(dp.parse_spec(text), 2, side, mf, 1, "cuda")]
tr.load_batch(imgs, tgts, masks); tr.step(); torch.cuda.synchronize()
print("graph kernels (exact):", tr.graph_kernel_count)
from cuda.bindings import runtime as rt
g = tr._graph
err, _, n = rt.cudaGraphGetNodes(rt.cudaGraph_t(init_value=g.raw_cuda_graph()), 0)
print("all nodes", n)
from cuda.bindings import driver as drv
graph = drv.CUgraph(init_value=g.raw_cuda_graph())
err, _, n = drv.cuGraphGetNodes(graph, 0)
err, nodes, n = drv.cuGraphGetNodes(graph, n)
from collections import Counter
names = Counter()
for nd in nodes[:n]:
    err, kind = drv.cuGraphNodeGetType(nd)
    if kind == drv.CUgraphNodeType.CU_GRAPH_NODE_TYPE_KERNEL:
        err2, params = drv.cuGraphKernelNodeGetParams(nd)
        err3, name = drv.cuFuncGetName(params.func)
        names[(name.decode() if isinstance(name, bytes) else str(name))[:60]] += 1
for k_, v in names.most_common():
    print(v, k_)
print("engine count", graph_kernel_nodes(g))
