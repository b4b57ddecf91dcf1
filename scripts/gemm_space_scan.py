import sys, os, json
sys.path.insert(0, '/root/repo')
import torch
from paper_2210_09603_b200 import Plan, Graph, schedule_space, workloads as W
dev = torch.device('cuda', 0)
rnd = lambda s, dt=torch.bfloat16: torch.empty(s, device=dev).uniform_(-1, 1).to(dt)
for (m, n, k) in [(8192, 768, 3072), (8192, 3072, 768)]:
    ins = [rnd((m, k)), rnd((k, n)), rnd((n,))]
    outs = [torch.empty((m, n), device=dev, dtype=torch.bfloat16)]
    dag = W.matmul_bias_relu_dag(m, n, k)
    res = []
    for cfg in schedule_space('matmul'):
        ex = Plan(dag, cfg).bind(ins, outs)
        g = Graph([ex] * 10); g.launch(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.launch(); e1.record(); torch.cuda.synchronize()
        res.append((e0.elapsed_time(e1) / 10 * 1e3, f"bm{cfg.block_m} bn{cfg.block_n} sk{cfg.split_k} st{cfg.stages} r{cfg.raster}"))
    res.sort()
    print(m, n, k, res[:6])
