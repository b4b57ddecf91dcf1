#!/usr/bin/env python
"""Runs one workload of the sweep (for ncu captures and per-kernel timing).

  python scripts/run_case.py --case ffn|qk|pv|conv:<layer-name>|gemm:M,N,K [--iters N] [--bn 256]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W

    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="ffn")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--raster", type=int, default=0)
    ap.add_argument("--grid", type=int, default=0)
    ap.add_argument("--nchw", action="store_true")
    ap.add_argument("--bm", type=int, default=128)
    ap.add_argument("--sk", type=int, default=1)
    ap.add_argument("--bt", action="store_true", help="store B K-major (transposed)")
    ap.add_argument("--f32out", action="store_true")
    ap.add_argument("--math", default="auto", help="auto | bf16 | tf32 | fp32_simt | halo")
    ap.add_argument("--trace", action="store_true", help="print the per-tile role timeline of CTA 0/1")
    ap.add_argument("--gap", action="store_true", help="globaltimer gap between two graph-chained launches")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    rnd = lambda s, dt=torch.bfloat16: torch.empty(s, device=dev).uniform_(-1, 1).to(dt)
    cfg = ScheduleConfig(block_m=a.bm, block_n=a.bn or 128, stages=a.stages, raster=a.raster, grid=a.grid, split_k=a.sk,
                         math=a.math)
    if a.case == "ffn":
        T = W.BERT_TOKENS
        cfg.block_n = a.bn or 256
        ins = [rnd((T, 768)), rnd((768, 3072)), rnd((3072,)), rnd((3072, 768)), rnd((768,))]
        outs = [torch.empty((T, 768), device=dev, dtype=torch.bfloat16)]
        dag, flops = W.ffn_dag(T), 4.0 * T * 768 * 3072
    elif a.case.startswith("gemm:"):
        m, n, k = map(int, a.case[5:].split(","))
        bmat = rnd((n, k)).t() if a.bt else rnd((k, n))
        ins = [rnd((m, k)), bmat, rnd((n,))]
        outs = [torch.empty((m, n), device=dev, dtype=torch.float32 if a.f32out else torch.bfloat16)]
        dag, flops = W.matmul_bias_relu_dag(m, n, k), 2.0 * m * n * k
    elif a.case in ("qk", "pv"):
        H = W.BERT_HEADS
        if a.case == "qk":
            ins = [rnd((H, 128, 64)), rnd((H, 128, 64))]
            outs = [torch.empty((H, 128, 128), device=dev, dtype=torch.bfloat16)]
            dag = W.attention_scores_dag(H)
        else:
            ins = [rnd((H, 128, 128)), rnd((H, 128, 64))]
            outs = [torch.empty((H, 128, 64), device=dev, dtype=torch.bfloat16)]
            dag = W.attention_context_dag(H)
        flops = 2.0 * H * 128 * 128 * 64
    else:
        name = a.case.split(":", 1)[1]
        L = next(x for x in W.RESNET50 if x.name == name)
        B = W.RESNET_BATCH
        cl = not a.nchw
        fmt = torch.channels_last if cl else torch.contiguous_format
        if L.c < 8 and cl:  # padded channels-last view (NHWC4 for C <= 4, else NHWC8), as bench.py
            cp = 4 if L.c <= 4 else 8
            xb = torch.zeros((B, L.h, L.h, cp), device=dev, dtype=torch.bfloat16)
            xb[..., :L.c] = rnd((B, L.h, L.h, L.c))
            x0 = xb.as_strided((B, L.c, L.h, L.h), (L.h * L.h * cp, 1, L.h * cp, cp))
        else:
            x0 = rnd((B, L.c, L.h, L.h)).contiguous(memory_format=fmt)
        ins = [x0,
               rnd((L.f, L.c, L.k, L.k)).contiguous(memory_format=fmt), rnd((L.f,), torch.float32),
               rnd((L.f,), torch.float32)]
        ho = L.out_hw()
        outs = [torch.empty((B, L.f, ho, ho), device=dev, dtype=torch.bfloat16).contiguous(memory_format=fmt)]
        dag, flops = W.conv_bn_relu_dag(L, B), L.flops(B)
        if not a.bn:
            cfg.block_n = 256 if L.f >= 256 else (128 if L.f >= 128 else 64)
    if a.trace or a.gap:
        os.environ["TMB_TRACE"] = "1"
    plan = Plan(dag, cfg)
    ex = plan.bind(ins, outs)
    if a.gap:
        import numpy as np
        from paper_2210_09603_b200 import Graph
        exs = [ex] + [plan.bind(ins, outs) for _ in range(3)]
        g = Graph(exs)
        for _ in range(3):
            g.launch()
        torch.cuda.synchronize()
        prev = None
        for j, e in enumerate(exs):
            tr = e.trace(0)
            st, su, en = (tr[:, 0, k].astype(np.int64) for k in (7, 14, 15))
            dl = tr[:, 1, 15].astype(np.int64)
            if j == len(exs) - 1:
                arr = tr[:, 2:15, 15].astype(np.int64)  # per-warp arrival at the final barrier
                print("  warp arrival at final barrier, CTA 0 (us after entry):",
                      " ".join(f"{(x - st[0]) / 1e3:.2f}" for x in arr[0]))
                print(f"  CTA 0: exit {(en[0] - st[0]) / 1e3:.2f}, MMA warp past barrier "
                      f"{(tr[0, 1, 14] - st[0]) / 1e3:.2f}, dealloc done {(dl[0] - st[0]) / 1e3:.2f}")
            line = (f"launch {j}: entry span {(st.max() - st.min()) / 1e3:.2f} us, life {(en.max() - st.min()) / 1e3:.2f} us,"
                    f" dealloc done +{(dl.max() - en.max()) / 1e3:.2f} us after the last exit")
            if prev is not None:
                line += f"  | gap from previous last exit to first entry {(st.min() - prev) / 1e3:.2f} us"
            prev = en.max()
            print(line)
    for _ in range(3):
        ex.launch()
    torch.cuda.synchronize()
    # a CUDA graph of `iters` back-to-back launches: device time without host launch cost
    from paper_2210_09603_b200 import Graph
    g = Graph([ex] * a.iters)
    g.launch()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.launch()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    if a.trace:
        import numpy as np
        ex.launch()
        torch.cuda.synchronize()
        tr = ex.trace(0)
        names = ["prodF", "prodL", "mmaF", "mmaL", "epiRdy", "epiAcc", "epiDone", "-", "ld0", "ldback", "bufok",
                 "staged", "stored", "staged1", "-"]
        for cta in (0, 1, tr.shape[0] - 1):
            print(f"CTA {cta} (cycles):")
            for i in range(64):
                row = tr[cta, i, :15].copy()
                row[7] = 0
                if not row.any():
                    continue
                print(f"  tile {i:2d} " + " ".join(f"{n}={v:7d}" for n, v in zip(names, row)))
        done = tr[:, :, 6]
        span = done.max(axis=1)
        mma = np.where(tr[:, :, 3] > 0, tr[:, :, 3] - tr[:, :, 2], 0)
        epi = np.where(tr[:, :, 6] > 0, tr[:, :, 6] - tr[:, :, 5], 0)
        st, su, en = (tr[:, 0, j].astype(np.int64) for j in (7, 14, 15))
        print(f"globaltimer: CTA entry spread {(st.max() - st.min()) / 1e3:.2f} us; setup median "
              f"{np.median(su - st) / 1e3:.2f} us; CTA life median {np.median(en - st) / 1e3:.2f} us, "
              f"first entry -> last exit {(en.max() - st.min()) / 1e3:.2f} us")
        print(f"CTA span cycles: min {span.min()} median {np.median(span):.0f} max {span.max()}; "
              f"per-tile MMA issue span mean {mma[mma > 0].mean():.0f}; epilogue mean {epi[epi > 0].mean():.0f}")
    print(json.dumps({"case": a.case, "ms": ms, "tflops": flops / ms / 1e9, "launches": ex.num_launches,
                      "kernel": ex.kernel_info(0),
                      "plan": plan.describe()["kernels"][0]["A"] + " x " + plan.describe()["kernels"][0]["B"]}))


if __name__ == "__main__":
    main()
