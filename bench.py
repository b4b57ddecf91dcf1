#!/usr/bin/env python
"""Benchmark of the fused task-mapped GEMM / implicit-GEMM conv path on B200.

One step = one batch-sharded sweep of BASELINE.json configs[4] on every rank:
  * the 53 ResNet-50 conv layers as implicit GEMM with the
    fused BN-fold + ReLU epilogue, batch 32 per GPU, bf16, channels-last;
  * the BERT-base FFN chain (8192 tokens = batch 64 x seq 128, 768->3072 GELU
    ->768 + residual), bf16;
  * the BERT-base attention batched matmuls (12x16 = 192 heads, seq 128, d 64):
    S = 0.125 Q K^T and O = S V, bf16;
then the step's result tensors are gathered to rank 0 (the only collective).
value = algorithmic FLOPs of all ranks / max-over-ranks step time (weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused GEMM/conv TFLOP/s & % tensor peak at 1/2/4/8 B200 vs ref CPU"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops", 1590.0), d.get("hbm_gbs", 6650.0), "measured"
    return 1590.0, 6650.0, "fallback"


# ------------------------------------------------------------------ clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- workload --
def cfg_str(cfg):
    return f"bm{cfg.block_m}/bn{cfg.block_n}/sk{cfg.split_k}/{'deep' if cfg.pipeline else 'db'}/r{cfg.raster}"


def build_sweep(torch, device, seed=0, tuner=None, tune_mode="auto", log=None):
    """Allocates inputs/weights/outputs of one sweep and binds the fused plans.
    Each distinct workload is tuned over schedule_space on the device (or its
    cached best config is reused); returns (items, tuning report)."""
    from paper_2210_09603_b200 import Plan, ScheduleConfig, workloads as W

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    treport = {"tuned": 0, "cached": 0, "seconds": 0.0, "configs": {}}

    def rnd(shape, dtype=torch.bfloat16, cl=False):
        t = torch.empty(shape, device=device, dtype=torch.float32).uniform_(-1, 1, generator=g).to(dtype)
        return t.contiguous(memory_format=torch.channels_last) if cl else t

    def conv_input(L, B):
        if L.c < 8:  # 16-byte padded channels-last (NHWC8): the TMA-able layout for C < 8
            xb = torch.zeros((B, L.h, L.h, 8), device=device, dtype=torch.bfloat16)
            xb[..., :L.c] = rnd((B, L.h, L.h, L.c))
            return xb.as_strided((B, L.c, L.h, L.h), (L.h * L.h * 8, 1, L.h * 8, 8))
        return rnd((B, L.c, L.h, L.h), cl=True)

    def pick(key, dag, ins, outs, default):
        if tuner is None or tune_mode == "off":
            return default
        cfg, secs, cached = tuner.tune(key, dag, ins, outs, force=(tune_mode == "force"))
        treport["seconds"] += secs
        treport["tuned" if not cached else "cached"] += 1
        treport["configs"][key] = cfg_str(cfg)
        if log:
            log(f"{key}: {treport['configs'][key]} ({'cached' if cached else f'tuned in {secs:.1f}s'})")
        return cfg

    items = []  # (name, group, flops, exec, inputs(list), outputs(list), result?)
    B = W.RESNET_BATCH
    for L in W.RESNET50:
        dag = W.conv_bn_relu_dag(L, B)
        ho = L.out_hw()
        plan = None
        for rep in range(L.count):
            x = conv_input(L, B)
            w = rnd((L.f, L.c, L.k, L.k), cl=True)
            scale = rnd((L.f,), torch.float32)
            shift = rnd((L.f,), torch.float32)
            z = torch.empty((B, L.f, ho, ho), device=device, dtype=torch.bfloat16).contiguous(
                memory_format=torch.channels_last)
            if plan is None:
                default = ScheduleConfig(block_n=256 if L.f >= 256 else (128 if L.f >= 128 else 64))
                cfg = pick(f"conv:{L.name}:b{B}:nhwc", dag, [x, w, scale, shift], [z], default)
                plan = Plan(dag, cfg)
            ex = plan.bind([x, w, scale, shift], [z])
            items.append(dict(name=f"{L.name}#{rep}", group="conv", flops=L.flops(B), exec=ex, inputs=[x],
                              outputs=[z], plan=plan, cfg=cfg_str(cfg)))
    # FFN chain
    T = W.BERT_TOKENS
    dag = W.ffn_dag(T)
    x = rnd((T, W.BERT_HIDDEN))
    ffn_in = [x, rnd((W.BERT_HIDDEN, W.BERT_FFN)), rnd((W.BERT_FFN,)), rnd((W.BERT_FFN, W.BERT_HIDDEN)),
              rnd((W.BERT_HIDDEN,))]
    o = torch.empty((T, W.BERT_HIDDEN), device=device, dtype=torch.bfloat16)
    plan = Plan(dag, pick(f"ffn:t{T}", dag, ffn_in, [o], ScheduleConfig(block_m=256, block_n=256)))
    items.append(dict(name="bert.ffn", group="ffn", flops=2.0 * T * W.BERT_HIDDEN * W.BERT_FFN * 2,
                      exec=plan.bind(ffn_in, [o]), inputs=[x], outputs=[o], plan=plan, result=True))
    # attention batched matmuls
    H, S, D = W.BERT_HEADS, W.BERT_SEQ, W.BERT_HEAD_DIM
    q, k, v = rnd((H, S, D)), rnd((H, S, D)), rnd((H, S, D))
    s = torch.empty((H, S, S), device=device, dtype=torch.bfloat16)
    dag1 = W.attention_scores_dag(H)
    p1 = Plan(dag1, pick(f"attn.qk:h{H}", dag1, [q, k], [s], ScheduleConfig(block_n=128)))
    items.append(dict(name="bert.qk", group="attn", flops=2.0 * H * S * S * D, exec=p1.bind([q, k], [s]),
                      inputs=[q, k], outputs=[s], plan=p1))
    oc = torch.empty((H, S, D), device=device, dtype=torch.bfloat16)
    dag2 = W.attention_context_dag(H)
    p2 = Plan(dag2, pick(f"attn.pv:h{H}", dag2, [s, v], [oc], ScheduleConfig(block_n=64)))
    items.append(dict(name="bert.pv", group="attn", flops=2.0 * H * S * S * D, exec=p2.bind([s, v], [oc]),
                      inputs=[v], outputs=[oc], plan=p2, result=True))
    items[52]["result"] = True  # last conv layer (l4.ds) output
    return items, treport


def sweep_flops(items):
    return sum(it["flops"] for it in items)


def algorithmic_bytes(it):
    """compulsory bytes of one launch: inputs read once + outputs written once."""
    n = 0
    for t in it["exec"]._keep[0] + it["exec"]._keep[1]:
        n += t.numel() * t.element_size()
    return n


# ----------------------------------------------------------- CPU reference --
def cpu_sample_tasks():
    """A bounded sample of the same sweep for the reference CPU interpreter:
    conv layers on one image and 8 filters, FFN on 2 tokens, one attention head.
    Returns [(dag_json, inputs, out_shapes, flops, port_fn)]."""
    from oracle import port
    from paper_2210_09603_b200 import workloads as W

    rng = port.Rng(99)
    tasks = []
    for L in [W.RESNET50[i] for i in (3, 9, 15, 20, 21, 16)]:
        dag = W.conv_bn_relu_dag(L, 1, f=8)
        ho = L.out_hw()
        ins = {"X": rng.tensor((1, L.c, L.h, L.h)), "W": rng.tensor((8, L.c, L.k, L.k)),
               "Scale": rng.tensor((8,)), "Shift": rng.tensor((8,))}
        fn = (lambda ins=ins, L=L: port.conv_bn_relu(ins["X"], ins["W"], ins["Scale"], ins["Shift"], L.s, L.p))
        tasks.append((dag.to_json(), ins, {"Z": (1, 8, ho, ho)}, 2.0 * ho * ho * 8 * L.c * L.k * L.k, fn))
    t = 2
    dag = W.ffn_dag(t)
    ins = {"X": rng.tensor((t, 768)), "W1": rng.tensor((768, 3072)), "b1": rng.tensor((3072,)),
           "W2": rng.tensor((3072, 768)), "b2": rng.tensor((768,))}
    fn = (lambda ins=ins: port.ffn(ins["X"], ins["W1"], ins["b1"], ins["W2"], ins["b2"]))
    tasks.append((dag.to_json(), ins, {"O": (t, 768)}, 2.0 * t * 768 * 3072 * 2, fn))
    dag = W.attention_scores_dag(1)
    ins = {"Q": rng.tensor((1, 128, 64)), "K": rng.tensor((1, 128, 64))}
    fn = (lambda ins=ins: 0.125 * port.matmul(ins["Q"][0], ins["K"][0].T))
    tasks.append((dag.to_json(), ins, {"S": (1, 128, 128)}, 2.0 * 128 * 128 * 64, fn))
    return tasks


def run_cpu_sample(tasks, threads):
    """Runs the sample on `threads` host threads; returns (flops, seconds, kind).
    kind "reference" = the reference's reference_eval compiled from its sources
    (oracle/_ref); "port" = the numpy restatement when that library is absent."""
    import concurrent.futures as cf
    import oracle
    kind = "reference" if oracle.ref_available() else "port"

    def one(task):
        dag_json, ins, outs, _, fn = task
        if kind == "reference":
            oracle.ref_eval(dag_json, ins, list(outs), outs)
        else:
            fn()

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, tasks))
    return sum(t[3] for t in tasks), time.perf_counter() - t0, kind


def traffic_of(group):
    """DRAM bytes per launch of a kernel group from the committed ncu capture
    (profiles/traffic.json, scripts/traffic_from_launches.py), else None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f)[group]["dram_bytes_per_launch"]
    except Exception:
        return None


# -------------------------------------------------------------------- main --
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tune", default="auto", choices=["auto", "force", "off"],
                    help="auto: reuse tuning_cache.json entries, tune the rest on the device")
    ap.add_argument("--tuning-cache", default=os.path.join(ROOT, "tuning_cache.json"))
    ap.add_argument("--per-item", action="store_true", help="print per-launch times to stderr")
    ap.add_argument("--launch-list", action="store_true",
                    help="replay exactly one step and exit (for the ncu launch list / traffic capture)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    threads = args.cpu_threads or os.cpu_count() or 1

    if args.impl == "reference":
        if rank != 0:
            return
        tasks = cpu_sample_tasks()
        for _ in range(args.warmup):
            run_cpu_sample(tasks, threads)
        fl, secs = 0.0, 0.0
        kind = "reference"
        for _ in range(args.steps):
            f, s, kind = run_cpu_sample(tasks, threads)
            fl += f
            secs += s
        value = fl / secs / 1e12
        sample = "per step: 6 ResNet-50 conv layers (1 image, 8 filters) + FFN (2 tokens) + 1 attention head"
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "configs[4] sweep sample on host CPU (taskmap::reference_eval)",
                       "threads": threads},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }))
        return

    import torch
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=device)

    from paper_2210_09603_b200.tuning import TuningCache
    tuner = TuningCache(args.tuning_cache if rank == 0 else None)
    if rank != 0 and os.path.exists(args.tuning_cache):
        tuner = TuningCache(args.tuning_cache)  # read-only on other ranks
    t_build = time.perf_counter()
    items, treport = build_sweep(torch, device, seed=1234 + rank, tuner=tuner, tune_mode=args.tune,
                                 log=(lambda m: print(m, file=sys.stderr)) if rank == 0 else None)
    t_build = time.perf_counter() - t_build
    if rank == 0 and treport["tuned"]:
        tuner.save()
    flops_rank = sweep_flops(items)
    stream = torch.cuda.current_stream()
    results = [t for it in items if it.get("result") for t in it["outputs"]]
    from paper_2210_09603_b200.sharding import gather_buffers, gather_to_root
    gather_bufs = gather_buffers(results) if dist is not None else None

    # the whole sweep replays as one CUDA graph (no per-kernel host launch cost);
    # a second, timed graph with an event around every exec gives the per-launch
    # breakdown (measured separately so its event nodes do not perturb `value`)
    from paper_2210_09603_b200 import Graph
    graph = Graph([it["exec"] for it in items])
    tgraph = Graph([it["exec"] for it in items], timed=True)

    def step():
        graph.launch(stream)

    def gather():
        if dist is not None:
            gather_to_root(results, 0, gather_bufs)

    if args.launch_list:
        step()
        torch.cuda.synchronize()
        print(json.dumps({"launch_list": True, "launches_per_step": sum(it["exec"].num_launches for it in items),
                          "names": [it["name"] for it in items]}))
        return
    for _ in range(args.warmup):
        step()
        gather()
    torch.cuda.synchronize()

    # ---- timed region: K steps, clocks sampled
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for s in range(args.steps):
        step()
        gather()
    t1.record(stream)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = clk.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if dist is not None:
        tt = torch.tensor([ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    # ---- per-launch breakdown: the timed graph, K more steps
    per_item = [0.0] * len(items)
    for s in range(args.steps):
        tgraph.launch(stream)
        torch.cuda.synchronize()
        for i, t in enumerate(tgraph.exec_ms()):
            per_item[i] += t / args.steps

    # ---- e2e through the C ABI with host buffers: H2D inputs, launch, D2H results
    host_in = [[t.cpu().pin_memory() for t in it["inputs"]] for it in items]
    host_out = [[torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in it["outputs"]] if it.get("result") else []
                for it in items]
    h2d = sum(t.numel() * t.element_size() for ts in host_in for t in ts)
    d2h = sum(t.numel() * t.element_size() for ts in host_out for t in ts)

    # inputs stream in on a copy stream; each workload's kernels start as soon
    # as its own inputs have landed, so H2D of later layers overlaps compute
    copy_stream = torch.cuda.Stream(device=device)
    in_ready = [torch.cuda.Event() for _ in items]

    def e2e_step():
        copy_stream.wait_stream(stream)  # the previous step is done reading these buffers
        with torch.cuda.stream(copy_stream):
            for ev, it, hin in zip(in_ready, items, host_in):
                for d, h in zip(it["inputs"], hin):
                    d.copy_(h, non_blocking=True)
                ev.record(copy_stream)
        for ev, it, hout in zip(in_ready, items, host_out):
            stream.wait_event(ev)
            it["exec"].launch(stream)
            for d, h in zip(it["outputs"], hout):
                h.copy_(d, non_blocking=True)
        gather()

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e2e_steps = max(2, min(args.steps, 5))
    if dist is not None:
        dist.barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist is not None:
        tt = torch.tensor([e2e_ms], device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())

    if rank != 0:
        dist.destroy_process_group()
        return

    from paper_2210_09603_b200 import schedule_space
    peak_tf, peak_bw, peak_src = peaks()
    total_flops = flops_rank * world
    value = total_flops / (ms / 1e3) / 1e12
    groups = {}
    for it, t in zip(items, per_item):
        g = groups.setdefault(it["group"], {"flops": 0.0, "ms": 0.0, "bytes": 0, "launches": 0})
        g["flops"] += it["flops"]
        g["ms"] += t
        g["bytes"] += algorithmic_bytes(it)
        g["launches"] += it["exec"].num_launches
    for g in groups.values():
        g["tflops"] = g["flops"] / (g["ms"] / 1e3) / 1e12
        g["frac_of_peak"] = g["tflops"] / peak_tf
        g["ms_share"] = g["ms"] / sum(x["ms"] for x in groups.values())
    dom = max(groups, key=lambda k: groups[k]["ms"])
    dg = groups[dom]
    if args.per_item:
        # per launch: time, TFLOP/s, roofline lower bound max(flops/peak, bytes/bw), fraction of it
        sol_total = 0.0
        for it, t in zip(items, per_item):
            by = algorithmic_bytes(it)
            sol = max(it["flops"] / (peak_tf * 1e12), by / (peak_bw * 1e9)) * 1e3
            sol_total += sol
            print(f"{it['name']:12s} {t * 1e3:8.1f} us  {it['flops'] / (t / 1e3) / 1e12:7.1f} TFLOP/s  "
                  f"AI {it['flops'] / by:6.0f}  SOL {sol * 1e3:6.1f} us ({sol / t:5.1%})  {it.get('cfg', '')}", file=sys.stderr)
        print(f"sum {sum(per_item) * 1e3:.1f} us, SOL {sol_total * 1e3:.1f} us", file=sys.stderr)
    launches = sum(it["exec"].num_launches for it in items)

    cpu = None
    if not args.no_cpu_baseline:
        tasks = cpu_sample_tasks()
        f, s, kind = run_cpu_sample(tasks, threads)
        cpu = {"value": f / s / 1e12, "unit": "TFLOP/s", "cores": threads, "kind": kind,
               "sample": "6 ResNet-50 conv layers (1 image, 8 filters) + FFN (2 tokens) + 1 attention head, "
                         f"{s:.1f} s on {threads} host threads"}
    out = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "configs[4]: batch-sharded sweep = 53 ResNet-50 conv+BN+ReLU (batch 32/GPU) + "
                               "BERT FFN chain (64x128 tokens/GPU) + BERT attention QK^T/PV (192 heads/GPU)",
                   "per_gpu_batch": {"resnet": 32, "bert_tokens": 8192, "bert_heads": 192},
                   "parallelism": f"batch-sharded x{world}, final gather to rank 0",
                   "l2": "inputs larger than L2 (~1 GB of activations per step)",
                   "frac_of_peak": value / world / peak_tf,
                   "tuning": {"mode": args.tune, "workloads_tuned": treport["tuned"],
                              "workloads_cached": treport["cached"],
                              "tuning_time_s": round(treport["seconds"], 2),
                              "setup_time_s": round(t_build, 2),
                              "space_size": len(schedule_space("matmul"))}},
        "roofline": {"bound": "tensor", "kernel": f"tm_gemm_kernel ({dom} launches)",
                     "achieved": dg["tflops"], "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": dg["tflops"] / peak_tf, "traffic": traffic_of(dom),
                     "algorithmic_bytes_per_launch": dg["bytes"] / max(1, dg["launches"]),
                     "peak_source": f"{peak_src} bf16 burst"},
        "breakdown": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                      for k, v in groups.items()},
        "e2e": {"value": total_flops / (e2e_ms / 1e3) / 1e12, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "schedule": "per-workload C-ABI launches; H2D on a copy stream overlapping compute"},
        "gpu_launches": launches * args.steps,
        "launch": "one CUDA graph per step (all fused kernels of the sweep)",
        "clocks": clocks,
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
