#!/usr/bin/env python
"""Tunes (tm_tune over schedule_space) every per-GPU workload shape of the
strong-scaling sweep at N = 1, 2, 4, 8 on one GPU -- rank 0's shard of each world
size, which equals every rank's shard for these even splits -- and saves the
best configs to tuning_cache.json, so bench.py --gpus N replays tuned schedules.

  python scripts/pretune_shards.py [--worlds 1,2,4,8] [--force]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    from paper_2210_09603_b200.sharding import sweep_shard
    from paper_2210_09603_b200.tuning import TuningCache
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    cache = TuningCache(os.path.join(ROOT, "tuning_cache.json"))
    dev = torch.device("cuda", 0)
    for w in (int(x) for x in a.worlds.split(",")):
        t0 = time.time()
        items, rep = bench.build_sweep(torch, dev, sweep_shard(0, w), tuner=cache,
                                       tune_mode="force" if a.force else "auto", log=lambda m: print(m, flush=True))
        cache.save()
        print(f"world {w}: tuned {rep['tuned']} cached {rep['cached']} in {rep['seconds']:.1f}s "
              f"(wall {time.time() - t0:.1f}s)", flush=True)
        del items
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
