"""One forward of the ResNet-50 chain (batch 32, tuned schedules from
tuning_cache.json) for the ncu launch list: warm-up eager pass, then one graph
replay.  Usage: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv python scripts/chain_once.py"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch  # noqa: E402

from paper_2210_09603_b200.chain import ResNet50Chain  # noqa: E402
from paper_2210_09603_b200.tuning import TuningCache  # noqa: E402

cache = TuningCache(os.path.join(os.path.dirname(__file__), "..", "tuning_cache.json"))
c = ResNet50Chain(32, 224, tuner=cache)
assert c.tuned == 0, "tuning_cache.json lacks chain entries"
c.replay()
torch.cuda.synchronize()
for st in c.stages:
    print(st.dst, st.kind, file=sys.stderr)
