"""Persistent tuning cache over tm_tune (SURVEY.md §5 "tuning
cache only" checkpoint/resume): the best ScheduleConfig per workload key, so a
re-run skips tuning.  Cold tuning time is recorded with every entry."""
import json
import os
import time
from dataclasses import asdict
from typing import Dict, Optional

from .taskmap import ScheduleConfig, schedule_space, tune


# bumped whenever the tuner's correctness gate changes: entries verified by an
# older gate are re-tuned
GATE_VERSION = 2


class TuningCache:
    def __init__(self, path: Optional[str]):
        self.path = path
        self.entries: Dict[str, dict] = {}
        if path and os.path.exists(path):
            with open(path) as f:
                self.entries = json.load(f)

    def save(self):
        if self.path:
            tmp = self.path + ".tmp"
            with open(tmp, "w") as f:
                json.dump(self.entries, f, indent=1, sort_keys=True)
            os.replace(tmp, self.path)

    def lookup(self, key: str) -> Optional[ScheduleConfig]:
        """The cached best config of `key`, or None when absent or stale: a cached
        config must still be a member of the current schedule_space (and verified
        by the current gate), else the workload is re-tuned."""
        e = self.entries.get(key)
        if not e or e.get("gate") != GATE_VERSION:
            return None
        c = ScheduleConfig(**e["config"])
        return c if c in schedule_space("conv2d") else None  # conv2d = the matmul space + the halo family

    def tune(self, key: str, dag, inputs, outputs, reps: int = 5, force: bool = False):
        """Returns (config, seconds spent tuning now, cached?)."""
        if not force:
            c = self.lookup(key)
            if c is not None:
                return c, 0.0, True
        t0 = time.perf_counter()
        best, report = tune(dag, inputs, outputs, reps=reps)
        secs = time.perf_counter() - t0
        self.entries[key] = {"config": asdict(best), "best_ms": report["best_ms"],
                             "space_size": report["space_size"], "tuning_time_s": secs,
                             "n_correct": report["n_correct"], "n_unsupported": report["n_unsupported"],
                             "n_incorrect": report["n_incorrect"], "gate": GATE_VERSION}
        return best, secs, False
