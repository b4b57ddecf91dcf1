"""Persistent tuning cache over tm_tune (SURVEY.md §5 "tuning
cache only" checkpoint/resume): the best ScheduleConfig per workload key, so a
re-run skips tuning.  Cold tuning time is recorded with every entry."""
import json
import os
import time
from dataclasses import asdict
from typing import Dict, Optional

from .taskmap import ScheduleConfig, tune


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
        e = self.entries.get(key)
        return ScheduleConfig(**e["config"]) if e else None

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
                             "n_correct": sum(1 for r in report["results"] if r["correct"])}
        return best, secs, False
