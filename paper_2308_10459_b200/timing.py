"""Live kernel timing with CUDA events on the launching stream.

Events are recorded around selected launches inside the timed region and
resolved after it; launches that exited early (a PCG kernel after the solve
converged) are excluded by the caller's bookkeeping, not here.
"""

from __future__ import annotations

import torch


class KernelTimer:
    def __init__(self):
        self.pending = {}
        self.open = {}
        self.enabled = True

    def begin(self, name):
        if not self.enabled:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.open[name] = ev

    def end(self, name):
        if not self.enabled:
            return
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        self.pending.setdefault(name, []).append((self.open.pop(name), ev))

    def drop_last(self, name, k):
        if k > 0 and name in self.pending:
            del self.pending[name][-k:]

    def resolve(self) -> dict:
        """{name: list of durations in ms} (synchronises)."""
        torch.cuda.synchronize()
        return {k: [a.elapsed_time(b) for a, b in v] for k, v in self.pending.items()}

    def reset(self):
        self.pending.clear()
        self.open.clear()
