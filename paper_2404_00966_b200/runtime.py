"""Budget accounting and the (host-side) runtime shim (reference runtime.py).

On this framework the data-parallel work runs on the GPU; ParallelRuntime
is kept so callers written against the reference keep working (its worker
count cannot change answers, runtime.py:1-8).
"""

from __future__ import annotations

import os

DEFAULT_MEMORY_UNITS = 1 << 20
DEFAULT_CONCURRENCY = 4096


class BudgetError(ValueError):
    """Invalid budget configuration or overflow (runtime.py:33-34)."""


class MemoryBudget:
    """Counts candidate-row units in use (runtime.py:56-88)."""

    def __init__(self, capacity=DEFAULT_MEMORY_UNITS):
        if capacity < 1:
            raise BudgetError("budget capacity must be >= 1")
        self.capacity = int(capacity)
        self.in_use = 0
        self.peak = 0

    def try_reserve(self, units):
        if units < 0:
            raise BudgetError("cannot reserve a negative unit count")
        if self.in_use + units > self.capacity:
            return False
        self.in_use += units
        self.peak = max(self.peak, self.in_use)
        return True

    def release(self, units):
        if units < 0:
            raise BudgetError("cannot release a negative unit count")
        if units > self.in_use:
            raise BudgetError("release below zero")
        self.in_use -= units


class ParallelRuntime:
    """Accepted for API compatibility; device kernels do the parallel work."""

    def __init__(self, workers=None, concurrency_capacity=DEFAULT_CONCURRENCY):
        self.workers = int(workers) if workers else (os.cpu_count() or 1)
        if self.workers < 1:
            raise ValueError("worker_count must be >= 1")
        self.concurrency_capacity = concurrency_capacity

    def close(self):
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
