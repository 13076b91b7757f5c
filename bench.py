#!/usr/bin/env python
"""Benchmark: GTS batch range + kNN search on B200 (BASELINE.json metric
"range/kNN queries/sec ... vs CPU ref; distance evals/sec").

Default workload = BASELINE.json configs[1]: synthetic words (a-z, length
U[1,34]) n=1,000,000, edit distance, a 10,000-query batch answered as one
range batch (r=1) plus one kNN batch (k=10).  One step = both batches.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload words|dna|tloc]

value  : queries/sec with the query batch resident in HBM (device-timed).
e2e    : the same through the host C ABI (gts_*_batch_host): H2D of the
         query batch from pinned memory and D2H of the CSR answers inside
         the timed region.
With N>1 (torchrun), each rank holds its own shard of n objects (weak
scaling); every rank answers the full batch on its shard and the per-shard
answers are merged (paper_2404_00966_b200/sharded.py); value counts
shard-queries (queries x shards) per second.
"""

from __future__ import annotations

import argparse
import ctypes as C
import gc
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALPHA_WORDS = "abcdefghijklmnopqrstuvwxyz"
GEN_SEED, QUERY_SEED = 12, 13   # device generator (gts_generate_clustered) seeds

WORKLOADS = {
    # configs[1] -- the headline
    "words": dict(metric="edit", n=1_000_000, nq=10_000, min_len=1, max_len=34, alphabet=ALPHA_WORDS,
                  radius=1.0, k=10, config_index=1),
    # configs[3] (static part): DNA len 108
    "dna": dict(metric="edit", n=1_000_000, nq=10_000, min_len=108, max_len=108, alphabet="ACGT",
                radius=8.0, k=10, config_index=3),
    # configs[3] streaming: per step 1,000 deletes + 1,000 re-inserts, then the batch
    "dna_stream": dict(metric="edit", n=1_000_000, nq=10_000, min_len=108, max_len=108, alphabet="ACGT",
                       radius=8.0, k=10, config_index=3, updates=1000, cache_capacity=4096),
    # configs[0]: T-Loc-like 2-D L2, CPU-reference-runnable
    "tloc": dict(metric="l2", n=100_000, nq=1_000, dim=2, radius=0.0582588, k=10, config_index=0),
    # configs[2]: 128-d L2 n=1M, kNN k=10, 100k-query batch (clustered)
    "vec128": dict(metric="l2", n=1_000_000, nq=100_000, dim=128, clusters=1000, spread=0.05, noise=0.01,
                   radius=0.5, k=10, config_index=2),
    # configs[4] single shard: 32-d L1, 12.5M per GPU at 8 GPUs, kNN k=100.
    # C5 uses the reference generator's default spread (generate_clustered(...,
    # spread=0.01), data.py:405); C3 (vec128) keeps SURVEY §8(d)'s 0.05
    "l1shard": dict(metric="l1", n=12_500_000, nq=100_000, dim=32, clusters=12_500, spread=0.01, noise=0.01,
                    radius=0.5, k=100, config_index=4),
    # configs[4] whole: 32-d L1 n=100M, kNN k=100, 1M-query batch; the
    # collection and the queries are generated on the device (Philox,
    # gts_generate_clustered), one shard per GPU, built on the device
    "l1_100m": dict(metric="l1", n=100_000_000, nq=1_000_000, dim=32, clusters=100_000, spread=0.01, noise=0.01,
                    radius=0.5, k=100, config_index=4, device_gen=True, modes=(1,)),
}


# ---------------------------------------------------------------------------
# synthetic data (vectorised; same distribution as the reference generators)
# ---------------------------------------------------------------------------

def gen_strings(n, seed, min_len, max_len, alphabet):
    rng = np.random.default_rng(seed)
    lens = rng.integers(min_len, max_len + 1, size=n).astype(np.int64)
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=off[1:])
    alpha = np.frombuffer(alphabet.encode("utf-32-le"), dtype=np.int32)
    codes = alpha[rng.integers(0, alpha.size, size=int(off[-1]))].astype(np.int32)
    return codes, off


def string_queries(codes, off, nq, seed, alphabet):
    """Half members, half members with 1-2 random edits (test_acceptance.py:74-89)."""
    rng = np.random.default_rng(seed)
    n = off.size - 1
    alpha = np.frombuffer(alphabet.encode("utf-32-le"), dtype=np.int32)
    out = []
    for i, r in enumerate(rng.integers(0, n, nq)):
        s = list(codes[off[r]:off[r + 1]])
        if i >= nq // 2:
            for _ in range(int(rng.integers(1, 3))):
                c = int(alpha[int(rng.integers(0, alpha.size))])
                if s and rng.integers(0, 2):
                    s[int(rng.integers(0, len(s)))] = c
                else:
                    s.insert(int(rng.integers(0, len(s) + 1)), c)
        out.append(np.array(s, dtype=np.int32))
    qoff = np.zeros(nq + 1, dtype=np.int64)
    np.cumsum([len(s) for s in out], out=qoff[1:])
    qcodes = np.concatenate(out) if out else np.zeros(0, np.int32)
    return qcodes.astype(np.int32), qoff


def make_workload(name, rank, args, world=1, keep_full=False):
    """Synthetic data of the named shape.  The collection (n objects, seed 12)
    and the query batch (seed 13) do not depend on the rank: with N ranks the
    collection is split into N contiguous id ranges (one shard per GPU,
    strong scaling over one fixed collection) and every rank holds the same
    replicated batch.  w["n"] is this rank's shard size, w["n_total"] the
    collection's; keep_full keeps the whole collection (rank 0's parity
    check at N > 1)."""
    w = dict(WORKLOADS[name])
    if args.n:
        w["n"] = args.n
    if args.nq:
        w["nq"] = args.nq
    n_total = w["n"]
    lo, hi = n_total * rank // world, n_total * (rank + 1) // world
    seed = 12
    full = {}
    if w.get("device_gen"):
        # generated on the device by Engine (no host copy of the collection)
        w["ids"] = np.arange(lo, hi, dtype=np.int64)
        w["n"], w["n_total"], w["shard"] = hi - lo, n_total, (lo, hi)
        return w
    if w["metric"] == "edit":
        codes, off = gen_strings(n_total, seed, w["min_len"], w["max_len"], w["alphabet"])
        qcodes, qoff = string_queries(codes, off, w["nq"], 13, w["alphabet"])
        if keep_full:
            full = dict(codes=codes, off=off)
        w.update(codes=codes[off[lo]:off[hi]], off=off[lo:hi + 1] - off[lo], qcodes=qcodes, qoff=qoff)
    elif "clusters" in w:
        # clustered vectors: centers U[0,1)^D, members N(center, spread); queries are
        # members + N(0, noise); fp32-representable
        rng = np.random.default_rng(seed)
        D = w["dim"]
        centers = rng.uniform(0.0, 1.0, size=(w["clusters"], D)).astype(np.float32)
        mat = np.empty((n_total, D), dtype=np.float32)
        step = 1 << 20
        for a in range(0, n_total, step):
            b = min(n_total, a + step)
            assign = rng.integers(0, w["clusters"], size=b - a)
            mat[a:b] = centers[assign] + rng.normal(0.0, w["spread"], size=(b - a, D)).astype(np.float32)
        qr = np.random.default_rng(13)
        qi = qr.integers(0, n_total, size=w["nq"])
        q = mat[qi] + qr.normal(0.0, w["noise"], size=(w["nq"], D)).astype(np.float32)
        if keep_full:
            full = dict(mat=mat.astype(np.float64))
        w.update(mat=mat[lo:hi].astype(np.float64), q=q.astype(np.float32).astype(np.float64))
    else:
        rng = np.random.default_rng(seed)
        mat = rng.uniform(0.0, 1.0, size=(n_total, w["dim"])).astype(np.float32).astype(np.float64)
        q = np.random.default_rng(13).uniform(0.0, 1.0, size=(w["nq"], w["dim"])).astype(np.float32).astype(np.float64)
        if keep_full:
            full = dict(mat=mat)
        w.update(mat=mat[lo:hi], q=q)
    w["ids"] = np.arange(lo, hi, dtype=np.int64)
    w["n"], w["n_total"], w["shard"] = hi - lo, n_total, (lo, hi)
    if keep_full:
        full["ids"] = np.arange(n_total, dtype=np.int64)
        w["full"] = full
    return w


def bench_config(args, w, world):
    """The `config` object -- identical in both arms (same workload, sizes,
    tree geometry and budget)."""
    from oracle import oracle as O   # tree_height only (pure arithmetic, tree.py:60-78)
    n_total = w.get("n_total", w["n"])
    _, split = O.tree_height(max(n_total // world, 1), 20)
    return {
        "workload": f"{args.workload} (BASELINE.json configs[{w['config_index']}])",
        "n": n_total, "n_per_gpu": n_total // world, "nq": w["nq"], "radius": w["radius"], "k": w["k"],
        "node_capacity": 20, "levels_per_shard": split + 1,
        "memory_units": "device default: per-layer child tables of min(2^24 strings / 2^26 vectors, free HBM / (64 B x levels)) rows",
        "l2_policy": "index payload+tables exceed nothing: words (~25 MB) stay L2-resident by design; "
                     "no flush between steps (device-resident index is the operating point)",
        "parallelism": (f"{world} shards (contiguous id ranges, one GTS tree per GPU), replicated query batch; "
                        "kNN probe radii all-reduced (MIN), answers all-to-all'd to query owners and merged "
                        "on device" if world > 1 else "one GPU, one tree"),
    }


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.

    In-process NVML (pynvml), initialised when the sampler is created (before
    warm-up), so no nvidia-smi start-up lands inside a timed step.  Default
    mode "between": one synchronous sample after each timed step's final
    sync (tick()), outside that step's device interval -- an NVML call
    concurrent with a step measured 5-20 ms and stretched steps that
    synchronise with the host several times (words: 99-171 ms steps against
    84 ms of kernels).  GTS_CLOCK_MODE=full keeps the polling thread."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20), ("hw_thermal_slowdown", 0x40),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, gpu_index, interval_ms=200):
        import threading
        self.interval = interval_ms / 1e3
        self.samples = []
        self.on = threading.Event()
        self.quit = threading.Event()
        self.err = None
        self.call_ms = []
        self.mode = os.environ.get("GTS_CLOCK_MODE", "between")   # between | full | clock | none | off
        if self.mode == "off":
            self.nv, self.th = None, None
            self.err = "sampler off (GTS_CLOCK_MODE=off)"
            return
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[gpu_index]) if vis and vis.split(",")[0].isdigit() else gpu_index
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv = None
            self.err = f"nvml unavailable: {e}"
        self.th = None
        if self.mode != "between":
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    def _sample(self):
        t0 = time.perf_counter()
        sm = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        t1 = time.perf_counter()
        rs = 0 if self.mode == "clock" else self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        t2 = time.perf_counter()
        self.call_ms.append((round((t1 - t0) * 1e3, 2), round((t2 - t1) * 1e3, 2)))
        return sm, rs

    def _run(self):
        while not self.quit.is_set():
            if self.on.is_set() and self.nv is not None and self.mode != "none":
                try:
                    self.samples.append(self._sample())
                except Exception as e:  # noqa: BLE001
                    self.err = str(e)
            self.quit.wait(self.interval)

    def start(self):
        self.samples = []
        self.on.set()

    def tick(self):
        """One sample now (mode "between": called between timed steps)."""
        if self.mode == "between" and self.nv is not None:
            try:
                self.samples.append(self._sample())
            except Exception as e:  # noqa: BLE001
                self.err = str(e)

    def stop(self):
        self.on.clear()
        # one sample right at the end so even a short timed region has one
        if self.nv is not None and self.mode != "none":
            try:
                self.samples.append(self._sample())
            except Exception:  # noqa: BLE001
                pass
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "no samples"], "samples": 0}
        reasons = sorted({nm for _, r in self.samples for nm, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(self.samples),
                "source": "nvml (in-process, " + ("sampled after each timed step)" if self.mode == "between"
                                                  else "polling thread)"),
                "nvml_call_ms_max": max((a + b for a, b in self.call_ms), default=None)}

    def close(self):
        self.quit.set()
        if self.th is not None:
            self.th.join(timeout=1.0)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

class Engine:
    """Thin C-ABI driver (the same calls the Python drop-in makes)."""

    def __init__(self, w, device):
        from paper_2404_00966_b200 import _lib
        self.L = _lib.lib()
        self._lib = _lib
        self.w = w
        self.edit = w["metric"] == "edit"
        code = {"edit": 0, "l1": 1, "l2": 2}[w["metric"]]
        p = _lib.ptr
        n = w["n"]
        self.modes = w.get("modes", (0, 1))
        if w.get("device_gen"):
            self._init_device_gen(w, device)
            return
        if self.edit:
            self.ds = _lib.GtsDataset(code, n, 0, None, p(w["codes"], _lib._i32p), p(w["off"], _lib._i64p),
                                      p(w["ids"], _lib._i64p))
        else:
            self.ds = _lib.GtsDataset(code, n, w["dim"], p(w["mat"], _lib._f64p), None, None, p(w["ids"], _lib._i64p))
        nc = 20
        mh, sp = C.c_int64(), C.c_int64()
        _lib.check(self.L.gts_tree_height(n, nc, C.byref(mh), C.byref(sp)))
        levels = sp.value + 1
        nodes = self.L.gts_node_count(levels, nc)
        self.arrs = dict(
            pivot_id=np.zeros(nodes + 1, np.int64), pivot_row=np.zeros(nodes + 1, np.int64),
            pos=np.zeros(nodes + 1, np.int64), size=np.zeros(nodes + 1, np.int64),
            min_dis=np.zeros(nodes + 1), max_dis=np.zeros(nodes + 1), rows=np.zeros(n, np.int64),
            dis=np.zeros(n), tomb=np.zeros(n, np.uint8))
        a = self.arrs
        self.tree = _lib.GtsTree(nc, levels, sp.value, nodes, n, p(a["pivot_id"], _lib._i64p),
                                 p(a["pivot_row"], _lib._i64p), p(a["pos"], _lib._i64p), p(a["size"], _lib._i64p),
                                 p(a["min_dis"], _lib._f64p), p(a["max_dis"], _lib._f64p), p(a["rows"], _lib._i64p),
                                 p(a["dis"], _lib._f64p), p(a["tomb"], _lib._u8p))
        root_row = int(np.random.default_rng(0).integers(0, n))
        t0 = time.perf_counter()
        # device bulk build (csrc/devbuild.cuh; bit-identical to the host
        # builder); GTS_HOST_BUILD=1 uses the host C++/OpenMP builder
        self.build_where = "host" if os.environ.get("GTS_HOST_BUILD") == "1" else "device"
        if self.build_where == "host":
            _lib.check(self.L.gts_build_tree(C.byref(self.ds), root_row, 0, C.byref(self.tree)))
        else:
            _lib.check(self.L.gts_build_tree_device(C.byref(self.ds), root_row, device, C.byref(self.tree)))
        self.build_s = time.perf_counter() - t0
        self.levels = levels
        h = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(self.L.gts_index_create(C.byref(self.ds), C.byref(self.tree), device, C.byref(h)))
        self.upload_s = time.perf_counter() - t0
        self.ix = h
        nq = w["nq"]
        self.radii = np.full(nq, w["radius"], dtype=np.float64)
        self.ks = np.full(nq, w["k"], dtype=np.int64)
        if self.edit:
            self.qb = _lib.GtsQueryBatch(code, nq, 0, None, p(w["qcodes"], _lib._i32p), p(w["qoff"], _lib._i64p))
        else:
            self.qb = _lib.GtsQueryBatch(code, nq, w["dim"], p(w["q"], _lib._f64p), None, None)
        self.code = code

    def _init_device_gen(self, w, device):
        """Collection shard and query batch generated on the device
        (gts_generate_clustered), tree built on the device from the float32
        payloads (gts_build_tree_device_f32), index over them
        (gts_index_create_f32dev): nothing of the collection touches the host."""
        import torch
        _lib, L, p = self._lib, self.L, self._lib.ptr
        n, D, nq = w["n"], w["dim"], w["nq"]
        code = {"l1": 1, "l2": 2}[w["metric"]]
        dev = torch.device("cuda", device)
        t0 = time.perf_counter()
        x = torch.empty((max(n, 1), D), dtype=torch.float32, device=dev)
        qd = torch.empty((max(nq, 1), D), dtype=torch.float32, device=dev)
        st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        lo = w["shard"][0]
        _lib.check(L.gts_generate_clustered(GEN_SEED, w["n_total"], D, w["clusters"], w["spread"], lo, n, 0, 0.0,
                                            C.c_void_p(x.data_ptr()), st))
        _lib.check(L.gts_generate_clustered(GEN_SEED, w["n_total"], D, w["clusters"], w["spread"], 0, nq, QUERY_SEED,
                                            w["noise"], C.c_void_p(qd.data_ptr()), st))
        torch.cuda.synchronize(dev)
        self.gen_s = time.perf_counter() - t0
        w["q"] = qd[:nq].double().cpu().numpy()
        del qd
        nc = 20
        mh, sp = C.c_int64(), C.c_int64()
        _lib.check(L.gts_tree_height(n, nc, C.byref(mh), C.byref(sp)))
        levels = sp.value + 1
        nodes = L.gts_node_count(levels, nc)
        self.arrs = dict(
            pivot_id=np.zeros(nodes + 1, np.int64), pivot_row=np.zeros(nodes + 1, np.int64),
            pos=np.zeros(nodes + 1, np.int64), size=np.zeros(nodes + 1, np.int64),
            min_dis=np.zeros(nodes + 1), max_dis=np.zeros(nodes + 1), rows=np.zeros(n, np.int64),
            dis=np.zeros(n), tomb=np.zeros(n, np.uint8))
        a = self.arrs
        self.tree = _lib.GtsTree(nc, levels, sp.value, nodes, n, p(a["pivot_id"], _lib._i64p),
                                 p(a["pivot_row"], _lib._i64p), p(a["pos"], _lib._i64p), p(a["size"], _lib._i64p),
                                 p(a["min_dis"], _lib._f64p), p(a["max_dis"], _lib._f64p), p(a["rows"], _lib._i64p),
                                 p(a["dis"], _lib._f64p), p(a["tomb"], _lib._u8p))
        root_row = int(np.random.default_rng(0).integers(0, n))
        t0 = time.perf_counter()
        _lib.check(L.gts_build_tree_device_f32(code, n, D, C.c_void_p(x.data_ptr()), p(w["ids"], _lib._i64p),
                                               root_row, device, C.byref(self.tree)))
        self.build_s = time.perf_counter() - t0
        self.build_where = "device (float32 payloads generated on the device)"
        self.levels = levels
        h = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(L.gts_index_create_f32dev(C.byref(self.tree), code, D, C.c_void_p(x.data_ptr()),
                                             p(w["ids"], _lib._i64p), device, C.byref(h)))
        self.upload_s = time.perf_counter() - t0
        del x
        torch.cuda.empty_cache()
        self.ix = h
        self.radii = np.full(nq, w["radius"], dtype=np.float64)
        self.ks = np.full(nq, w["k"], dtype=np.int64)
        self.qb = _lib.GtsQueryBatch(code, nq, D, p(w["q"], _lib._f64p), None, None)
        self.code = code

    def upload(self, stream):
        q = C.c_void_p()
        self._lib.check(self.L.gts_queries_upload(self.ix, C.byref(self.qb), C.c_void_p(stream), C.byref(q)))
        self.q = q

    def step_device(self, stream):
        """Range + kNN batch (or the workload's modes) on device-resident
        queries; results stay in HBM."""
        res = []
        for mode in self.modes:
            h = C.c_void_p()
            if mode == 0:
                rc = self.L.gts_range_batch(self.ix, self.q, self._lib.ptr(self.radii, self._lib._f64p), 0, 1,
                                            C.c_void_p(stream), C.byref(h))
            else:
                rc = self.L.gts_knn_batch(self.ix, self.q, self._lib.ptr(self.ks, self._lib._i64p), 0, 1,
                                          C.c_void_p(stream), C.byref(h))
            self._lib.check(rc)
            res.append(h)
        return res

    def info(self, h):
        nq, tot, peak = C.c_int64(), C.c_int64(), C.c_int64()
        self._lib.check(self.L.gts_result_info(h, C.byref(nq), C.byref(tot), C.byref(peak), None))
        return nq.value, tot.value

    def free(self, hs):
        for h in hs:
            self.L.gts_result_free(h)

    def fetch(self, h, stream):
        """Host copy of a result CSR: (offsets, ids, dis)."""
        nq, tot = self.info(h)
        off = np.zeros(nq + 1, np.int64)
        ids = np.zeros(max(tot, 1), np.int64)
        dis = np.zeros(max(tot, 1), np.float64)
        p = self._lib.ptr
        self._lib.check(self.L.gts_result_copy(h, p(off, self._lib._i64p), p(ids, self._lib._i64p),
                                               p(dis, self._lib._f64p), None, None, C.c_void_p(stream)))
        import torch
        torch.cuda.synchronize()
        return off, ids[:tot], dis[:tot]


def run_stream(args, rank, world, local_rank):
    """configs[3]: StreamingIndex (the user-facing API) on 1M DNA strings; a
    step = 1,000 deletes + 1,000 re-inserts of the same ids with mutated
    payloads, then one 10k-query range (r=8) + kNN (k=10) batch over the live
    set (tree minus tombstones plus the device pending cache; a cache overflow
    rebuilds inside the step, as updates.py:121 does)."""
    import torch
    import paper_2404_00966_b200 as P
    from paper_2404_00966_b200 import _lib
    from paper_2404_00966_b200.search import HBM_SIZED
    torch.cuda.set_device(local_rank)
    w = make_workload("dna_stream", rank, args)
    codes, off = w["codes"], w["off"]
    alpha = w["alphabet"]
    strs = ["".join(map(chr, codes[off[i]:off[i + 1]])) for i in range(off.size - 1)]
    q = ["".join(map(chr, w["qcodes"][w["qoff"][i]:w["qoff"][i + 1]])) for i in range(w["nq"])]
    t0 = time.perf_counter()
    si = P.StreamingIndex(P.Dataset.from_strings(strs, P.EDIT, ids=w["ids"]), P.TreeConfig(20, 0),
                          cache_capacity=w["cache_capacity"], memory_units=HBM_SIZED)
    build_s = time.perf_counter() - t0
    rng = np.random.default_rng(5)
    # deleted ids are re-inserted in the same step, so the live id set never
    # changes: draw from a fixed pool (no per-step sort of 1M Python ints)
    pool = np.asarray(w["ids"][:200_000], dtype=np.int64)

    def step():
        dels = rng.choice(pool, w["updates"], replace=False)
        ins = []
        for oid in dels:
            s_ = list(strs[int(oid) - int(w["ids"][0])])
            for _ in range(3):
                s_[int(rng.integers(0, len(s_)))] = alpha[int(rng.integers(0, len(alpha)))]
            ins.append((int(oid), "".join(s_)))
        t0 = time.perf_counter()
        si.batch_update(inserts=ins, deletes=[int(x) for x in dels])
        t1 = time.perf_counter()
        a, _ = si.query_range(q, w["radius"])
        t2 = time.perf_counter()
        b, _ = si.query_knn(q, w["k"])
        t3 = time.perf_counter()
        if os.environ.get("GTS_STREAM_TRACE"):
            print(f"[stream] update {1e3 * (t1 - t0):.1f} ms  range {1e3 * (t2 - t1):.1f} ms  "
                  f"knn {1e3 * (t3 - t2):.1f} ms  rebuilds {si.rebuild_count}", file=sys.stderr, flush=True)
        return sum(x[0].size for x in a) + sum(x[0].size for x in b)

    clocks = ClockSampler(local_rank, args.clock_ms)
    gc.collect()
    gc.disable()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    rb0 = si.rebuild_count
    clocks.start()
    tot = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        tot += time.perf_counter() - t0
        clocks.tick()
    ms = tot * 1e3 / args.steps
    clk = clocks.stop()
    clocks.close()
    gc.enable()
    if rank != 0:
        return None
    nq = w["nq"]
    return {
        "metric": "range+kNN queries/sec (streaming)", "value": round(2 * nq / (ms / 1e3), 3), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8 symbols / int32 bit-parallel DP",
        "data": "synthetic",
        "config": {"workload": "dna_stream (BASELINE.json configs[3])", "n_per_gpu": w["n"], "nq": nq,
                   "radius": w["radius"], "k": w["k"], "updates_per_step": f"{w['updates']} deletes + {w['updates']} re-inserts",
                   "cache_capacity": w["cache_capacity"],
                   "timing": "wall clock around whole steps through the Python StreamingIndex API (updates, "
                             "H2D of the batch, search of tree + device cache, D2H of answers, rebuilds)"},
        "clocks": clk, "rebuilds_in_timed_steps": si.rebuild_count - rb0, "initial_build_s": round(build_s, 2),
        "gpu_launches": int(_lib.launch_count() - launches0),
    }


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2404_00966_b200 import _lib

    torch.cuda.set_device(local_rank)
    w = make_workload(args.workload, rank, args)
    eng = Engine(w, local_rank)
    stream = torch.cuda.Stream()
    sp = stream.cuda_stream
    nq = w["nq"]
    eng.upload(sp)

    def barrier():
        if world > 1:
            dist.barrier()

    def one_step():
        eng.free(eng.step_device(sp))

    clocks = ClockSampler(local_rank, args.clock_ms)
    # no Python garbage-collector pauses inside timed steps (a gen-2 pass over
    # the interpreter's objects idles the GPU for 100s of ms between calls)
    gc.collect()
    gc.disable()
    # warm-up
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()

    hs = eng.step_device(sp)
    torch.cuda.synchronize()
    totals = [eng.info(h)[1] for h in hs]
    # the answers of the timed batch per mode (0 range, 1 kNN), kept for the parity check
    gpu_answers = {m: eng.fetch(h, sp) for m, h in zip(eng.modes, hs)}
    eng.free(hs)
    tot_of = dict(zip(eng.modes, totals))

    # timed region (value): inputs resident in HBM.  Each step ends with a
    # device sync (the step's answers are complete), as a serving loop would.
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    ea = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    eb = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev0.record(stream)
    for i in range(args.steps):
        ea[i].record(stream)
        one_step()
        eb[i].record(stream)
        eb[i].synchronize()
        clocks.tick()
    ev1.record(stream)
    torch.cuda.synchronize()
    step_ms = [round(ea[i].elapsed_time(eb[i]), 3) for i in range(args.steps)]
    wall_ms = (time.perf_counter() - t_wall) * 1e3 / args.steps
    barrier()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    clocks.close()
    # the K steps' device intervals (each from its first launch to its final
    # sync); the clock samples between steps are outside them
    ms = sum(ea[i].elapsed_time(eb[i]) for i in range(args.steps)) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # profiling pass (after the timed region, not timed): per-kernel event
    # times + algorithmic work counters for the roofline
    _lib.lib().gts_profile_enable(1)
    _lib.profile_read(reset=True)
    one_step()
    torch.cuda.synchronize()
    prof = _lib.profile_read(reset=True)
    _lib.lib().gts_profile_enable(0)

    # e2e through the host C ABI with pinned buffers
    e2e_ms, h2d, d2h = run_e2e(eng, w, args, sp, max(totals))
    gc.enable()

    if rank != 0:
        return None
    nmodes = len(eng.modes)
    qps = nmodes * nq / (ms / 1e3)
    # the dominant leaf-verification kernel of this workload (whichever ran)
    cands = ("k_leafgroup_edit", "k_leaf_edit") if eng.edit else ("k_leafgroup_mma3", "k_leafgroup_mma2", "k_leafgroup_mma", "k_leafgroup_tile", "k_leafgroup_vec",
                                                                     "k_verify")
    kname = max(cands, key=lambda k: prof["kernels"].get(k, {"ms": 0.0})["ms"])
    kver = dict(prof["kernels"].get(kname, {"ms": 0.0, "count": 0}), name=kname)
    work = prof["work"]
    step_ms_prof = sum(v["ms"] for v in prof["kernels"].values())
    out = {
        "metric": "range+kNN queries/sec" if nmodes == 2 else "kNN queries/sec",
        "value": round(qps, 3),
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "wall_ms_per_step": round(wall_ms, 4),
        "step_ms": step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8 symbols / int32 bit-parallel DP" if eng.edit else "f32 screen + f64 exact recheck",
        "data": "synthetic",
        "config": bench_config(args, w, world),
        "range_answers_per_step": tot_of.get(0),
        "knn_answers_per_step": tot_of.get(1),
        "distance_evals_per_s": round(work["pairs"] / (step_ms_prof / 1e3), 1) if step_ms_prof else None,
        "build_s": round(eng.build_s, 3),
        "build_where": eng.build_where,
        "index_upload_s": round(eng.upload_s, 3),
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": {"value": round(nmodes * nq / (e2e_ms / 1e3), 3), "unit": "queries/s",
                "ms_per_step": round(e2e_ms, 4), "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "profile": prof,
    }
    out["roofline"] = roofline(eng, prof, kver, step_ms_prof)
    out["roofline"]["traversal"] = traversal_roofline(prof, args.workload, w.get("dim") if w["metric"] != "edit" else None)
    out["roofline"]["traffic"] = ncu_traffic(args.workload, kname)
    if out["roofline"]["traffic"] is not None:
        out["roofline"]["traffic_note"] = ("DRAM bytes (read + write) of one launch of this kernel from the "
                                           "committed ncu --set full capture (profiles/ncu_traffic.json); "
                                           "compare with achieved x average launch time")
    if world == 1 and not args.no_cpu_baseline:
        if w.get("device_gen"):
            out["cpu_baseline"], out["parity"] = scan_baseline(w, gpu_answers, eng.modes)
        else:
            out["cpu_baseline"], out["parity"] = cpu_baseline(w, args, gpu_answers)
    return out


def run_sharded(args, rank, world, local_rank):
    """N > 1: one shard of the fixed collection per GPU (strong scaling), the
    same query batch on every rank.  A step = range batch + kNN batch, each
    answered by every shard and merged on the query owners
    (paper_2404_00966_b200/sharded.py: kNN probe radii all-reduced with MIN,
    answers all-to-all'd to their owner, k_merge_rank on the owner's GPU).
    value = the batch's queries / max-over-ranks device time."""
    import torch
    import torch.distributed as dist
    from paper_2404_00966_b200 import _lib
    from paper_2404_00966_b200.sharded import ShardExchange, ShardSearcher, sharded_step

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    w = make_workload(args.workload, rank, args, world, keep_full=(rank == 0 and not args.no_cpu_baseline))
    want_parity = rank == 0 and not args.no_cpu_baseline
    eng = Engine(w, local_rank)
    stream = torch.cuda.Stream(dev)
    sp = stream.cuda_stream
    nq = w["nq"]
    ss = ShardSearcher(eng.ix, dev, stream=sp)
    ex = ShardExchange(nq, dev)
    ks_dev = torch.from_numpy(eng.ks).to(dev)
    nmodes = len(eng.modes)

    def one_step():
        with torch.cuda.stream(stream):
            return sharded_step(ss, ex, eng.radii, eng.ks, ks_dev, eng.modes)

    with torch.cuda.stream(stream):
        ss.upload(eng.qb)
    clocks = ClockSampler(local_rank, args.clock_ms)
    gc.collect()
    gc.disable()
    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    ans = one_step()
    torch.cuda.synchronize()
    own_answers = [tuple(t.cpu().numpy() for t in a) for a in ans]

    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = _lib.launch_count()
    ea = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    eb = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for i in range(args.steps):
        ea[i].record(stream)
        one_step()
        eb[i].record(stream)
        eb[i].synchronize()
        clocks.tick()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    step_ms = [ea[i].elapsed_time(eb[i]) for i in range(args.steps)]
    t = torch.tensor([sum(step_ms) / args.steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    dist.barrier()

    # e2e: H2D of the pinned host batch + search + exchange + D2H of the
    # owner's answers, every step
    if eng.edit:
        pc = torch.from_numpy(w["qcodes"]).pin_memory()
        po = torch.from_numpy(w["qoff"]).pin_memory()
        qb = _lib.GtsQueryBatch(0, nq, 0, None, C.cast(pc.data_ptr(), _lib._i32p), C.cast(po.data_ptr(), _lib._i64p))
        h2d = pc.numel() * 4 + po.numel() * 8
    else:
        pv = torch.from_numpy(w["q"]).pin_memory()
        qb = _lib.GtsQueryBatch(eng.code, nq, w["dim"], C.cast(pv.data_ptr(), _lib._f64p), None, None)
        h2d = pv.numel() * 8
    d2h = [0]
    pinned = {}

    def e2e_step():
        with torch.cuda.stream(stream):
            ss.upload(qb)
            res = sharded_step(ss, ex, eng.radii, eng.ks, ks_dev, eng.modes)
            b = 0
            for i, part in enumerate(res):
                for j, tns in enumerate(part):
                    host = pinned.get((i, j))
                    if host is None or host.numel() < tns.numel():
                        host = pinned[(i, j)] = torch.empty(int(tns.numel() * 1.25) + 1024, dtype=tns.dtype,
                                                            pin_memory=True)
                    host[:tns.numel()].copy_(tns, non_blocking=True)
                    b += tns.numel() * tns.element_size()
            stream.synchronize()
            d2h[0] = b

    for _ in range(max(1, args.warmup // 2)):
        e2e_step()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    clocks.close()
    gc.enable()

    # parity of rank 0's owned queries against brute force over the whole collection
    parity = None
    if want_parity:
        parity = sharded_parity(w, ex.own, own_answers)
    ss.free()
    if rank != 0:
        return None
    return {
        "metric": "range+kNN queries/sec" if nmodes == 2 else "kNN queries/sec",
        "value": round(nmodes * nq / (ms / 1e3), 3), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "step_ms_rank0": [round(x, 3) for x in step_ms], "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": "u8 symbols / int32 bit-parallel DP" if eng.edit else "f32 screen + f64 exact recheck",
        "data": "synthetic", "config": bench_config(args, w, world),
        "build_s_rank0": round(eng.build_s, 3), "index_upload_s_rank0": round(eng.upload_s, 3),
        "clocks": clk, "gpu_launches": int(launches),
        "e2e": {"value": round(nmodes * nq / (e2e_ms / 1e3), 3), "unit": "queries/s", "ms_per_step": round(e2e_ms, 4),
                "h2d_bytes_per_step": int(h2d + nq * 8 * nmodes), "d2h_bytes_per_step": int(d2h[0])},
        "parity": parity,
    }


def sharded_parity(w, own, answers, n_sample=32):
    """Rank 0's merged answers for a sample of its owned queries vs the
    oracle's brute force over the whole collection (oracle.py:19-36)."""
    from oracle import oracle as O
    lo, hi = own
    if w.get("device_gen"):
        idx = np.sort(np.random.default_rng(0).choice(np.arange(lo, hi), size=min(n_sample, hi - lo), replace=False))
        modes = w.get("modes", (0, 1))
        want, _ = chunked_brute(w, idx, modes, os.cpu_count() or 1)
        mism = 0
        for m, (off, ids, dis) in zip(modes, answers):
            for j, q in enumerate(idx):
                a, b = off[q - lo], off[q - lo + 1]
                if not (np.array_equal(ids[a:b], want[m][j][0]) and np.array_equal(dis[a:b], want[m][j][1])):
                    mism += 1
        return {"checked": len(modes) * idx.size, "mismatches": mism, "tolerated": 0,
                "against": "oracle brute force over the whole (device-regenerated) collection, sample of rank 0's "
                           "owned queries"}
    f = w["full"]
    if w["metric"] == "edit":
        data = O.Payloads(O.EDIT, codes=f["codes"], off=f["off"], ids=f["ids"])
    else:
        data = O.Payloads({"l1": O.L1, "l2": O.L2}[w["metric"]], vec=f["mat"], ids=f["ids"])
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(np.arange(lo, hi), size=min(n_sample, hi - lo), replace=False))
    qs = oracle_queries(O, w, idx)
    thr = os.cpu_count() or 1
    want = [O.brute(data, qs, O.RANGE, radii=np.full(idx.size, w["radius"]), threads=thr).answers(),
            O.brute(data, qs, O.KNN, ks=np.full(idx.size, w["k"]), threads=thr).answers()]
    mism = 0
    for (off, ids, dis), wa in zip(answers, want):
        for j, q in enumerate(idx):
            a, b = off[q - lo], off[q - lo + 1]
            if not (np.array_equal(ids[a:b], wa[j][0]) and np.array_equal(dis[a:b], wa[j][1])):
                mism += 1
    return {"checked": 2 * idx.size, "mismatches": mism, "tolerated": 0,
            "against": "oracle brute force over the whole collection (range and kNN (distance, id) lists), "
                       "sample of rank 0's owned queries"}


def run_e2e(eng, w, args, sp, max_total):
    import torch
    from paper_2404_00966_b200 import _lib
    nq = w["nq"]
    # pinned copies of the host inputs
    if eng.edit:
        pc = torch.from_numpy(w["qcodes"]).pin_memory()
        po = torch.from_numpy(w["qoff"]).pin_memory()
        qb = _lib.GtsQueryBatch(0, nq, 0, None, C.cast(pc.data_ptr(), _lib._i32p), C.cast(po.data_ptr(), _lib._i64p))
        h2d_in = pc.numel() * 4 + po.numel() * 8
    else:
        pv = torch.from_numpy(w["q"]).pin_memory()
        qb = _lib.GtsQueryBatch(eng.code, nq, w["dim"], C.cast(pv.data_ptr(), _lib._f64p), None, None)
        h2d_in = pv.numel() * 8
    prad = torch.from_numpy(eng.radii).pin_memory()
    pks = torch.from_numpy(eng.ks).pin_memory()
    cap = int(max_total * 1.25) + 1024
    o_off = torch.empty(nq + 1, dtype=torch.int64).pin_memory()
    o_ids = torch.empty(cap, dtype=torch.int64).pin_memory()
    o_dis = torch.empty(cap, dtype=torch.float64).pin_memory()
    o_ver = torch.empty(nq, dtype=torch.int64).pin_memory()
    o_pr = torch.empty(nq, dtype=torch.int64).pin_memory()
    L = eng.L
    bytes_out = [0]

    def step():
        b = 0
        for mode in eng.modes:
            h = C.c_void_p()
            if mode == 0:
                rc = L.gts_range_batch_host(eng.ix, C.byref(qb), C.cast(prad.data_ptr(), _lib._f64p), 0, 1,
                                            C.c_void_p(sp), C.byref(h))
            else:
                rc = L.gts_knn_batch_host(eng.ix, C.byref(qb), C.cast(pks.data_ptr(), _lib._i64p), 0, 1,
                                          C.c_void_p(sp), C.byref(h))
            _lib.check(rc)
            _, tot = eng.info(h)
            if tot > cap:
                raise RuntimeError("e2e output buffer too small")
            _lib.check(L.gts_result_copy(h, C.cast(o_off.data_ptr(), _lib._i64p), C.cast(o_ids.data_ptr(), _lib._i64p),
                                         C.cast(o_dis.data_ptr(), _lib._f64p), C.cast(o_ver.data_ptr(), _lib._i64p),
                                         C.cast(o_pr.data_ptr(), _lib._i64p), C.c_void_p(sp)))
            b += (nq + 1) * 8 + tot * 16 + 2 * nq * 8
            L.gts_result_free(h)
        bytes_out[0] = b

    for _ in range(max(1, args.warmup // 2)):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    h2d = len(eng.modes) * (h2d_in + nq * 8)
    return ms, h2d, bytes_out[0]


def roofline(eng, prof, kver, step_ms_prof):
    """Roofline of the dominant kernel.  achieved = ALGORITHMIC work of the
    step / that kernel's device time (CUDA events around each
    launch, profiling pass); peak = MEASURED_PEAKS.json, else the measured
    integer peak (edit) or the B200_PROFILING.md fallback."""
    from paper_2404_00966_b200 import _lib
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    work = prof["work"]
    t = kver["ms"] / 1e3 if kver["ms"] else None
    share = kver["ms"] / step_ms_prof if step_ms_prof else None
    common = {"kernel": kver["name"], "kernel_ms_per_step": round(kver["ms"], 4),
              "kernel_launches_per_step": kver["count"], "kernel_share_of_step": round(share, 4) if share else None,
              "pairs_per_step": work["pairs"], "entries_scanned_per_step": work["entries"]}
    if eng.edit:
        ops = C.c_double()
        _lib.check(_lib.lib().gts_bench_int_peak(C.byref(ops), None))
        peak = ops.value / 1e12
        achieved = work["word_steps"] * OPS_PER_WORD_STEP / t / 1e12 if t else None
        return dict(common, **{
            "bound": "int", "achieved": round(achieved, 3) if achieved else None, "peak": round(peak, 3),
            "unit": "Tops/s", "frac": round(achieved / peak, 4) if achieved else None, "traffic": None,
            "work_unit": f"word-step = one text symbol x one 32-bit pattern word = {OPS_PER_WORD_STEP} int ops "
                         "(the minimal Hyyro recurrence: 7 LOP3 + 1 add + 2 shifts)",
            "word_steps_per_step": work["word_steps"],
            "peak_source": "gts_bench_int_peak: best of LOP3-only / IMAD-only / mixed 16-chain loops on all SMs, "
                           "measured in this run (MEASURED_PEAKS.json has no integer peak)"})
    D = eng.w.get("dim", 2)
    if kver["name"] in ("k_leafgroup_mma", "k_leafgroup_mma2", "k_leafgroup_mma3"):
        tf = peaks.get("bf16_tflops_sustained") or peaks.get("bf16_tflops") or 1590.0
        flops = work["pairs"] * 2 * D
        achieved = flops / t / 1e12 if t else None
        return dict(common, **{
            "bound": "tensor", "achieved": round(achieved, 3) if achieved else None, "peak": tf,
            "unit": "TFLOP/s", "frac": round(achieved / tf, 5) if achieved else None, "traffic": None,
            "work_unit": f"2*D = {2 * D} bf16 tensor flops per lemma-1-passing (query, entry) pair",
            "peak_source": "MEASURED_PEAKS.json bf16" if peaks else "fallback 1590 TFLOP/s (B200_PROFILING.md)"})
    if kver["name"] == "k_leafgroup_tile":
        # register-tiled fp32 distances for every (query, entry) pair of an item:
        # 2 fp32 ops per dimension (L1: sub, |.|-add; L2: sub, fma counted once)
        ops = work["entries"] * 2 * D
        fp = C.c_double()
        _lib.check(_lib.lib().gts_bench_fp32_peak(C.byref(fp), None))
        pk = fp.value / 1e12
        achieved = ops / t / 1e12 if t else None
        return dict(common, **{
            "bound": "fp32", "achieved": round(achieved, 3) if achieved else None, "peak": round(pk, 2),
            "unit": "Tops/s", "frac": round(achieved / pk, 4) if achieved else None, "traffic": None,
            "work_unit": f"2*D = {2 * D} fp32 lane-ops per (query, entry) pair of an item",
            "peak_source": "gts_bench_fp32_peak: best of FADD-only / FFMA-only 16-chain loops on all SMs, measured "
                           "in this run (MEASURED_PEAKS.json has no fp32 peak)"})
    hbm = peaks.get("hbm_gbs", 6650.0)
    bytes_alg = work["entries"] * 8 + work["pairs"] * 4 * D
    achieved = bytes_alg / t / 1e9 if t else None
    return dict(common, **{
        "bound": "hbm", "achieved": round(achieved, 2) if achieved else None, "peak": hbm, "unit": "GB/s",
        "frac": round(achieved / hbm, 4) if achieved else None, "traffic": None,
        "work_unit": "8 B per (query, entry) scanned + 4*D B per lemma-1-passing pair",
        "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"})


def traversal_roofline(prof, workload, dim=None):
    """Roofline of the list-table traversal (k_expand / k_expand_grouped,
    search.py:405-477).  HBM leg: algorithmic bytes per SURVEY.md §8(d)
    (parent row, N_c 16-byte child records, the evaluated children's pivot
    payloads, the emitted 16-byte rows) / the launches' device time.  For
    vectors the grouped kernel stages each node's child pivots in shared
    memory once per item of rows, so the per-(row, child) payload bytes of
    that model never reach HBM (hbm frac can exceed 1); its bound is then
    the fp32 pipe: 2*Dp lane-ops per evaluated child distance (sub + fma /
    |.|-add), against the in-run gts_bench_fp32_peak.  `bound` names the
    leg with the larger fraction."""
    from paper_2404_00966_b200 import _lib
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = json.load(open(peaks_path)) if os.path.exists(peaks_path) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    k = prof["kernels"].get("k_expand")
    ex = prof.get("expand", {})
    if not k or not k["ms"]:
        return None
    gbs = ex.get("bytes", 0) / (k["ms"] / 1e3) / 1e9
    out = {"kernel": "k_expand", "launches_per_step": k["count"], "ms_per_step": round(k["ms"], 4),
           "bytes_per_step": int(ex.get("bytes", 0)), "rows_in": int(ex.get("rows_in", 0)),
           "rows_out": int(ex.get("rows_out", 0)), "distances": int(ex.get("evaluated", 0)),
           "bound": "hbm", "achieved": round(gbs, 2), "peak": hbm,
           "unit": "GB/s", "frac": round(gbs / hbm, 4),
           "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650 GB/s (B200_PROFILING.md)"}
    if dim and dim >= 16 and ex.get("evaluated"):
        dp = (dim + 3) // 4 * 4
        fp = C.c_double()
        _lib.check(_lib.lib().gts_bench_fp32_peak(C.byref(fp), None))
        pk = fp.value / 1e12
        ach = ex["evaluated"] * 2 * dp / (k["ms"] / 1e3) / 1e12
        out["fp32"] = {"achieved": round(ach, 3), "peak": round(pk, 2), "unit": "Tops/s", "frac": round(ach / pk, 4),
                       "work_unit": f"2*Dp = {2 * dp} fp32 lane-ops per evaluated child distance",
                       "peak_source": "gts_bench_fp32_peak (in-run)"}
        if ach / pk > out["frac"] or out["frac"] > 1:
            # the fp32 leg bounds it: report that leg at the top level
            out["hbm"] = {key: out[key] for key in ("achieved", "peak", "unit", "frac", "peak_source")}
            out.update({key: out["fp32"][key] for key in ("achieved", "peak", "unit", "frac", "peak_source")})
            out["bound"] = "fp32"
    out["traffic"] = ncu_traffic(workload, "k_expand") or ncu_traffic(workload, "k_expand_tile")
    return out


def ncu_traffic(workload, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed ncu --set full capture summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    tab = json.load(open(path))
    e = tab.get(f"{workload}:{kernel}")
    return e["dram_bytes_per_launch"] if isinstance(e, dict) else e


# Algorithmic integer ops per word-step: the 10-op Hyyro recurrence.
OPS_PER_WORD_STEP = 10


# ---------------------------------------------------------------------------
# CPU reference (oracle port) -- cpu_baseline leg and --impl reference
# ---------------------------------------------------------------------------

def oracle_setup(w):
    from oracle import oracle as O
    if w["metric"] == "edit":
        data = O.Payloads(O.EDIT, codes=w["codes"], off=w["off"], ids=w["ids"])
    else:
        data = O.Payloads({"l1": O.L1, "l2": O.L2}[w["metric"]], vec=w["mat"], ids=w["ids"])
    t0 = time.perf_counter()
    tree = O.build(data, 20, 0, threads=os.cpu_count() or 1)
    return O, data, tree, time.perf_counter() - t0


def oracle_queries(O, w, idx):
    if w["metric"] == "edit":
        qs = [w["qcodes"][w["qoff"][i]:w["qoff"][i + 1]] for i in idx]
        off = np.zeros(len(qs) + 1, np.int64)
        np.cumsum([len(s) for s in qs], out=off[1:])
        codes = np.concatenate(qs) if qs else np.zeros(0, np.int32)
        return O.Payloads(O.EDIT, codes=codes, off=off)
    return O.Payloads({"l1": O.L1, "l2": O.L2}[w["metric"]], vec=w["q"][idx])


def time_oracle(O, data, tree, w, n_range, n_knn, threads, seed=0):
    """Time the oracle port's BatchSearcher on a sample of the batch; returns
    {mode: (count, seconds, query indices, oracle Result)}."""
    rng = np.random.default_rng(seed)
    out = {}
    for mode, cnt, name in ((O.RANGE, n_range, "range"), (O.KNN, n_knn, "knn")):
        idx = np.sort(rng.choice(w["nq"], size=min(cnt, w["nq"]), replace=False))
        qs = oracle_queries(O, w, idx)
        t0 = time.perf_counter()
        res = O.search(tree, data, qs, mode, radii=np.full(len(idx), w["radius"]), ks=np.full(len(idx), w["k"]),
                       threads=threads)
        out[name] = (len(idx), time.perf_counter() - t0, idx, res)
    return out


def parity_check(O, data, w, t, gpu_answers, threads):
    """Compare the GPU answers of the timed batch with the oracle on the
    sampled queries: range = the reference engine's id and
    distance lists exactly; kNN = the reference engine's distance list exactly
    and the canonical brute-force (distance, id) top-k (oracle.brute_knn,
    oracle.py:30-36) exactly.  Float distances are compared bit for bit; the
    north-star tolerance (ids within 1e-5 relative of r / the k-th distance,
    distances within 1e-5 relative) is reported separately as `tolerated`."""
    checked = mism = tol = 0
    worst = []
    for name, gi in (("range", 0), ("knn", 1)):
        if name not in t:
            continue
        _, _, idx, ref = t[name]
        off, ids, dis = gpu_answers[gi]
        brute = None
        if name == "knn":
            brute = O.brute(data, oracle_queries(O, w, idx), O.KNN, ks=np.full(len(idx), w["k"]), threads=threads)
        ref_ans = ref.answers()
        br_ans = brute.answers() if brute is not None else None
        for j, q in enumerate(idx):
            g_ids, g_dis = ids[off[q]:off[q + 1]], dis[off[q]:off[q + 1]]
            r_ids, r_dis = ref_ans[j]
            checked += 1
            if name == "range":
                ok = np.array_equal(g_ids, r_ids) and np.array_equal(g_dis, r_dis)
                bound = w["radius"]
            else:
                b_ids, b_dis = br_ans[j]
                ok = (np.array_equal(g_dis, r_dis) and np.array_equal(g_ids, b_ids)
                      and np.array_equal(g_dis, b_dis))
                bound = float(r_dis[-1]) if r_dis.size else 0.0
            if ok:
                continue
            # north-star float tolerance: ids may differ only within 1e-5 relative
            # of the radius / k-th distance, distances within 1e-5 relative
            within = False
            if w["metric"] != "edit" and g_ids.size and r_ids.size:
                band = 1e-5 * max(bound, 1e-30)
                gd = dict(zip(g_ids.tolist(), g_dis.tolist()))
                rd = dict(zip(r_ids.tolist(), r_dis.tolist()))
                sym = set(gd) ^ set(rd)
                within = all(abs((gd.get(i, rd.get(i))) - bound) <= band for i in sym) and all(
                    abs(gd[i] - rd[i]) <= 1e-5 * max(abs(rd[i]), 1e-30) for i in set(gd) & set(rd))
            if within:
                tol += 1
            else:
                mism += 1
                if len(worst) < 4:
                    worst.append({"mode": name, "query": int(q), "gpu": [g_ids[:8].tolist(), g_dis[:8].tolist()],
                                  "oracle": [r_ids[:8].tolist(), r_dis[:8].tolist()]})
    out = {"checked": checked, "mismatches": mism, "tolerated": tol,
           "against": "oracle port BatchSearcher (range ids+distances, kNN distances) + oracle brute force "
                      "(kNN canonical (distance, id) top-k), on the cpu_baseline sample of the timed batch"}
    if worst:
        out["first_mismatches"] = worst
    return out


def chunked_brute(w, idx, modes, threads, chunk=1 << 23):
    """Oracle brute force (oracle.py:19-47) over a device-generated
    collection: chunks are regenerated on the device (the same Philox
    stream), copied to the host as float64 and scanned; per-query answers
    are merged by (distance, id) (k smallest for kNN).  Returns
    ({mode: [(ids, dis)] per query}, scan seconds)."""
    import torch
    from oracle import oracle as O
    from paper_2404_00966_b200 import _lib
    met = {"l1": O.L1, "l2": O.L2}[w["metric"]]
    qs = O.Payloads(met, vec=w["q"][idx])
    parts = {m: [[] for _ in idx] for m in modes}
    secs = 0.0
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = torch.empty((chunk, w["dim"]), dtype=torch.float32, device=dev)
    for a in range(0, w["n_total"], chunk):
        b = min(w["n_total"], a + chunk)
        _lib.check(_lib.lib().gts_generate_clustered(GEN_SEED, w["n_total"], w["dim"], w["clusters"], w["spread"],
                                                     a, b - a, 0, 0.0, C.c_void_p(buf.data_ptr()), None))
        torch.cuda.synchronize()
        data = O.Payloads(met, vec=buf[:b - a].double().cpu().numpy(), ids=np.arange(a, b, dtype=np.int64))
        t0 = time.perf_counter()
        for m in modes:
            r = O.brute(data, qs, m, radii=np.full(len(idx), w["radius"]), ks=np.full(len(idx), w["k"]),
                        threads=threads)
            for j, (ii, dd) in enumerate(r.answers()):
                parts[m][j].append((ii, dd))
        secs += time.perf_counter() - t0
    out = {}
    for m in modes:
        lst = []
        for j in range(len(idx)):
            ii = np.concatenate([p[0] for p in parts[m][j]])
            dd = np.concatenate([p[1] for p in parts[m][j]])
            o = np.lexsort((ii, dd))
            if m == 1:
                o = o[: w["k"]]
            lst.append((ii[o], dd[o]))
        out[m] = lst
    return out, secs


def scan_baseline(w, gpu_answers, modes, n_sample=32):
    """CPU baseline + parity for a device-generated collection: the oracle's
    brute-force scan -- the reference's pruning-off mode (_scan_all,
    search.py:338-355) -- on a sample of the batch, all host threads."""
    thr = os.cpu_count() or 1
    idx = np.sort(np.random.default_rng(0).choice(w["nq"], size=min(n_sample, w["nq"]), replace=False))
    want, secs = chunked_brute(w, idx, modes, thr)
    mism = 0
    for m in modes:
        off, ids, dis = gpu_answers[m]
        for j, q in enumerate(idx):
            if not (np.array_equal(ids[off[q]:off[q + 1]], want[m][j][0])
                    and np.array_equal(dis[off[q]:off[q + 1]], want[m][j][1])):
                mism += 1
    cb = {"value": round(len(modes) * len(idx) / secs, 4), "unit": "queries/s", "cores": thr, "kind": "port",
          "sample": f"{len(idx)} queries x {len(modes)} mode(s) of the batch, oracle brute-force scan over all "
                    f"{w['n_total']} objects (the reference's pruning-off mode, search.py:338-355), {thr} threads; "
                    "the collection regenerated in chunks (device Philox) and scanned in float64"}
    par = {"checked": len(idx) * len(modes), "mismatches": mism, "tolerated": 0,
           "against": "oracle brute force over the whole collection, (distance, id) lists"}
    return cb, par


def cpu_baseline(w, args, gpu_answers=None):
    O, data, tree, build_s = oracle_setup(w)
    threads = os.cpu_count() or 1
    n_range, n_knn = (256, 64) if w["metric"] == "edit" else ((1000, 1000) if w["n"] <= 100_000 else (32, 32))
    t = time_oracle(O, data, tree, w, n_range, n_knn, threads)
    per_q = (t["range"][1] / t["range"][0] + t["knn"][1] / t["knn"][0]) / 2
    cb = {
        "value": round(1.0 / per_q, 3), "unit": "queries/s", "cores": threads, "kind": "port",
        "sample": f"{t['range'][0]} range + {t['knn'][0]} kNN queries of the same batch on the same 1-shard index "
                  f"(oracle/gts_oracle.c = restated reference BatchSearcher, {threads} threads over query slices); "
                  f"range {t['range'][0] / t['range'][1]:.2f} q/s, kNN {t['knn'][0] / t['knn'][1]:.2f} q/s; "
                  f"value = 1 / mean per-query time at the bench's 1:1 range:kNN mix",
        "oracle_build_s": round(build_s, 2),
    }
    par = parity_check(O, data, w, t, gpu_answers, threads) if gpu_answers is not None else None
    return cb, par


def run_reference_scan(args, w, world):
    """Reference arm for a device-generated collection (configs[4] whole):
    the oracle's brute-force scan (the reference's pruning-off mode,
    search.py:338-355) over the collection, regenerated in chunks; one scan
    serves every step's sample (4 queries per step)."""
    import torch
    from paper_2404_00966_b200 import _lib
    torch.cuda.set_device(0)
    nq = w["nq"]
    qd = torch.empty((nq, w["dim"]), dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().gts_generate_clustered(GEN_SEED, w["n_total"], w["dim"], w["clusters"], w["spread"], 0, nq,
                                                 QUERY_SEED, w["noise"], C.c_void_p(qd.data_ptr()), None))
    w["q"] = qd.double().cpu().numpy()
    modes = w.get("modes", (0, 1))
    idx = np.sort(np.random.default_rng(1).choice(nq, size=min(nq, 4 * args.steps), replace=False))
    _, secs = chunked_brute(w, idx, modes, os.cpu_count() or 1)
    v = len(modes) * len(idx) / secs
    thr = os.cpu_count() or 1
    return {
        "impl": "reference", "metric": "range+kNN queries/sec" if len(modes) == 2 else "kNN queries/sec",
        "value": round(v, 4), "unit": "queries/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64 (CPU)", "data": "synthetic", "config": bench_config(args, w, world),
        "cpu_baseline": {"value": round(v, 4), "unit": "queries/s", "cores": thr, "kind": "port",
                         "sample": f"4 queries per step, oracle brute-force scan over all {w['n_total']} objects "
                                   f"(pruning-off mode), {thr} threads"},
        "e2e": {"value": round(v, 4), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def run_reference(args, rank, world):
    if rank != 0:
        return None
    w = make_workload(args.workload, 0, args)
    if w.get("device_gen"):
        return run_reference_scan(args, w, world)
    O, data, tree, build_s = oracle_setup(w)
    threads = os.cpu_count() or 1
    n_r, n_k = (32, 32) if w["metric"] == "edit" else ((500, 500) if w["n"] <= 100_000 else (16, 16))
    for i in range(args.warmup):
        time_oracle(O, data, tree, w, 4, 4, threads, seed=100 + i)
    tot_q, tot_t = 0, 0.0
    for i in range(args.steps):
        t = time_oracle(O, data, tree, w, n_r, n_k, threads, seed=i)
        tot_q += t["range"][0] + t["knn"][0]
        tot_t += t["range"][1] + t["knn"][1]
    v = tot_q / tot_t
    sample = (f"per step {n_r} range + {n_k} kNN queries of the {w['nq']}-query batch, oracle port "
              f"(restated reference BatchSearcher in C, {threads} threads over query slices)")
    return {
        "impl": "reference", "metric": "range+kNN queries/sec", "value": round(v, 3), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(tot_t / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/int64 (CPU)",
        "data": "synthetic", "config": bench_config(args, w, world),
        "cpu_baseline": {"value": round(v, 3), "unit": "queries/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": round(v, 3), "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "oracle_build_s": round(build_s, 2),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="words")
    # --objects / --queries: the same, for use behind torchrun (which claims "--n")
    ap.add_argument("--n", "--objects", dest="n", type=int, default=0)
    ap.add_argument("--nq", "--queries", dest="nq", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling interval in the timed region")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        # one process per GPU: re-launch this command under torchrun
        import socket
        import subprocess
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    # diagnostics: GTS_BENCH_ONE_DEVICE=1 puts every rank on cuda:0 (exercises
    # the N>1 merge path on a one-GPU box; use GTS_DIST_BACKEND=gloo with it)
    if os.environ.get("GTS_BENCH_ONE_DEVICE") == "1":
        local_rank = 0
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local_rank)
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(os.environ.get("GTS_DIST_BACKEND", "nccl"))
        if args.workload == "dna_stream":
            out = run_stream(args, rank, world, local_rank)
        elif world > 1:
            out = run_sharded(args, rank, world, local_rank)
        else:
            out = run_ours(args, rank, world, local_rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
    if out is not None:
        print(json.dumps(out), flush=True)
        par = out.get("parity")
        if par and par.get("mismatches"):
            sys.stderr.write(f"PARITY FAILURE: {par['mismatches']} of {par['checked']} sampled queries differ "
                             "from the oracle\n")
            sys.exit(3)


if __name__ == "__main__":
    main()
