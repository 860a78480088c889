#!/usr/bin/env python3
"""Benchmark of the B200 elastic-distance engine on BASELINE.json's workloads.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2] [--all]

Headline (one JSON line on rank 0): BASELINE.json configs[1] -- CDTW (w = 10%)
1-NN with early abandoning, 256 queries x 4096 candidates, length 512, warped-
prototype data (seeded, synthetic).  A step = one full 1-NN pass (all queries)
with inputs resident in HBM; L2 is flushed (256 MiB write) between steps.
`e2e` runs the same workload through the public Python API from host arrays.

Multi-GPU: one process per GPU (torchrun); every rank searches its own 256
queries against the same candidates -- queries shard with no data-path
collective, so scaling is "weak"; the step time is the max over ranks.

`--impl reference` times the reference's own compiled kernel
(oracle/_ref/_speedups*.so, built from /root/reference/pkg/src/elastik/_speedups.pyx)
driven by the restated nn_search loop, in a process pool over all host cores,
on a bounded sample of queries per step; rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "1-NN queries/s"
UNIT = "queries/s"
OPS_PER_CELL = {"dtw": 5, "cdtw": 5, "wdtw": 6, "erp": 7, "msm": 10, "twe": 9}


# ---------------------------------------------------------------- distributed plumbing

def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def dist_init(backend):
    import torch.distributed as dist

    rank, _, world = dist_env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group(backend=backend, rank=rank, world_size=world)
    return rank, world


def dist_max(x: float, device="cpu") -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_barrier():
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        dist.barrier()


def shard_seed(base: int, rank: int) -> int:
    """Weak scaling: rank r searches its own query set (same candidates)."""
    return base + 1 + 1000 * rank


# ---------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 8:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[4 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- workloads

def base_name(name):
    """'c2_fp32' -> 'c2': the FP32-mode lines run the same workload in float32."""
    return name[:-5] if name.endswith("_fp32") else name


def precision_of(name):
    return "float32" if name.endswith("_fp32") else "float64"


def spec_for(name):
    from paper_2102_05221_b200 import DistanceSpec

    name = base_name(name)
    return {
        "c1": DistanceSpec(kind="dtw"),
        "c2": DistanceSpec(kind="cdtw", window=51),
        "c3w": DistanceSpec(kind="wdtw", wdtw_g=0.05),
        "c3e": DistanceSpec(kind="erp", window=25, erp_gap=0.0),
        "c4m": DistanceSpec(kind="msm", msm_c=1.0),
        "c4t": DistanceSpec(kind="twe", twe_nu=0.001, twe_lambda=1.0),
        "c5": DistanceSpec(kind="cdtw", window=51),
    }[name]


def pinned_copy(a):
    """A numpy view of page-locked host memory holding a copy of `a` (the tensor is kept alive)."""
    import torch

    t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
    out = t.numpy()
    out[...] = a
    _PINNED.append(t)
    return out


_PINNED = []


def nn_data(name, rank=0):
    from paper_2102_05221_b200 import datagen

    wl = {"c1": datagen.C1, "c2": datagen.C2, "c4m": datagen.C4, "c4t": datagen.C4}[base_name(name)]
    C, cl, protos = datagen.warped_prototypes(wl.n_candidates, wl.length, wl.classes, wl.sigma, wl.seed)
    Q, ql, _ = datagen.warped_prototypes(wl.n_queries, wl.length, wl.classes, wl.sigma,
                                         shard_seed(wl.seed, rank), protos=protos)
    return wl, Q, ql, C, cl


WORKLOAD_NAMES = {
    "c1": "c1_dtw_1nn_16x256_L128", "c2": "c2_cdtw_w51_1nn_256x4096_L512",
    "c3w": "c3_wdtw_g0.05_allpairs_1024_L256", "c3e": "c3_erp_gap0_w25_allpairs_1024_L256",
    "c4m": "c4_msm_c1_1nn_512x8192_L512", "c4t": "c4_twe_nu0.001_lam1_1nn_512x8192_L512",
    "c5": "c5_cdtw_w51_subseq_q1024_stream2^20",
}
# the optional FP32 mode (north star: within 1e-5 relative, NN-index mismatch rate reported)
FP32_NAMES = {n + "_fp32": WORKLOAD_NAMES[n] + "_fp32" for n in ("c2", "c3w", "c3e", "c4m", "c4t")}
NN_NAMES = ("c1", "c2", "c4m", "c4t")


# ---------------------------------------------------------------- our arm

class Runner:
    """Device-resident inputs + one timed 'step' for each workload kind."""

    def __init__(self, name, rank, device):
        import torch

        from paper_2102_05221_b200 import _lib

        self.name, self.rank, self.device = name, rank, device
        self.base, self.precision = base_name(name), precision_of(name)
        self.torch = torch
        self.L = _lib.lib()
        self.lib = _lib
        self.spec = spec_for(name)
        self.kind = self.spec.kind
        t = lambda a, dt: torch.as_tensor(np.ascontiguousarray(a), dtype=dt, device=device)
        if self.base in NN_NAMES:
            wl, Q, ql, C, cl = nn_data(name, rank)
            self.host = (Q, C)
            self.nq, self.nc, self.Lq = Q.shape[0], C.shape[0], Q.shape[1]
            self.dQ, self.dC = t(Q.reshape(-1), torch.float64), t(C.reshape(-1), torch.float64)
            self.dqo = t(np.arange(self.nq) * self.Lq, torch.int64)
            self.dco = t(np.arange(self.nc) * self.Lq, torch.int64)
            self.dql = t(np.full(self.nq, self.Lq), torch.int32)
            self.dcl = t(np.full(self.nc, self.Lq), torch.int32)
            self.out = torch.empty(5 * self.nq, dtype=torch.int64, device=device)
            self.h = _lib.SpecHandle(self.spec, longest_lengths=[self.Lq], precision=self.precision)
            self.units = self.nq
            self.pairs = self.nq * self.nc
            self.cell_full = self.Lq * self.Lq
            self.unit = "queries/s"
        elif self.base in ("c3w", "c3e"):
            from paper_2102_05221_b200 import datagen

            X, _ = datagen.pairwise_workload(seed=3003 + rank)
            self.host = (X,)
            self.n, self.Lq = X.shape
            self.dX = t(X.reshape(-1), torch.float64)
            self.doff = t(np.arange(self.n) * self.Lq, torch.int64)
            self.dlen = t(np.full(self.n, self.Lq), torch.int32)
            self.dD = torch.empty(self.n * self.n, dtype=torch.float64, device=device)
            self.h = _lib.SpecHandle(self.spec, longest_lengths=[self.Lq], precision=self.precision)
            self.units = 1
            self.pairs = self.n * (self.n - 1) // 2
            self.cell_full = self.Lq * self.Lq
            self.unit = "matrices/s"
        else:  # c5
            from paper_2102_05221_b200 import datagen

            stream, q = datagen.subsequence_workload(seed=5005 + rank)
            self.host = (q, stream)
            self.Lq, self.nref = len(q), len(stream)
            self.dq, self.dref = t(q, torch.float64), t(stream, torch.float64)
            self.h = _lib.SpecHandle(self.spec)
            self.units = self.nref - self.Lq + 1
            self.pairs = self.units
            self.cell_full = self.Lq * self.Lq
            self.unit = "windows/s"
        self.last = {}
        self.pinned = None

    def step(self, stream_handle):
        import ctypes as C

        lib = self.lib
        if self.base in NN_NAMES:
            o = self.out.data_ptr()
            lib.check(self.L.ek_nn_dev(self.h.ref, 2, self.dQ.data_ptr(), self.dqo.data_ptr(), self.dql.data_ptr(),
                                       self.nq, self.dC.data_ptr(), self.dco.data_ptr(), self.dcl.data_ptr(), self.nc,
                                       self.Lq, 1, o, o + 8 * self.nq, o + 16 * self.nq, o + 24 * self.nq,
                                       o + 32 * self.nq, stream_handle))
        elif self.base in ("c3w", "c3e"):
            cells = np.zeros(1, dtype=np.int64)
            lib.check(self.L.ek_pairwise_dev(self.h.ref, 3, self.dX.data_ptr(), self.doff.data_ptr(),
                                             self.dlen.data_ptr(), self.n, self.Lq, 1, self.dD.data_ptr(),
                                             lib.iptr(cells), stream_handle))
            self.last["cells"] = int(cells[0])
        else:
            off = np.zeros(1, dtype=np.int64)
            d = np.zeros(1)
            cells = np.zeros(1, dtype=np.int64)
            comp = np.zeros(1, dtype=np.int64)
            ab = np.zeros(1, dtype=np.int64)
            lib.check(self.L.ek_subseq_dev(self.h.ref, 2, self.dq.data_ptr(), self.Lq, self.dref.data_ptr(),
                                           self.nref, 1, lib.iptr(off), lib.dptr(d), lib.iptr(cells),
                                           lib.iptr(comp), lib.iptr(ab), stream_handle))
            self.last.update(cells=int(cells[0]), offset=int(off[0]), dist=float(d[0]))
            _ = C

    def subseq_prefix(self, span):
        """(offset, distance) of the GPU search over the first `span` windows (parity, untimed)."""
        off = np.zeros(1, dtype=np.int64)
        d = np.zeros(1)
        z = [np.zeros(1, dtype=np.int64) for _ in range(3)]
        h = self.torch.cuda.current_stream().cuda_stream
        self.lib.check(self.L.ek_subseq_dev(self.h.ref, 2, self.dq.data_ptr(), self.Lq, self.dref.data_ptr(),
                                            span + self.Lq - 1, 1, self.lib.iptr(off), self.lib.dptr(d),
                                            *(self.lib.iptr(x) for x in z), h))
        return int(off[0]), float(d[0])

    def cells_after_step(self):
        if self.base in NN_NAMES:
            return int(self.out[2 * self.nq: 3 * self.nq].sum().item())
        return self.last.get("cells", 0)

    def e2e_call(self):
        """The same workload through the public API from host arrays (H2D + D2H inside)."""
        import paper_2102_05221_b200 as ekb
        from paper_2102_05221_b200 import SearchConfig

        if self.pinned is None:  # the step's inputs live in pinned host memory (copied in once, untimed)
            self.pinned = tuple(pinned_copy(a) for a in self.host)
        if self.base in NN_NAMES:
            Q, C = self.pinned
            ekb.nn_batch(self.spec, "eapruned", Q, C, precision=self.precision)
            return Q.nbytes + C.nbytes + 12 * (Q.shape[0] + C.shape[0]), 40 * Q.shape[0]
        if self.base in ("c3w", "c3e"):
            (X,) = self.pinned
            ekb.pairwise(self.spec, X, variant="pruned_only", precision=self.precision)
            return X.nbytes + 16 * X.shape[0], 8 * X.shape[0] ** 2 + 8
        q, stream = self.pinned
        ekb.subsequence_search(q, stream, SearchConfig(spec=self.spec, variant="eapruned", normalize=True))
        return q.nbytes + stream.nbytes, 40

    def e2e_pipelined(self, k):
        """k steps through the public streaming API (NNPipeline, two deep): every step uploads
        its queries and candidates from pinned host memory and reads its results back, and
        step i+1's upload overlaps step i's search.  Returns the wall time of the k steps."""
        import paper_2102_05221_b200 as ekb

        if self.pinned is None:
            self.pinned = tuple(pinned_copy(a) for a in self.host)
        Q, C = self.pinned
        t0 = time.perf_counter()
        for _ in ekb.nn_batch_stream(self.spec, "eapruned", ((Q, C) for _ in range(k)), precision=self.precision):
            pass
        return time.perf_counter() - t0


def phase_times(L):
    import ctypes as C

    ms = (C.c_double * 16)()
    names = (C.c_char_p * 16)()
    n = L.ek_phase_times(ms, names, 16)
    return {names[k].decode(): ms[k] for k in range(n)}


def time_steps(r, steps, warmup, flush):
    """Per-step device times (CUDA events on the launching stream), L2 flushed between steps."""
    torch = r.torch
    s = torch.cuda.current_stream()
    h = s.cuda_stream
    assert h != 0, "run on a non-default stream: the library maps handle 0 to its own stream"
    for _ in range(warmup):
        flush.zero_()
        r.step(h)
    torch.cuda.synchronize()
    r.L.ek_set_profiling(2)  # timed steps: only the events that bracket the DP kernels (the roofline's time)
    r.L.ek_launch_count(1)
    dist_barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    phases, cells = [], []
    t0 = time.perf_counter()
    for k in range(steps):
        flush.zero_()  # L2 flush (256 MiB write), outside the event pair
        ev[k][0].record(s)
        r.step(h)
        ev[k][1].record(s)
        ev[k][1].synchronize()
        phases.append(phase_times(r.L))
        cells.append(r.cells_after_step())
    torch.cuda.synchronize()
    dist_barrier()
    wall = time.perf_counter() - t0
    launches = int(r.L.ek_launch_count(0))
    # the full per-phase breakdown from extra, untimed steps (every phase mark is an event
    # between two kernels: ~2 us each on the device, kept out of the timed steps)
    r.L.ek_set_profiling(1)
    full = []
    for _ in range(3):
        flush.zero_()
        r.step(h)
        torch.cuda.synchronize()
        full.append(phase_times(r.L))
    r.L.ek_set_profiling(0)
    # the DP kernels' times stay the timed steps' own (their bracketing marks are recorded in
    # mode 2 too); every other phase comes from the full breakdown
    dp = ("nn_phase", "nn_fix", "triangle", "subseq_phase")
    phases = [{k: (p[k] if k.startswith(dp) and k in p else float(np.mean([f[k] for f in full]))) for k in full[0]}
              for p in phases]
    step_ms = [a.elapsed_time(b) for a, b in ev]
    return step_ms, phases, cells, launches, wall


# ---------------------------------------------------------------- the reference's CPU path

NN_PER_QUERY_S = {"c1": 0.003, "c2": 0.04, "c4m": 1.5, "c4t": 1.0}  # core-seconds, restated glue (sizing only)


class RefArm:
    """The reference's CPU implementation of the path on this host's cores: its own compiled
    kernel (oracle/_ref, built from /root/reference/pkg/src/elastik/_speedups.pyx) driven by
    the restated search loops (oracle/refdrive.py), or the C oracle port when _ref is absent.

    A persistent fork pool over all host cores shards independent units (queries, triangle
    rows, stream ranges).  It is created and warmed once, outside
    every timed step.  ``step()`` runs a bounded sample of the workload (sized for
    ``seconds`` of wall time) and returns its throughput plus the answers, which are the
    parity reference for the GPU's on the same inputs.
    """

    def __init__(self, name, lb="none", seconds=12.0, sample=None):
        from oracle import refdrive

        self.name, self.lb = base_name(name), lb
        self.cores = len(os.sched_getaffinity(0))
        self.kind = "reference" if refdrive.available() else "port"
        self.spec = spec_for(name)
        self.rd = refdrive
        self.env_s = 0.0
        cores = self.cores
        if self.name in NN_NAMES:
            wl, Q, ql, C, cl = nn_data(self.name, 0)
            self.Q, self.C = Q, C
            per_q = NN_PER_QUERY_S[self.name] * (6.0 if lb != "none" else 1.0)
            nq = sample or int(max(cores, min(Q.shape[0], seconds * cores / per_q)))
            self.items = list(range(min(nq, Q.shape[0])))
            self.unit, self.total = UNIT, Q.shape[0]
            if self.kind == "reference":
                t0 = time.perf_counter()
                env = refdrive.candidate_envelopes(self.spec, list(C), lb)  # classify_1nn builds them once
                self.env_s = time.perf_counter() - t0
                self.pool = refdrive.NNPool(self.spec, "eapruned", Q, C, lb, env, procs=cores)
        elif self.name in ("c3w", "c3e"):
            from paper_2102_05221_b200 import datagen

            X, _ = datagen.pairwise_workload()
            self.X = X
            n = X.shape[0]
            nrows = sample or max(2 * cores, min(n - 1, int(seconds * cores / 0.3)))
            self.items = sorted(set(np.linspace(0, n - 2, nrows).astype(int).tolist()))
            self.unit, self.total = "matrices/s", n * (n - 1) // 2
            if self.kind == "reference":
                self.pool = refdrive.PairwisePool(self.spec, X, "pruned_only", procs=cores)
        else:
            from paper_2102_05221_b200 import datagen

            stream, q = datagen.subsequence_workload()
            self.stream, self.q = stream, q
            nwin = len(stream) - len(q) + 1
            self.span = sample or min(nwin, int(seconds * cores / 2.5e-4))
            self.unit, self.total = "windows/s", nwin
            if self.kind == "reference":
                self.pool = refdrive.SubseqPool(self.spec, "eapruned", q, stream[: self.span + len(q) - 1], True,
                                                lb, procs=cores)
        if self.kind == "reference":
            self.pool.warm()

    def close(self):
        if self.kind == "reference":
            self.pool.close()

    def _run(self):
        if self.name in NN_NAMES:
            Qs = self.Q[self.items]
            if self.kind == "reference":
                return self.pool.run(self.items)
            from oracle import eko

            r = eko.nn(self.spec, "eapruned", Qs, self.C, threads=self.cores)
            return r["nn_index"], r["nn_distance"], r["cells"]
        if self.name in ("c3w", "c3e"):
            if self.kind == "reference":
                return self.pool.run(self.items)
            from oracle import eko

            D, _ = eko.pairwise(self.spec, self.X, threads=self.cores)
            return {i: D[i, i + 1:] for i in self.items}, 0
        if self.kind == "reference":
            return self.pool.run(0, self.span, chunk=2048)
        from oracle import eko

        return eko.subsequence(self.spec, "eapruned", self.q, self.stream[: self.span + len(self.q) - 1], True,
                               chunk=2048, threads=self.cores)

    def step(self):
        t0 = time.perf_counter()
        ans = self._run()
        wall = time.perf_counter() - t0
        if self.name in NN_NAMES:
            n = len(self.items)
            wall += self.env_s * n / self.total  # the serial envelope build, prorated to the sample
            value = n / wall
            sample = f"{n} of {self.total} queries x {self.C.shape[0]} candidates"
        elif self.name in ("c3w", "c3e"):
            npairs = sum(self.X.shape[0] - 1 - i for i in self.items)
            value = (npairs / self.total) / wall
            sample = f"{len(self.items)} upper-triangle rows ({npairs} of {self.total} pairs)"
        else:
            value = self.span / wall
            sample = f"first {self.span} of {self.total} windows (chunks of 2048, independent cutoffs)"
        sample += (f", lb={self.lb}, {wall:.1f} s wall, "
                   + ("persistent process pool, warmed before timing" if self.kind == "reference" else "threads"))
        return {"value": value, "unit": self.unit, "cores": self.cores, "kind": self.kind, "sample": sample,
                "wall_s": wall, "answers": ans}


REF_NOTE = ("reference = its own compiled _speedups kernel (oracle/_ref, built from _speedups.pyx) under a restated "
            "search loop (oracle/refdrive.py) that skips the Python facade (make_recurrence's tolist, "
            "engines.distance): faster per query than stock elastik, so the GPU ratios are conservative")


def parity_vs(ref, runner):
    """Bit-for-bit comparison of the GPU step's answers with the reference's on the sample."""
    ans = ref["answers"]
    if runner.base in NN_NAMES:
        ridx, rdist, _ = ans
        items = runner.ref_items
        gidx = runner.out[: runner.nq].cpu().numpy()[items]
        gdist = runner.out[runner.nq: 2 * runner.nq].cpu().numpy().view(np.float64)[items]
        return {"units": len(items), "what": "queries: nn index and distance",
                "idx_mismatch": int(np.sum(gidx != ridx)),
                "dist_mismatch": int(np.sum(gdist.view(np.int64) != np.asarray(rdist, np.float64).view(np.int64)))}
    if runner.base in ("c3w", "c3e"):
        rows, _ = ans
        D = runner.dD.view(runner.n, runner.n).cpu().numpy()
        bad = sum(int(np.sum(D[i, i + 1:].view(np.int64) != np.asarray(r).view(np.int64))) for i, r in rows.items())
        sym = int(np.sum(D.view(np.int64) != D.T.view(np.int64)))
        npairs = sum(len(r) for r in rows.values())
        return {"units": npairs, "what": "matrix entries of the sampled upper-triangle rows", "dist_mismatch": bad,
                "symmetry_mismatch": sym, "diag_nonzero": int(np.sum(np.diag(D) != 0.0))}
    off, d, _ = ans
    goff, gd = runner.subseq_prefix(runner.ref_span)
    return {"units": runner.ref_span, "what": "best (offset, distance) over the sampled windows",
            "idx_mismatch": int(goff != off), "dist_mismatch": int(np.float64(gd).view(np.int64) !=
                                                                    np.float64(d).view(np.int64))}


DOMINANT_KERNEL = {"c1": "k_nn", "c2": "k_nn", "c4m": "k_nn", "c4t": "k_nn", "c3w": "k_triangle",
                   "c3e": "k_triangle", "c5": "k_subseq_lb"}


def ncu_traffic(name):
    """(dram bytes per launch, source) of the config's dominant kernel, newest profiles/ summary."""
    import glob

    if name.endswith("_fp32"):
        return None
    profs = sorted(glob.glob(os.path.join(REPO, "profiles", f"r*_ncu_{name}_{DOMINANT_KERNEL[name]}*.json")))
    if not profs:
        return None
    try:
        return json.load(open(profs[-1])).get("dram_bytes_per_launch"), os.path.relpath(profs[-1], REPO)
    except (OSError, ValueError):
        return None


def run_ours(args):
    import torch

    rank, world = dist_init("nccl")
    _, local, _ = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2102_05221_b200 import _lib

    L = _lib.lib()
    _lib.check(L.ek_init(local))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    names = [args.config] + ([n for n in list(WORKLOAD_NAMES) + list(FP32_NAMES) if n != args.config]
                             if args.all else [])
    results = {}
    nn_index = {}  # FP64 1-NN answers per config (bit-identical to the reference's) for the FP32 mismatch rate
    peak_ops = L.ek_fp64_peak_ops()
    peak32_ops = L.ek_fp32_peak_ops() if any(n.endswith("_fp32") for n in names) else 0.0
    work_stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(work_stream)  # events and library launches share this stream
    for name in names:
        r = Runner(name, rank, dev)
        steps = args.steps if name == args.config else max(1, min(args.steps, 3))
        warm = args.warmup if name == args.config else 2  # (the second call on a stream sizes its workspace)
        with ClockSampler(local) as clk:
            step_ms, phases, cells, launches, wall = time_steps(r, steps, warm, flush)
        ms = float(np.mean(step_ms))
        ms_max = dist_max(ms, dev)
        value = world * r.units / (ms_max / 1e3)
        kern = [k for k in phases[0] if k.startswith(("nn_phase", "nn_fix", "triangle", "subseq_phase"))]
        kern_ms = float(np.mean([sum(p[k] for k in kern) for p in phases]))
        mean_cells = float(np.mean(cells))
        ops = mean_cells * OPS_PER_CELL[r.kind]
        achieved = ops / (kern_ms / 1e3) / 1e12
        fp32 = r.precision == "float32"
        peak = (peak32_ops if fp32 else peak_ops) / 1e12
        res = {
            "value": value, "unit": r.unit, "ms_per_step": ms_max, "step_ms": step_ms,
            "effective_gcups": world * r.pairs * r.cell_full / (ms_max / 1e3) / 1e9,
            "computed_gcups": world * mean_cells / (ms_max / 1e3) / 1e9,
            "computed_cells_per_step": mean_cells,
            "phases_ms": {k: float(np.mean([p.get(k, 0.0) for p in phases])) for k in phases[0]},
            "roofline": {"bound": "fp32_alu" if fp32 else "fp64_alu", "kernel": "+".join(kern), "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak > 0 else None,
                         "traffic": None, "ops_per_cell": OPS_PER_CELL[r.kind],
                         "peak_source": ("measured FP32 FADD/FMUL microbenchmark (ek_fp32_peak_ops)" if fp32 else
                                         "measured FP64 DADD/DMUL microbenchmark (ek_fp64_peak_ops)") +
                                        ", MEASURED_PEAKS.json has no non-tensor entry"},
            "dtype": "f32" if fp32 else "f64",
            "gpu_launches": launches // max(1, steps), "clocks": clk.summary(), "wall_s": wall,
        }
        # end to end through the public API with host buffers
        if rank == 0 and not args.no_e2e:
            t_e2e = []
            for k in range(max(1, min(steps, 10)) + 2):  # two untimed calls, then up to 10 timed
                t0 = time.perf_counter()
                hb, db = r.e2e_call()
                if k >= 2:
                    t_e2e.append(time.perf_counter() - t0)
            res["e2e"] = {"value": r.units / float(np.mean(t_e2e)), "unit": r.unit, "h2d_bytes_per_step": int(hb),
                          "d2h_bytes_per_step": int(db), "path": "public Python API (pinned numpy in, numpy out)"}
            if r.base in NN_NAMES:
                # the same calls pipelined two deep (NNPipeline): one call's upload overlaps the
                # previous call's search; the synchronous per-call number stays as e2e_sync
                k = max(2, min(steps, 64))  # the run's own step count (the pipeline's fill is inside the timed region)
                r.e2e_pipelined(4)  # untimed: slots allocated, each slot's workspace sized by its second batch
                dt = float(np.median([r.e2e_pipelined(k) for _ in range(3)]))  # three streams of k batches
                res["e2e_sync"] = dict(res["e2e"])
                res["e2e"] = {"value": k * r.units / dt, "unit": r.unit, "h2d_bytes_per_step": int(hb),
                              "d2h_bytes_per_step": int(db), "steps": k,
                              "path": "public Python API, streaming (search.NNPipeline: ek_nn_submit / ek_nn_collect, "
                                      "two batches in flight; pinned numpy in, numpy out, every step's inputs uploaded "
                                      "and its results read back inside the timed region)"}
        if r.base in NN_NAMES:
            idx = r.out[: r.nq].cpu().numpy().copy()
            if not fp32:
                nn_index[r.base] = idx
            elif r.base in nn_index:  # FP32 vs the FP64 (= reference) answers on the same queries
                res["nn_index_mismatch_rate"] = float(np.mean(idx != nn_index[r.base]))
        # the reference's CPU path on this host, same inputs (rank 0's), bounded sample; its
        # answers are the parity check of this run's GPU answers on that sample
        if rank == 0 and not fp32 and not args.no_cpu_baseline:
            ref = RefArm(name, seconds=args.cpu_seconds)
            try:
                cb = ref.step()
            finally:
                ref.close()
            res["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            res["cpu_baseline"]["note"] = REF_NOTE
            r.ref_items = getattr(ref, "items", None)
            r.ref_span = getattr(ref, "span", None)
            res["parity"] = parity_vs(cb, r)
            res["parity"]["against"] = cb["kind"] + " (" + ("oracle/_ref compiled _speedups" if cb["kind"] ==
                                                             "reference" else "oracle/ek_oracle.c") + ")"
        results[name] = res
        del r
        torch.cuda.empty_cache()
    if rank != 0:
        return
    head = results[args.config]
    line = {
        "metric": METRIC if args.config in ("c1", "c2", "c4m", "c4t") else f"{head['unit']}",
        "value": head["value"], "unit": head["unit"], "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": head["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded warped-prototype generator, paper_2102_05221_b200/datagen.py)",
        "config": {"workload": WORKLOAD_NAMES[args.config], "spec": repr(spec_for(args.config)),
                   "variant": "eapruned", "l2": "flushed between steps (256 MiB write)",
                   "shard": "queries per rank (same candidates), no data-path collective"},
        "effective_gcups": head["effective_gcups"], "computed_gcups": head["computed_gcups"],
        "roofline": head["roofline"], "phases_ms": head["phases_ms"], "gpu_launches": head["gpu_launches"],
        "clocks": head["clocks"],
    }
    if "e2e" in head:
        line["e2e"] = head["e2e"]
    if "e2e_sync" in head:
        line["e2e_sync"] = head["e2e_sync"]
    # dram bytes per launch of the dominant kernel from the committed `ncu --set full` summaries
    for name, res in results.items():
        tr = ncu_traffic(name)
        if tr:
            res["roofline"]["traffic"], res["roofline"]["traffic_source"] = tr
    for key in ("cpu_baseline", "parity"):
        if key in head:
            line[key] = head[key]
    if args.all:
        line["per_config"] = {n: {k: v for k, v in res.items() if k not in ("step_ms",)} for n, res in results.items()
                              if n != args.config}
    print(json.dumps(line), flush=True)


def run_reference(args):
    """The reference's CPU implementation, rank 0 only.

    Each step is a bounded sample of the workload on a persistent, warmed process pool over
    all host cores.  For dtw / cdtw workloads the reference's LB modes are timed too
    (lb="keogh2" is its cascaded LB_Keogh, search.py:104-112); `value` is the faster mode.
    """
    rank, world = dist_env()[0], dist_env()[2]
    if rank != 0:
        return
    name = args.config
    arm = RefArm(name, seconds=args.cpu_seconds)
    try:
        for _ in range(args.warmup):
            arm.step()
        cbs = [arm.step() for _ in range(args.steps)]
    finally:
        arm.close()
    vals = [c["value"] for c in cbs]
    by_lb = {"none": float(np.mean(vals))}
    if spec_for(name).kind in ("dtw", "cdtw") and arm.kind == "reference":
        arm2 = RefArm(name, lb="keogh2", seconds=args.cpu_seconds / 2)
        try:
            by_lb["keogh2"] = float(np.mean([arm2.step()["value"] for _ in range(max(1, min(args.steps, 2)))]))
        finally:
            arm2.close()
    best = max(by_lb, key=by_lb.get)
    value = by_lb[best]
    cb = cbs[-1]
    line = {
        "metric": METRIC if name in NN_NAMES else cb["unit"], "value": value,
        "unit": cb["unit"], "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean([c["wall_s"] for c in cbs])), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (seeded warped-prototype generator)",
        "config": {"workload": WORKLOAD_NAMES[name], "spec": repr(spec_for(name)), "variant": "eapruned",
                   "lb": best},
        "cpu_baseline": {"value": value, "unit": cb["unit"], "cores": cb["cores"], "kind": cb["kind"],
                         "sample": cb["sample"], "by_lb": by_lb, "note": REF_NOTE},
        "e2e": {"value": value, "unit": cb["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(WORKLOAD_NAMES), default="c2")
    ap.add_argument("--all", action="store_true", help="also measure every other BASELINE config")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="wall budget of one CPU-baseline sample")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to the contract minimum of 3", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
    _ = math
