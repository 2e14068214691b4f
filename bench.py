#!/usr/bin/env python
"""CPSJoin self-join benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 2] [--reps auto|R]

A step is one pass of the hot path over the whole synthetic workload:
MinHash embedding values (K1, t = 128) + 1-bit sketches (K1, 64 ell
functions) + the Chosen Path self-join with R repetitions (K2..K6), R the
smallest repetition count reaching the config's target recall against the
exact join (prefix-stable seeds).  `value` is measured with the CSR already
resident in HBM; `e2e` runs the public API from pinned host buffers with
the host->device copy of the CSR and the device->host read of the result
pairs inside every step.

--impl reference times the CPU implementation of the same path (the C
oracle port of the reference, all host threads) on a bounded sample of the
same workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "self-join sets/s at lambda=0.5, >=90% recall (embed + sketch + join)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", default="auto")
    ap.add_argument("--lambda", dest="lam", type=float, default=None,
                    help="similarity threshold (default: the config's first lambda, BASELINE.json)")
    ap.add_argument("--cpu-scale", type=float, default=None, help="CPU sample scale (default: auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # nvidia-smi in its own process at 500 ms; an in-process NVML thread
    # contends for the GIL with the launch path and slows the step (measured)
    ap.add_argument("--clock-source", default="points", choices=["points", "nvml", "smi"])
    ap.add_argument("--clock-ms", type=int, default=1000)
    ap.add_argument("--k1-transport", default="p2p", choices=["p2p", "collective"],
                    help="N>1: K1 rows stored on every GPU by the kernel (p2p) or an NCCL all-gather after it")
    ap.add_argument("--join-shard", default="frontier", choices=["frontier", "reps"],
                    help="N>1: split each tree's frontier at --frontier-depth across ranks, or whole repetitions")
    ap.add_argument("--frontier-depth", type=int, default=1)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: functional multi-rank run through host-staged collectives (not a bench number)")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-workload oracle comparison")
    ap.add_argument("--full-parity", action="store_true",
                    help="when the timed CPU baseline ran on a scaled sample, run the oracle once more (untimed) on "
                         "the whole workload so that parity.device_vs_oracle is always present")
    return ap.parse_args()


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------ clock sampling

class NvmlClockSampler:
    """SM clock + clock-event reasons polled in-process through NVML (the
    recipe's nvidia-smi fields) -- much lighter on the device than a polling
    nvidia-smi process, whose queries stall a busy GPU measurably."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4}

    def __init__(self, gpu: int, interval_s: float = 0.25):
        self.gpu, self.interval = gpu, interval_s
        self.samples = []
        self._stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
        except Exception:
            self.nv = None
            return self
        self._stop = threading.Event()

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                         self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
                except Exception:
                    pass
                self._stop.wait(self.interval)

        self.th = threading.Thread(target=loop, daemon=True)
        self.th.start()
        return self

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self.th.join(timeout=5)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML (in-process, 250 ms)"}


class NvmlPointSampler:
    """SM clock + clock-event reasons read through NVML from the main thread
    at fixed points inside the timed loops (first, middle and last step of
    each), while the GPU executes the queued work.  No polling process and
    no sampling thread: the periodic nvidia-smi queries measurably stalled
    the device (profiles/README.md)."""

    REASONS = NvmlClockSampler.REASONS

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.nv = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.nv = pynvml
            # warm the query path outside the timed region (first calls are slow)
            for _ in range(3):
                pynvml.nvmlDeviceGetClockInfo(self.h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            self.nv = None
        return self

    def __exit__(self, *exc):
        return False

    def sample(self):
        if self.nv is None:
            return
        try:
            self.samples.append((self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM),
                                 self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        except Exception:
            pass

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0, "source": "unavailable"}
        reasons = sorted({k for _, r in self.samples for k, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.samples),
                "source": "NVML from the launch thread as each timed loop (device, e2e) closes"}


class ClockSampler:
    # the recipe's clock fields minus power.draw (whose query was the one
    # that stalled the device mid-step in our measurements)
    FIELDS = ("index,clocks.sm,clocks.max.sm,clocks.mem,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int, interval_ms: int = 200):
        self.gpu = gpu
        self.proc = None
        self.interval_ms = interval_ms

    def __enter__(self):
        self.first = []
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # nvidia-smi's start-up (NVML init) stalls a busy device for up to
            # ~1 s: wait for its first sample before any timed work starts
            self.first.append(self.proc.stdout.readline())
            time.sleep(0.3)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            # the pre-roll sample is not inside the timed region
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for name, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ helpers

def measured_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "_fallback": True}


def int_peak(op_prefix: str, default: float):
    """Integer-pipe rate (per clk per SM) measured on the B200 by
    tools/int_peaks.cu (profiles/int_peaks_r01.json), else the default."""
    try:
        with open(os.path.join(ROOT, "profiles", "int_peaks_r01.json")) as f:
            for r in json.load(f)["results"]:
                if r["op"].startswith(op_prefix):
                    return float(r["ops_per_clk_per_sm"]), "measured, profiles/int_peaks_r01.json"
    except (OSError, KeyError, ValueError):
        pass
    return default, "assumed, SURVEY.md 8(d)"


def ncu_traffic(cfg: int, launch: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the
    dominant kernel from the committed ncu --set full capture, if it was
    taken on this config (profiles/ncu_traffic_r02.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic_r02.json")) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_launch"][launch]) if int(d["config"]) == cfg else None
    except (OSError, KeyError, ValueError):
        return None


def load_truth(cfg: int, scale: float, lam: float, tokens, offsets):
    from oracle.make_truth import csr_sha, truth_path
    path = truth_path(cfg, scale, lam)
    if not os.path.exists(path):
        return None
    z = np.load(path)
    if str(z["csr_sha"]) != csr_sha(tokens, offsets):
        log(f"truth file {path} does not match the generated workload; ignoring")
        return None
    return z["keys"]


def recall_of(a, b, truth) -> float:
    if truth is None or len(truth) == 0:
        return float("nan")
    keys = (np.asarray(a).astype(np.uint64) << np.uint64(32)) | np.asarray(b).astype(np.uint64)
    return float(np.isin(truth, keys).mean())


def workload_dict(w, cfg, R, rec, lam, extra=None):
    d = {"workload": f"{cfg.name} (BASELINE.json configs[{int(cfg.data_seed) - 1}])",
         "n_sets": int(w.n), "nnz_tokens": int(len(w.tokens)), "universe": int(w.d), "lambda": lam,
         "ell": cfg.ell, "t": 128, "repetitions": int(R), "recall": rec, "target_recall": cfg.recall,
         "epsilon": 0.1, "delta": 0.05, "limit": 250, "seeds": {"data": cfg.data_seed, "embed": cfg.emb_seed,
                                                                  "join": cfg.join_seed},
         "l2_policy": f"inputs larger than L2 (CSR {4 * len(w.tokens) / 1e6:.0f} MB + values "
                      f"{4 * 128 * w.n / 1e6:.0f} MB > 126 MB L2)"}
    if extra:
        d.update(extra)
    return d


# -------------------------------------------------------------- CPU (oracle)

def recall_truth(cfg_id: int, scale: float, w, lam: float):
    """Recall denominator: the exact-join truth file for this workload if one
    was generated (oracle/make_truth.py), else the planted pairs whose exact
    Jaccard is >= lambda (a proxy; stated in the output)."""
    t = load_truth(cfg_id, scale, lam, w.tokens, w.offsets)
    if t is not None:
        return t, "exact join (oracle/make_truth.py)"
    keys = []
    for a, b in w.planted_pairs.tolist():
        x = w.tokens[w.offsets[a]:w.offsets[a + 1]]
        y = w.tokens[w.offsets[b]:w.offsets[b + 1]]
        inter = len(np.intersect1d(x, y, assume_unique=True))
        if inter / (len(x) + len(y) - inter) >= lam:
            keys.append((min(a, b) << 32) | max(a, b))
    return np.unique(np.array(keys, dtype=np.uint64)), "planted pairs with J >= lambda (proxy, no truth file)"


class CpuArm:
    """The C oracle (port of the reference path) on one workload, all threads."""

    def __init__(self, w, cfg, threads: int):
        from oracle import oracle as O
        self.O, self.w, self.cfg, self.threads = O, w, cfg, threads
        self.lam = cfg.lambdas[0]

    def pipeline(self, reps: int):
        """embed_dataset + sketches + cpsjoin_self, timed: (seconds, JoinOut)."""
        t0 = time.perf_counter()
        _, _, out = self.O.full_pipeline(self.w.tokens, self.w.offsets, self.w.sizes, lam=self.lam, t=128,
                                         emb_seed=self.cfg.emb_seed, ell=self.cfg.ell, seed=self.cfg.join_seed,
                                         repetitions=reps, threads=self.threads)
        return time.perf_counter() - t0, out

    def choose_reps(self, truth):
        O, w, cfg = self.O, self.w, self.cfg
        values = O.minhash(w.tokens, w.offsets, O.embedding_tables(128, cfg.emb_seed), self.threads)
        mh, bt = O.sketch_tables(cfg.ell, cfg.join_seed)
        sk = O.sketch(w.tokens, w.offsets, mh, bt, self.threads)
        rec = 0.0
        for R in range(1, 11):
            out = O.self_join(w.tokens, w.offsets, w.sizes, values, sk, self.lam, repetitions=R,
                              seed=cfg.join_seed, threads=self.threads)
            rec = float(np.isin(truth, out.keys).mean()) if len(truth) else 1.0
            if rec >= cfg.recall:
                break
        return R, rec


def cpu_sample_scale(cfg_id: int, threads: int, budget_s: float = 15.0) -> float:
    """Largest workload fraction whose oracle pipeline should take about
    `budget_s` seconds, from a timed 10k-set calibration run (1.0 = full)."""
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    cfg = CONFIGS[cfg_id]
    n_full = cfg.n_background + cfg.n_planted
    s0 = min(1.0, 10_000 / n_full)
    w0 = generate(cfg_id, scale=s0)
    dt, _ = CpuArm(w0, cfg, threads).pipeline(3)
    return min(1.0, s0 * budget_s / max(dt, 1e-3))


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference(args, rank: int, world: int):
    from paper_1707_06814_b200.workloads import CONFIGS, generate
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    lam = args.lam if args.lam is not None else cfg.lambdas[0]
    threads = cpu_threads()
    # the GPU arm's exact workload when its recall truth is on file (c2: ~10 s
    # per step on 16 host threads), else a sample sized to ~15 s per step
    from oracle.make_truth import truth_path
    if args.cpu_scale:
        scale = args.cpu_scale
    elif os.path.exists(truth_path(args.config, args.scale, lam)):
        scale = args.scale
    else:
        scale = cpu_sample_scale(args.config, threads) * args.scale
        if scale > 0.8 * args.scale:
            scale = args.scale
    w = generate(args.config, scale=scale)
    truth, truth_src = recall_truth(args.config, scale, w, lam)
    arm = CpuArm(w, cfg, threads)
    arm.lam = lam
    R, rec = arm.choose_reps(truth)
    for _ in range(max(0, min(args.warmup, 1))):  # one warm-up: the port has no JIT or caches to warm
        arm.pipeline(R)
    times = [arm.pipeline(R)[0] for _ in range(args.steps)]
    total = sum(times)
    value = w.n * len(times) / total
    sample = (f"{cfg.name} x{scale:g}: {w.n} sets, embed+sketch+join R={R} (recall {rec:.3f} vs {truth_src}), "
              f"{total / len(times):.2f} s per step, {threads} threads")
    line = {"metric": METRIC, "value": value, "unit": "sets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded generator for the BASELINE.json config)",
            # the GPU arm's config dict (same workload keys) when the sample is the whole workload
            "config": workload_dict(w, cfg, R, rec, lam, {
                "recall_truth": truth_src, "n_true_pairs": int(len(truth)),
                **({} if scale == args.scale else {"sample_scale": scale})}),
            "parallelism": f"host CPU, {threads} threads (C port of the reference, oracle/cpsj_oracle.c)",
            "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "sets/s", "cores": threads, "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": "sets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- GPU arm

def parity_check(res, ref_keys, ref_sims, ref_counters) -> dict:
    """Bit-exact comparison of a GPU join result with another result: the
    unique pair keys, the f64 similarities and the five counters."""
    keys = (np.asarray(res.a).astype(np.uint64) << np.uint64(32)) | np.asarray(res.b).astype(np.uint64)
    c = res.counters
    got_c = [c.pre_candidates, c.candidates, c.results, c.max_depth, c.peak_live_members]
    same_keys = bool(np.array_equal(keys, ref_keys))
    same_sims = bool(same_keys and np.array_equal(np.asarray(res.similarity).view(np.uint64),
                                                  np.asarray(ref_sims).view(np.uint64)))
    return {"bit_exact": bool(same_keys and same_sims and got_c == list(ref_counters)), "keys": same_keys,
            "sims": same_sims, "counters": got_c == list(ref_counters), "n_pairs": int(len(keys))}


def run_ours(args, rank: int, world: int):
    import torch

    from paper_1707_06814_b200 import CPSJoinParams, Dataset, EmbeddingParams, cpsjoin_self_arrays, embed_dataset
    from paper_1707_06814_b200._native import Context
    from paper_1707_06814_b200.distributed import (PeerArrays, embed_sharded, embed_sharded_p2p,
                                                   embed_sharded_p2p_from_host, embedded_from_parts,
                                                   shard_frontier, shard_reps)
    from paper_1707_06814_b200.embed import embed_device_csr
    from paper_1707_06814_b200.workloads import CONFIGS, generate

    cfg = CONFIGS[args.config]
    lam = args.lam if args.lam is not None else cfg.lambdas[0]
    dev = torch.device("cuda", torch.cuda.current_device())
    t0 = time.time()
    w = generate(args.config, scale=args.scale)
    log(f"[rank {rank}] workload {cfg.name} x{args.scale}: n={w.n} nnz={len(w.tokens)} in {time.time() - t0:.1f}s")
    n = w.n
    ctx = Context.get()

    # pinned host inputs (the e2e source) and an HBM-resident copy (value)
    tok_pin = torch.from_numpy(w.tokens.view(np.int32)).pin_memory()
    off_pin = torch.from_numpy(w.offsets).pin_memory()
    ds = Dataset.from_csr(tok_pin.numpy().view(np.uint32), off_pin.numpy(), w.d)
    d_tok = tok_pin.to(dev)
    d_off = off_pin.to(dev)
    eparams = EmbeddingParams(t=128, seed=cfg.emb_seed)

    # repetitions: smallest R reaching the target recall (prefix-stable seeds)
    truth, truth_src = recall_truth(args.config, args.scale, w, lam)
    emb0 = embed_device_csr(eparams, d_tok, d_off, w.d, host_csr=(w.tokens, w.offsets))
    if args.reps != "auto":
        R = int(args.reps)
        res = cpsjoin_self_arrays(emb0, CPSJoinParams(lambda_=lam, ell=cfg.ell, seed=cfg.join_seed, repetitions=R))
        rec = recall_of(res.a, res.b, truth)
    else:
        for R in range(1, 11):
            res = cpsjoin_self_arrays(emb0, CPSJoinParams(lambda_=lam, ell=cfg.ell, seed=cfg.join_seed,
                                                          repetitions=R))
            rec = recall_of(res.a, res.b, truth)
            if rec >= cfg.recall:
                break
    log(f"[rank {rank}] R={R} recall={rec:.4f} truth={None if truth is None else len(truth)}")
    single = res  # the single-GPU join of this workload (every rank computes it once, untimed)
    del emb0
    params = CPSJoinParams(lambda_=lam, ell=cfg.ell, seed=cfg.join_seed, repetitions=R)

    stream = torch.cuda.current_stream(dev)
    k1_events = []

    skey = (cfg.ell, cfg.join_seed)

    peers = None
    side = torch.cuda.Stream(dev) if world > 1 else None
    if world > 1 and args.k1_transport == "p2p":
        # node-wide exchange buffers: K1 stores every row on every GPU, and
        # every rank pushes its CSR slice to every GPU (end to end)
        peers = PeerArrays(ctx, n, 128, cfg.ell, rank, world, nnz=len(w.tokens))

    def k1_sharded(t_tok, t_off, ev=None):
        if peers is not None:
            # set-sharded K1 with the all-gather fused into its epilogue
            vals, _ = embed_sharded_p2p(eparams, t_tok, t_off, w.d, None, rank, world, peers)
            if ev is not None:
                ev[1].record(stream)
            _, sk = embed_sharded_p2p(None, t_tok, t_off, w.d, skey, rank, world, peers)
        else:
            # set-sharded K1 + NCCL all-gather of the value / sketch rows
            vals, _ = embed_sharded(eparams, t_tok, t_off, w.d, None, rank, world)
            if ev is not None:
                ev[1].record(stream)
            _, sk = embed_sharded(None, t_tok, t_off, w.d, skey, rank, world)
        return embedded_from_parts(eparams, t_tok, t_off, w.d, vals, sk, skey)

    def join_sharded(emb):
        if args.join_shard == "reps":
            return shard_reps(emb, params, rank, world)
        return shard_frontier(emb, params, rank, world, depth=args.frontier_depth)

    def step_device():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        if world == 1:
            emb = embed_device_csr(eparams, d_tok, d_off, w.d)
            ev[1].record(stream)
            emb.sketches_device(*skey)
        else:
            emb = k1_sharded(d_tok, d_off, ev)
        ev[2].record(stream)
        k1_events.append(ev)
        return join_sharded(emb)

    h2d_rank = [int(w.tokens.nbytes + w.offsets.nbytes)]

    def step_e2e():
        if world == 1:
            emb = embed_dataset(eparams, ds, sketch=skey)
        elif peers is not None:
            # only this rank's CSR slice crosses PCIe; NVLink replicates it
            t_tok, t_off, vals, sk, h2d_rank[0] = embed_sharded_p2p_from_host(
                eparams, tok_pin, off_pin, w.d, skey, rank, world, peers, side_stream=side)
            emb = embedded_from_parts(eparams, t_tok, t_off, w.d, vals, sk, skey)
        else:
            t_tok = tok_pin.to(dev, non_blocking=True)
            t_off = off_pin.to(dev, non_blocking=True)
            emb = k1_sharded(t_tok, t_off)
        return join_sharded(emb)

    step_stats = {}

    def timed(fn, steps, probe=None):
        if world > 1:
            torch.distributed.barrier()
        # the join is host-driven (a few synchronisations per level): a
        # Python garbage-collection pause inside the timed region would idle
        # the device, so collect first and keep the collector off until the
        # region closes
        gc.collect()
        gc.disable()
        torch.cuda.synchronize()
        start = torch.cuda.Event(enable_timing=True)
        end = torch.cuda.Event(enable_timing=True)
        start.record(stream)
        out = None
        marks = []
        for i in range(steps):
            out = fn()
            marks.append(torch.cuda.Event(enable_timing=True))
            marks[-1].record(stream)
        end.record(stream)
        if probe is not None:
            # clock + throttle-reason sample as the timed region closes: any
            # NVML query issued while steps run stalled the device by 20-250 ms
            # in our measurements (profiles/README.md), so it is issued once
            # the last step is queued, before the closing synchronize
            probe()
        torch.cuda.synchronize()
        gc.enable()
        ms = start.elapsed_time(end)
        per = [a.elapsed_time(b) for a, b in zip([start] + marks[:-1], marks)]
        step_stats[getattr(fn, '__name__', 'step')] = {"min": min(per), "median": statistics.median(per),
                                                       "max": max(per)}
        log(f"[rank {rank}] {getattr(fn, '__name__', 'step')}: per-step ms min {min(per):.2f} "
            f"median {statistics.median(per):.2f} max {max(per):.2f} | " + " ".join(f"{x:.1f}" for x in per))
        if world > 1:
            t = torch.tensor([ms], device=dev) if torch.distributed.get_backend() == "nccl" else torch.tensor([ms])
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, out

    for _ in range(args.warmup):
        step_device()
        step_e2e()
    k1_events.clear()
    launches0 = ctx_launch_count(ctx)
    if args.clock_source == "smi":
        sampler = ClockSampler(dev.index, args.clock_ms)
    elif args.clock_source == "nvml":
        sampler = NvmlClockSampler(dev.index, args.clock_ms / 1e3)
    else:
        sampler = NvmlPointSampler(dev.index)
    probe = sampler.sample if isinstance(sampler, NvmlPointSampler) else None
    with sampler as clk:
        # nvidia-smi keeps perturbing the device for a while after its first
        # sample: run untimed steps for 3 s before the timed region
        t_settle = time.perf_counter()
        while time.perf_counter() - t_settle < 4.0:
            step_device()
            torch.cuda.synchronize()
        k1_events.clear()   # K1 launch times over the timed region only
        launches0 = ctx_launch_count(ctx)
        ms_dev, res = timed(step_device, args.steps, probe)
        launches = ctx_launch_count(ctx) - launches0
        # the e2e leg allocates its own device arrays (values, sketches, CSR):
        # untimed e2e steps first, so the caching allocator holds them before
        # the timed e2e region (at 10M sets the first e2e steps otherwise pay
        # GBs of fresh allocations)
        for _ in range(max(2, args.warmup)):
            step_e2e()
        torch.cuda.synchronize()
        ms_e2e, res_e2e = timed(step_e2e, args.steps, probe)
    value = n * args.steps / (ms_dev / 1e3)
    e2e_value = n * args.steps / (ms_e2e / 1e3)
    # the drop-in entry point (list[ResultPair]) once, outside the timed
    # region: what cpsjoin_self adds on top of the arrays form timed in e2e
    dropin_ms = None
    if world == 1:
        from paper_1707_06814_b200 import cpsjoin_self
        emb_d = embed_dataset(eparams, ds, sketch=skey)
        torch.cuda.synchronize()
        td = time.perf_counter()
        pairs_d, _ = cpsjoin_self(emb_d, params)
        dropin_ms = (time.perf_counter() - td) * 1e3
        del emb_d, pairs_d
    # per-kernel-class device time from one extra, separately profiled step
    ctx.profile(True)
    torch.cuda.synchronize()
    tp = time.perf_counter()
    step_device()
    torch.cuda.synchronize()
    wall_prof = (time.perf_counter() - tp) * 1e3
    prof = ctx.profile_read()
    ctx.profile(False)
    log(f"[rank {rank}] device step {ms_dev / args.steps:.2f} ms, e2e step {ms_e2e / args.steps:.2f} ms, "
        f"profiled step wall {wall_prof:.2f} ms: " + ", ".join(f"{k} {v[0]:.2f}" for k, v in prof.items()))

    # dominant kernel: K1 sketch launch (64 ell functions); algorithmic bytes
    # = CSR read once (4 nnz + 8 (n+1)) + sketch written (8 ell n)
    k1_val_ms = statistics.mean(a.elapsed_time(b) for a, b, _ in k1_events)
    k1_sk_ms = statistics.mean(b.elapsed_time(c) for _, b, c in k1_events)
    nnz = len(w.tokens)
    peaks = measured_peaks()
    sk_bytes = 4 * nnz + 8 * (n + 1) + 8 * cfg.ell * n
    achieved = sk_bytes / (k1_sk_ms / 1e3) / 1e9
    L = 1 if w.d <= 1 << 8 else 2 if w.d <= 1 << 16 else 3 if w.d <= 1 << 24 else 4
    f_clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    evals = nnz * 64 * cfg.ell
    # K1 keeps 16-bit hash entries in shared memory: L lookups x 2 B per
    # evaluation against the measured 126 B/clk/SM conflict-free LDS rate
    # (profiles/int_peaks_r01.json: LDS.64 15.76 lanes x 8 B per clk per SM)
    lookup_peak = 148 * f_clk * 126.0 / (2 * L)
    # with cached upper-byte entries (sorted tokens) a token needs T0 always,
    # T1 when tok >> 8 differs from its predecessor in the set, T2 when
    # tok >> 16 does: the minimum lookups per evaluation of this data
    tk = w.tokens
    first = np.zeros(len(tk), dtype=bool)
    first[w.offsets[:-1]] = True
    ch1 = np.ones(len(tk), dtype=bool)
    ch1[1:] = (tk[1:] >> 8) != (tk[:-1] >> 8)
    ch2 = np.ones(len(tk), dtype=bool)
    ch2[1:] = (tk[1:] >> 16) != (tk[:-1] >> 16)
    lookups_min = 1.0 + (float((ch1 | first).mean()) if L > 1 else 0.0) + (float((ch2 | first).mean()) if L > 2 else 0.0)
    lookup_peak_cached = 148 * f_clk * 126.0 / (2 * lookups_min)
    del first, ch1, ch2
    k4_ms = prof["k4_leaf"][0] + prof["point"][0]
    pre = res.counters.pre_candidates
    pairs_per_s = pre / (k4_ms / 1e3) if k4_ms > 0 else None
    popc_rate, popc_basis = int_peak("POPC", 16.0)
    popc_peak = 148 * popc_rate * f_clk / (2 * cfg.ell)  # 2 POPC per u64 word

    # ---- per-stage HBM rooflines from device-counted work:
    # bytes per unit x units counted by the join / profiled class time
    hbm = float(peaks["hbm_gbs"])
    st = res.stats
    visits, entries = int(st.get("internal_visits", 0)), int(st.get("split_entries", 0))
    vtok, ncand, nres = int(st.get("verify_tokens", 0)), int(res.counters.candidates), int(res.counters.results)

    def stage(bytes_, ms, unit_note, kernels):
        gbs = bytes_ / (ms / 1e3) / 1e9 if ms > 0 else None
        return {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": (gbs / hbm) if gbs else None,
                "algorithmic_bytes": int(bytes_), "ms_per_step": ms, "work": unit_note, "kernels": kernels}

    split_bytes = visits * (4 + 8 * cfg.ell + 4) + entries * (32 + 4 + 4)
    rooflines_stage = {
        "split": stage(split_bytes, prof["node"][0] + prof["split"][0],
                       f"{visits} internal-node member visits x (4 B id + {8 * cfg.ell} B sketch + 4 B survivor) + "
                       f"{entries} split entries x (32 B value-gather sector + 4 B survivor id + 4 B child member)",
                       "K2 node sketch/flags/survivors + K3 select/keys/sort/group/children + K7 subtree"),
        "verify": stage(4 * vtok + 16 * ncand + 16 * nres, prof["k5_verify"][0],
                        f"{ncand} candidates: 4 B x {vtok} row tokens + 16 B pair/offsets; 16 B per kept result",
                        "K5 k_verify"),
        "dedup": stage(16 * nres + 16 * int(len(res.a)), prof["k6_dedup"][0],
                       f"{nres} verified results read (u64 key + f64 sim) + {len(res.a)} unique written",
                       "K6 sort + unique"),
    }

    # ---- parity at benchmark scale: the timed device result, the e2e result
    # and the single-GPU join must agree bit for bit, and (one rank, N = 1,
    # full workload) with the C oracle port of the reference
    skeys = (single.a.astype(np.uint64) << np.uint64(32)) | single.b.astype(np.uint64)
    sc = single.counters
    scnt = [sc.pre_candidates, sc.candidates, sc.results, sc.max_depth, sc.peak_live_members]
    parity = {"device_vs_single_gpu": parity_check(res, skeys, single.similarity, scnt),
              "e2e_vs_single_gpu": parity_check(res_e2e, skeys, single.similarity, scnt)}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # the same algorithm on the host: the oracle port, all threads, same
        # R (bit-identical output, so the same recall) on the whole workload
        # when it fits the ~15 s budget, else on a scaled sample
        threads = cpu_threads()
        cscale = args.cpu_scale or cpu_sample_scale(args.config, threads) * args.scale
        if cscale > 0.8 * args.scale:
            cscale = args.scale
        cw = w if cscale == args.scale else generate(args.config, scale=cscale)
        arm = CpuArm(cw, cfg, threads)
        arm.lam = lam
        cdt, cout = arm.pipeline(R)
        crec = recall_of(cout.a, cout.b, truth) if cw is w else None
        cpu = {"value": cw.n / cdt, "unit": "sets/s", "cores": threads, "kind": "port",
               "sample": f"{cfg.name} x{cscale:g}: {cw.n} sets, embed+sketch+join R={R}"
                         + (f" (recall {crec:.3f})" if crec is not None else "") + f", {cdt:.2f} s"}
        if cw is not w and args.full_parity and not args.no_parity:
            # the timed CPU sample was a scaled workload: the oracle once more,
            # untimed, on the whole workload for the bit-exact comparison
            farm = CpuArm(w, cfg, threads)
            farm.lam = lam
            _, cout = farm.pipeline(R)
            cw = w
        if cw is w and not args.no_parity:
            ocnt = [cout.pre_candidates, cout.candidates, cout.results, cout.max_depth, cout.peak_live_members]
            parity["device_vs_oracle"] = parity_check(res, cout.keys, cout.sims, ocnt)
            parity["vs"] = "C oracle port of the reference on the full workload (same seeds, R)"
    elif rank == 0 and world == 1 and not args.no_parity:
        arm = CpuArm(w, cfg, cpu_threads())
        arm.lam = lam
        _, cout = arm.pipeline(R)
        ocnt = [cout.pre_candidates, cout.candidates, cout.results, cout.max_depth, cout.peak_live_members]
        parity["device_vs_oracle"] = parity_check(res, cout.keys, cout.sims, ocnt)
        parity["vs"] = "C oracle port of the reference on the full workload (same seeds, R)"
    parity["bit_exact"] = all(v["bit_exact"] for k, v in parity.items() if isinstance(v, dict))
    if not parity["bit_exact"]:
        log(f"[rank {rank}] PARITY FAILURE: {parity}")

    h2d_total = int(w.tokens.nbytes + w.offsets.nbytes)
    if world > 1:
        hb = torch.tensor([h2d_rank[0]], dtype=torch.int64,
                          device=dev if torch.distributed.get_backend() == "nccl" else "cpu")
        torch.distributed.all_reduce(hb)
        h2d_total = int(hb.item())
    d2h = int(len(res_e2e.a) * 16)
    line = {
        "metric": METRIC, "value": value, "unit": "sets/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_dev / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded generator for BASELINE.json config; Mann et al. datasets unavailable)",
        # config = the workload only, so both arms print the same dict
        "config": workload_dict(w, cfg, R, rec, lam, {"recall_truth": truth_src, "n_true_pairs": int(len(truth))}),
        "parallelism": ("single GPU" if world == 1 else
                        f"K1 set-sharded over {world} GPUs, rows stored to every GPU "
                        f"{'by the kernel over NVLink (fused all-gather)' if args.k1_transport == 'p2p' else 'by an NCCL all-gather'}; "
                        + (f"join frontier sharded at depth {args.frontier_depth} (size-balanced cut; every "
                           f"rank builds the levels above it) + pair gather" if args.join_shard == "frontier"
                           else "repetitions sharded round-robin + pair gather")),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
                     "frac": achieved / float(peaks["hbm_gbs"]), "traffic": ncu_traffic(args.config, "sketch"),
                     "kernel": "k_sketch_s16<L, PFX> sketch launch (K1, 64*ell functions)",
                     "algorithmic_bytes": sk_bytes, "avg_launch_ms": k1_sk_ms,
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)",
                     "note": "the dominant kernel is bound by shared-memory table lookups, not HBM: "
                             "roofline_smem.frac is its bound; HBM bytes are the CSR read + sketch write "
                             "(traffic = the token stream re-read once per 128-function chunk)"},
        "roofline_smem": {"bound": "shared-memory lookups (16-bit entries, 126 B/clk/SM measured LDS rate)",
                          "achieved_evals_per_s": evals / (k1_sk_ms / 1e3),
                          "peak_evals_per_s": lookup_peak_cached,
                          "frac": evals / (k1_sk_ms / 1e3) / lookup_peak_cached,
                          "lookups_per_eval_min": lookups_min,
                          "peak_evals_per_s_all_key_bytes": lookup_peak,
                          "frac_all_key_bytes": evals / (k1_sk_ms / 1e3) / lookup_peak, "key_bytes": L,
                          "values_launch_ms": k1_val_ms,
                          "note": "peak = 148 SMs x sm_max_mhz x 126 B/clk / (2 B x lookups per evaluation); "
                                  "lookups_per_eval_min counts T0 per token plus T1/T2 only where a sorted set's "
                                  "upper key bytes change (the kernel's cached-entry path); frac_all_key_bytes is "
                                  "round 1's denominator (every key byte looked up for every token) and can "
                                  "exceed 1.  ncu of the same launch (profiles/ncu_k1_s16_r02_c2.csv): shared "
                                  "wavefronts 88% of peak incl. the token shuffles, ALU pipe 76%, issue 74%"},
        "roofline_int": {"kernel": "k_leaf_tiles + k_point (K4 BruteForce)", "pairs_per_s": pairs_per_s,
                         "peak_pairs_per_s": popc_peak,
                         "frac": (pairs_per_s / popc_peak) if pairs_per_s else None,
                         "peak_basis": f"POPC {popc_rate:.2f}/clk/SM ({popc_basis}) x 148 x sm_max_mhz / (2 ell)",
                         "note": "naive bound (2 ell POPC per pair); the kernels count 32-bit words in triplets "
                                 "(popc(x^y^z) + 2 popc(maj)), 1.5 ell POPC per fully compared pair, and exit "
                                 "early after 5/8 of the words for most pairs, so they can exceed frac 1"},
        "roofline_stages": rooflines_stage,
        "kernels_ms_per_step": {k: v[0] for k, v in prof.items()},
        "kernels_note": "device time per class from one extra profiled step (events around each class)",
        "per_step_ms": step_stats,
        "join_counters": {"pre_candidates": pre, "candidates": res.counters.candidates,
                          "results": res.counters.results, "max_depth": res.counters.max_depth,
                          "pairs": int(len(res.a))},
        "parity": parity,
        "e2e": {"value": e2e_value, "unit": "sets/s", "h2d_bytes_per_step": h2d_total, "d2h_bytes_per_step": d2h,
                "ms_per_step": ms_e2e / args.steps,
                "api": ("embed_dataset(EmbeddingParams, Dataset, sketch=(ell, seed)) + cpsjoin_self_arrays "
                        "(the drop-in's array form; cpsjoin_self builds list[ResultPair] from it)" if world == 1 else
                        "embed_sharded_p2p_from_host (each rank copies only its CSR slice host->device, "
                        "NVLink replicates it) + shard_frontier"),
                "h2d_bytes_per_rank": h2d_rank[0],
                "dropin_cpsjoin_self_ms": dropin_ms},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
        "impl": "ours",
    }
    if args.dist_backend == "gloo" and world > 1:
        line["functional_only"] = ("gloo backend: collectives staged through the host, possibly several ranks on "
                                   "one GPU -- a functional check of the N-rank path, not a bench number")
    if rank == 0:
        print(json.dumps(line), flush=True)


def ctx_launch_count(ctx) -> int:
    """Own kernels launched so far on this context (K1 + join kernels)."""
    return ctx.launch_counts()[0]


def relaunch_under_torchrun(n: int) -> None:
    """`python bench.py --gpus N` (N > 1) without a launcher: re-execute
    this command under torch.distributed.run with N ranks on this node (the
    same launch the driver uses), so --gpus always means N processes."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log(f"bench: --gpus {n} without WORLD_SIZE: relaunching as {' '.join(cmd[1:6])} ...")
    sys.stdout.flush()
    sys.stderr.flush()
    os.execv(sys.executable, cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > torch.cuda.device_count() and args.dist_backend == "nccl":
        raise SystemExit(f"bench: {world} ranks but {torch.cuda.device_count()} GPU(s); NCCL needs one GPU per "
                         "rank (--dist-backend gloo runs the N-rank path functionally on fewer GPUs)")
    if args.dist_backend == "gloo":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            torch.distributed.init_process_group("gloo")
    try:
        run_ours(args, rank, world)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
