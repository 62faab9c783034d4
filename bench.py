#!/usr/bin/env python
"""DDCCANet fit+transform throughput on B200 (images/s), one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload caltech256] [--impl ours|reference]

A step = one full DDCCANet fit (layer-wise moments -> NCCL reduction ->
device solve, for every layer) plus one full transform (forward + sign hash
+ block histograms) over the workload's M synthetic images. `value` is
device-resident throughput (inputs already in HBM, block counts left in
HBM); `e2e` is the same work through the public API with host buffers:
pinned-host -> device copy of the images and a device -> host copy of the
feature counts inside the timed region. Multi-GPU (torchrun): samples are
sharded by whole 128-sample batches (weak scaling would be --weak; default
is the fixed M of the named workload, i.e. strong scaling over the corpus).

`--impl reference` times the reference algorithm on the host cores: the CPU
oracle (oracle/, a numpy restatement of ddccanet pinned to golden vectors of
the reference) on a bounded sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = ("orl", "eth80", "caltech256", "caltech256x10", "three_stage")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="caltech256", choices=WORKLOADS)
    ap.add_argument("--m", type=int, default=None, help="override the number of images")
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-sample", type=int, default=64, help="images in the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--deterministic", type=int, default=1)
    ap.add_argument("--classify", action="store_true",
                    help="also run the device NN classifier on the step's counts (accuracy, fp64 GEMM rate)")
    ap.add_argument("--moments", default="blocked", choices=("exact", "blocked"),
                    help="lag-product precision of layers >= 2 (ExecSettings.moments)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def compute_peaks(sm_mhz: float):
    """FP32 / FP64 / TF32-tensor peaks: profiles/round2_peaks.json (tools/measure_peaks.py, measured on
    this pool's B200 at its max clock) scaled to the clock the timed region ran at; else derived."""
    sms = 148
    out = {"ffma_tflops": sms * 128 * 2 * sm_mhz * 1e6 / 1e12, "dfma_tflops": sms * 64 * 2 * sm_mhz * 1e6 / 1e12,
           "tf32_tflops": sms * 4096 * sm_mhz * 1e6 / 1e12, "source": "derived (148 SMs x per-clock rate x clock)"}
    f = ROOT / "profiles" / "round2_peaks.json"
    if f.exists():
        d = json.loads(f.read_text())
        # the issue-rate ceilings (256 FFMA / 128 DFMA flop per clock per SM) stay the denominators when a
        # microbenchmark falls short of them (the DMMA path reaches 127 of 128 FP64 flop per clock)
        for key, ceil in (("ffma", 256.0), ("dfma", 128.0)):
            per_clk = max(ceil, d.get(f"{key}_flop_per_clk_per_sm") or 0.0)
            out[f"{key}_tflops"] = sms * per_clk * sm_mhz * 1e6 / 1e12
        if d.get("tf32_flop_per_clk_per_sm"):
            out["tf32_tflops"] = sms * d["tf32_flop_per_clk_per_sm"] * sm_mhz * 1e6 / 1e12
        out["source"] = ("max(issue ceiling, profiles/round2_peaks.json microbenchmark) flop per clock per SM for "
                         "FFMA / DFMA, measured tcgen05 TF32 MMA rate (tc_probe) x 148 SMs x the median SM clock "
                         f"{sm_mhz:.0f} MHz of the timed region")
    return out


# ---------------------------------------------------------------------------- clocks

class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region (NVML, else nvidia-smi -lms 100)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def _nvml_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")
        if vis and vis[0].strip().isdigit() and self.idx < len(vis):
            return int(vis[self.idx])
        return self.idx

    def _poll_nvml(self, nv, h):
        """NVML every 2 ms: short timed regions (ORL: ~20 ms) still get samples."""
        names = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                 ("sw_power_cap", 0x4))
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = get_reasons(h)
            except Exception:
                break
            self.rows.append(["", str(sm), str(mx), "", ""] + ["Active" if bits & b else "Not Active" for _, b in names])
            self._first.set()
            if self._halt.wait(0.002):
                break

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self._nvml_index())
            self._halt = threading.Event()
            self._first = threading.Event()
            self.thread = threading.Thread(target=self._poll_nvml, args=(nv, h), daemon=True)
            self.nvml = True
            self.thread.start()
            self._first.wait(1.0)  # at least one sample before the timed region starts
            return
        except Exception:
            self.nvml = False
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if getattr(self, "nvml", False):
            self._halt.set()
            self.thread.join(timeout=5)
        elif self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        else:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for k, nm in enumerate(names):
                if r[5 + k].lower() == "active":
                    reasons.add(nm)
        load = [s for s in sm if s > 500] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "source": "nvml 2 ms" if getattr(self, "nvml", False) else "nvidia-smi 100 ms"}


# ---------------------------------------------------------------------------- CPU reference (oracle)

def cpu_reference(workload: str, n_img: int, threads: int, reps: int = 1, warm: int = 0, seed: int = 0):
    """Oracle fit + transform on a bounded sample; returns (img/s list, sample description, threads)."""
    from threadpoolctl import threadpool_limits

    import oracle as O
    from paper_2209_13027_b200 import synthetic

    cfg = synthetic.CONFIGS[workload]
    v1, lab = synthetic.blob_images(n_img, cfg["p"], cfg["q"], cfg["classes"], seed=seed)
    v2 = synthetic.second_view(v1, lab, cfg["view2"], cfg["classes"], seed=seed + 1)
    v1, v2 = v1.astype(np.float64), v2.astype(np.float64)
    classes = cfg["classes"]
    specs = [(L, O.Geometry(l1, l2), True) for L, l1, l2 in cfg["layers"]]
    enc = O.EncodeCfg(*cfg["block"])
    # the reference parallelizes over sample batches (execution.py:41-57): use one batch per thread
    batch = max(1, -(-n_img // threads))
    rates = []
    with threadpool_limits(limits=1), O.Pool(threads=threads) as pool:
        for i in range(warm + reps):
            t0 = time.perf_counter()
            layers = O.train(v1, v2, lab, classes, specs, batch=batch, pool=pool)
            O.features(v1, v2, layers, enc, batch=batch, pool=pool)
            dt = time.perf_counter() - t0
            if i >= warm:
                rates.append(n_img / dt)
    sample = (f"{n_img} images of the {workload} workload ({cfg['p']}x{cfg['q']}, {classes} classes), "
              f"fit+transform by the numpy oracle, {threads} threads (batch {batch}/thread, BLAS 1 thread)")
    return rates, sample


def cpu_baseline(workload: str, sample: int, reps: int = 3):
    """The reference algorithm on this box's host cores: all cores (one sample batch
    per thread, median of `reps`) and one thread (one batch, the reference's run_bench pinning)."""
    threads = os.cpu_count() or 1
    rates, desc = cpu_reference(workload, sample, threads, reps=reps)
    one_n = max(4, min(16, sample // 4))
    one, one_desc = cpu_reference(workload, one_n, 1, reps=1)
    return {"value": statistics.median(rates), "unit": "images/s", "cores": threads, "kind": "port",
            "sample": desc, "runs": rates, "median_of": len(rates),
            "one_thread": {"value": one[0], "unit": "images/s", "cores": 1, "sample": one_desc},
            "note": "oracle/ is a numpy restatement of the reference's calls (same numpy/BLAS operations, pinned to "
                    "golden vectors of the unmodified reference); profiles/round2_port_vs_reference.json times it "
                    "against the unmodified reference on one sample"}


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_img = min(args.cpu_sample, 64)
    rates, sample = cpu_reference(args.workload, n_img, threads, reps=args.steps, warm=args.warmup)
    v = statistics.median(rates)
    one_n = max(4, min(16, n_img // 4))
    one, one_desc = cpu_reference(args.workload, one_n, 1, reps=1)
    from paper_2209_13027_b200 import synthetic

    cfg = synthetic.CONFIGS[args.workload]
    line = {
        "metric": "images/sec fit+transform", "value": v, "unit": "images/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * n_img / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "images": cfg["m"], "sample_images": n_img,
                   "image": [cfg["p"], cfg["q"]], "classes": cfg["classes"], "layers": cfg["layers"],
                   "block": cfg["block"]},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": threads, "kind": "port", "sample": sample,
                         "runs": rates, "one_thread": {"value": one[0], "unit": "images/s", "cores": 1,
                                                       "sample": one_desc}},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm

def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import torch.distributed as dist

    import paper_2209_13027_b200 as P
    from paper_2209_13027_b200 import engine as E
    from paper_2209_13027_b200 import synthetic
    from paper_2209_13027_b200.execution import shard_range

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = synthetic.CONFIGS[args.workload]
    M = args.m or cfg["m"]
    p, q, classes = cfg["p"], cfg["q"], cfg["classes"]
    bs = 128
    nb = -(-M // bs)
    mine = shard_range(nb, rank, world)
    s0, s1 = min(M, mine.start * bs), min(M, mine.stop * bs)  # a rank may own no batch (s0 == s1)
    ex = P.Executor(P.ExecSettings(deterministic=bool(args.deterministic), moments=args.moments), device=local_rank)
    layer_cfgs = [P.LayerConfig(L, P.PatchGeometry(l1, l2)) for L, l1, l2 in cfg["layers"]]
    enc = P.EncoderConfig(*cfg["block"])

    # synthetic corpus for this rank's shard, generated on the device (not timed)
    with torch.cuda.stream(ex.stream):
        img1, lab = synthetic.blob_images_device(M, p, q, classes, seed=0, device=dev, start=s0, stop=s1)
        img2 = synthetic.second_view_device(img1, cfg["view2"], seed=1, executor=ex)
        labels = torch.from_numpy(lab.astype(np.int32)).to(dev)
    ex.synchronize()

    eng = E.Engine(ex)
    prof = {}
    eng.profile = prof

    plan, groups, featlen = eng.feature_geometry(p, q, [E.DeviceLayer(c.geom, True, c.filters, None, None, None,
                                                                      None, None) for c in layer_cfgs], enc)
    kind = E.count_kind(plan.bpc)
    out_bytes = (s1 - s0) * featlen * (2 if kind == 2 else 1)
    stream_counts = out_bytes > (48 << 30)  # e.g. 3-stage: counts are digested per super-batch, never stored whole
    digest = torch.zeros(1, dtype=torch.int64, device=dev)

    def sink(a, b, counts):
        digest.add_(counts.view(torch.uint8)[:, :4096].sum())  # keeps every super-batch's output live

    counts_buf = [None if stream_counts else torch.empty((s1 - s0, featlen), dtype=torch.int16 if kind == 2 else
                                                         torch.uint8, device=dev)]
    # inputs smaller than L2 are flushed between steps (write > L2 bytes)
    in_bytes = 2 * (s1 - s0) * p * q * 4
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if in_bytes < (256 << 20) else None

    def step():
        if flush is not None:
            with torch.cuda.stream(ex.stream):
                flush.fill_(1)
        res = eng.fit(img1, img2, labels, classes, layer_cfgs, bs, 1e-4, n_global=M, first_sample=s0)
        counts, plan_ = eng.transform_counts(img1, img2, res.layers, enc, bs, out=counts_buf[0],
                                             sink=sink if stream_counts else None)
        return counts, plan_

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        step()
    ex.synchronize()
    prof.clear()
    eng.work.clear()
    eng.launches = 0
    barrier()
    torch.cuda.synchronize()
    clk = ClockSampler(local_rank)
    clk.start()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(ex.stream)
    for _ in range(args.steps):
        step()
    t_end.record(ex.stream)
    t_end.synchronize()
    barrier()
    torch.cuda.synchronize()
    clocks = clk.stop()
    ms = t_start.elapsed_time(t_end) / args.steps
    launches = eng.launches // max(1, args.steps)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = M / (ms_max / 1000.0)

    # per-kernel shares (events bracket single-kernel C-ABI calls on the same stream)
    kern = {}
    for name, evs in prof.items():
        times = [a.elapsed_time(b) for a, b in evs]
        w = dict(eng.work.get(name) or {})
        if w.get("calls"):
            # per-launch algorithmic work = total over the timed steps / launches
            for key in ("flops", "bytes", "gram_flops", "tensor_flops"):
                if key in w:
                    w[key] = w[key] / w["calls"]
        kern[name] = {"ms_avg": sum(times) / len(times), "launches": len(times),
                      "ms_per_step": sum(times) / args.steps, "work": w or None}

    # optional downstream check: NN classifier on the step's device counts,
    # half the images as training rows (every class on both sides), accuracy + fp64 GEMM rate
    downstream = None
    if args.classify and world == 1 and counts_buf[0] is not None:
        cls_of = np.arange(s1 - s0) // classes % 2 == 0
        tr_idx = torch.from_numpy(np.nonzero(cls_of)[0]).to(dev)
        te_idx = torch.from_numpy(np.nonzero(~cls_of)[0]).to(dev)
        lab_h = lab.astype(np.int64)
        with torch.cuda.stream(ex.stream):
            ctr = counts_buf[0].index_select(0, tr_idx)
            cte = counts_buf[0].index_select(0, te_idx)
        model = P.classify.fit(P.CountFeatures(ctr, plan, enc), lab_h[cls_of], executor=ex)
        ex.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(ex.stream)
        rep = P.classify.evaluate(model, P.CountFeatures(cte, plan, enc), lab_h[~cls_of], executor=ex)
        b.record(ex.stream)
        b.synchronize()
        t_ms = a.elapsed_time(b)
        flop = 2.0 * int(cls_of.sum()) * int((~cls_of).sum()) * featlen
        sm_mhz = (clocks.get("sm_mhz") or 1965.0)
        peak64 = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12
        downstream = {"classifier": "nearest_neighbor euclidean on device counts (classify.py:109-143)",
                      "train": int(cls_of.sum()), "test": int((~cls_of).sum()), "accuracy": rep.accuracy,
                      "ms": t_ms, "tflops_fp64": flop / (t_ms / 1e3) / 1e12, "peak_fp64_tflops": peak64,
                      "frac": flop / (t_ms / 1e3) / 1e12 / peak64}
        del ctr, cte, model

    # e2e through the public API with host buffers
    e2e = None
    eng.maps_cache = None
    del counts_buf[:]
    torch.cuda.empty_cache()
    if stream_counts:
        e2e = {"value": None, "unit": "images/s", "unavailable": "feature counts (%.0f GB) exceed host memory; "
               "device run digests them per super-batch" % (out_bytes / 1e9)}
    elif not args.no_e2e:
        h1 = img1.cpu().pin_memory()
        h2 = img2.cpu().pin_memory()
        hl = torch.from_numpy(lab.astype(np.int64))
        host_counts = torch.empty((s1 - s0, featlen), dtype=torch.int16 if kind == 2 else torch.uint8).pin_memory()
        # this rank's rows of the M-image dataset (pinned: chunked async upload)
        ds = P.ViewPairDataset.shard(h1, h2, hl.numpy(), s0, M, classes)
        net = P.NetworkConfig(tuple(layer_cfgs), batch=P.BatchSpec(bs))
        pcfg = type("Cfg", (), {"net": net, "encoder": enc})()

        def e2e_step():
            bank = P.train_network(ds, net, ex)
            P.compute_feature_counts(ds, bank, pcfg, ex, host_out=host_counts)
            ds._device_state = None  # next step uploads again (H2D inside the timed region)
            return bank

        for _ in range(max(1, min(2, args.warmup))):
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        # timed on the caller's (current) stream: compute_feature_counts orders it after the
        # executor's kernels AND the streamed device->host copies of every step, while the
        # executor's stream runs ahead into the next step's upload + fit (steps pipeline over
        # PCIe: step k's counts download while step k+1's images upload)
        cur = torch.cuda.current_stream(dev)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(cur)
        for _ in range(args.steps):
            e2e_step()
        cur.wait_stream(ex.stream)
        b.record(cur)
        b.synchronize()
        wall = (time.perf_counter() - t0) / args.steps
        ms_e = max(a.elapsed_time(b) / args.steps, wall * 1000.0)
        t = torch.tensor([ms_e], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        # whole-job bytes per step (every rank copies its own shard's images in and counts out)
        h2d = 2 * M * p * q * 4 + M * 8
        d2h = M * featlen * host_counts.element_size()
        e2e = {"value": M / (float(t.item()) / 1000.0), "unit": "images/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(t.item())}

    if rank != 0:
        return
    pk, pk_kind = peaks()
    sm_mhz = clocks.get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    cp = compute_peaks(sm_mhz)

    def kernel_roofline(name):
        k = kern[name]
        w = k["work"] or {}
        if not w.get("flops") and not w.get("bytes"):
            return None
        t = k["ms_avg"] / 1e3
        ach = w.get("flops", 0.0) / t / 1e12
        r = {"kernel": name, "share_of_step": k["ms_per_step"] / ms, "ms_per_launch": k["ms_avg"]}
        if w.get("kind") == "tensor":
            # algorithmic flops = the convolution's own 2 * taps * filters per pixel (single pass);
            # executed = what the tensor pipe ran (two-term f16 split: 3 MMAs per product, banded B of
            # K = 16 per tap row). peak = the measured dense bf16 rate (MEASURED_PEAKS.json; kind::f16
            # runs at the bf16 rate); f16_mma_tflops = the tcgen05 f16 rate at this clock (2x the
            # measured TF32 MMA rate: a K16 f16 MMA takes the cycles of a K8 tf32 one, f16_probe.cu)
            ex_tf = w.get("tensor_flops", 0.0) / t / 1e12
            f16 = 2.0 * cp["tf32_tflops"]
            r.update({"bound": "tensor", "achieved": ach, "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
                      "frac": ach / pk["bf16_tflops"], "executed_tflops": ex_tf, "f16_mma_tflops": f16,
                      "tensor_pipe_frac": ex_tf / f16, "vs_ffma_peak": ach / cp["ffma_tflops"],
                      "note": "tcgen05 kind::f16, power-of-two scaled two-term split (3 MMAs per product) x "
                              "banded B (16 K columns per 7 taps): executed = 6.9x algorithmic at 7x7; "
                              "tensor_pipe_frac = executed over the f16 MMA rate; vs_ffma_peak = algorithmic "
                              "rate over the FP32 CUDA-core peak the FFMA kernel is capped by"})
        elif w.get("kind") == "fma":
            r.update({"bound": "fp32_fma", "achieved": ach, "peak": cp["ffma_tflops"], "unit": "TFLOP/s",
                      "frac": ach / cp["ffma_tflops"]})
        elif w.get("kind") == "fp64":
            r.update({"bound": "fp64_fma", "achieved": ach, "peak": cp["dfma_tflops"], "unit": "TFLOP/s",
                      "frac": ach / cp["dfma_tflops"]})
        elif w.get("kind") == "hbm":
            gbs = w["bytes"] / t / 1e9
            r.update({"bound": "hbm", "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                      "frac": gbs / pk["hbm_gbs"]})
        if w.get("bytes"):
            r["hbm_achieved_gbs"] = w["bytes"] / t / 1e9
            r["hbm_peak_gbs"] = pk["hbm_gbs"]
        return r

    rooflines = {n: r for n in kern for r in [kernel_roofline(n)] if r is not None}
    roof = None
    if rooflines:
        top = max(rooflines, key=lambda n: kern[n]["ms_per_step"])
        roof = dict(rooflines[top])
        roof["traffic"] = None
    # DDCCA statistics in the full-GEMM convention (2 views x 2 d^2 per patch), i.e. the
    # work a 3xTF32 tcgen05 Gram would do: a GEMM-equivalent rate, not tensor-pipe use (the exact lag
    # form runs on the FP64 pipe and uses no tensor cores)
    gram = None
    mom = [k for k in kern if k.startswith("moments_l") and (kern[k]["work"] or {}).get("gram_flops")]
    if mom:
        gfl = sum(kern[k]["work"]["gram_flops"] * kern[k]["launches"] / args.steps for k in mom)
        gms = sum(kern[k]["ms_per_step"] for k in mom)
        tf32 = cp["tf32_tflops"]
        ach = gfl / (gms / 1e3) / 1e12
        gram = {"kernels": mom, "gemm_equiv_flop_per_step": gfl, "ms_per_step": gms,
                "gemm_equiv_tflops": ach, "tf32_dense_peak_tflops": tf32,
                "gemm_equiv_frac_of_tf32_peak": ach / tf32, "gemm_equiv_frac_of_3xtf32_ceiling": ach / (tf32 / 3.0),
                "tensor_pipe_used": False,
                "note": "GEMM-equivalent bookkeeping: the exact FP64 lag form (85 DFMA per pixel at 7x7) does the "
                        "statistics a 3xTF32 Gram (2 d^2 = 4802 flop per patch) would; this is the Gram-convention "
                        "rate, the tensor pipe is idle in these kernels"}
    # DRAM bytes per launch of the same kernels from the committed ncu launch list
    tf = ROOT / "profiles" / "traffic.json"
    tfd = json.loads(tf.read_text()) if tf.exists() else {}
    for r in ([roof] if roof is not None else []) + list(rooflines.values()):
        name = r["kernel"]
        conv_k = "conv_resp_tc_kernel" if r.get("bound") == "hbm" else "conv_c_kernel"
        lag_k = "lag_tma_blk_kernel" if r.get("bound") == "fp32_fma" else "lag_tma_kernel"
        kname = {"conv_hist": "conv_hist_tc_kernel" if r.get("bound") == "tensor" else "conv_hist_kernel",
                 "conv_l1": conv_k, "conv_l2": conv_k}.get(name, lag_k if name.startswith("moments") else name)
        k = tfd.get("kernels", {}).get(kname) if tfd.get("workload", "caltech256") == args.workload else None
        if k:
            r["traffic"] = k["dram_bytes_per_launch"]
            r["traffic_unit"] = "bytes/launch (dram read+write)"
            r["traffic_source"] = "profiles/traffic.json: " + tfd.get("source", "")
            w = kern[name]["work"] or {}
            if w.get("bytes"):
                r["algorithmic_bytes"] = w["bytes"]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(args.workload, args.cpu_sample)
    line = {
        "metric": "images/sec fit+transform", "value": value, "unit": "images/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 stats/solve, f32 conv", "data": "synthetic",
        "config": {"workload": args.workload, "images": M, "image": [p, q], "classes": classes,
                   "layers": cfg["layers"], "block": cfg["block"], "batch": bs, "featlen": featlen,
                   "counts": ["u8", "u8-saturating", "u16"][kind], "parallelism": f"dp{world} (sample shards)",
                   "l2_flush": ("inputs (%.1f GB) larger than L2" % (in_bytes / 1e9)) if flush is None else
                               "256 MB L2 flush write before every step (inputs smaller than L2)",
                   "counts_output": "streamed+digested per super-batch" if stream_counts else "kept in HBM",
                   "deterministic": bool(args.deterministic)},
        "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "roofline": roof, "cpu_baseline": cpu, "gram": gram,
        "downstream": downstream,
        "kernels": kern, "rooflines": rooflines, "peaks_source": pk_kind, "compute_peaks": cp,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("DDCCA_BENCH_GLOO") == "1":
            # functional dry run of the multi-rank path with fewer GPUs than ranks (host-side
            # gloo collectives; no kernel waits on another rank). Never a performance number.
            local_rank = local_rank % torch.cuda.device_count()
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
