"""Timeline of the e2e step (bench.py's `e2e`): copies and kernels per step from torch.profiler
(CUPTI), to see what of the PCIe traffic overlaps the device work (GPU).

python tools/e2e_timeline.py [workload] [steps]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402
from paper_2209_13027_b200 import synthetic  # noqa: E402


def union(iv):
    tot, end = 0.0, -1e30
    for a, b in sorted(iv):
        if b <= end:
            continue
        tot += b - max(a, end)
        end = b
    return tot


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "caltech256"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cfg = synthetic.CONFIGS[wl]
    M, p, q, classes = cfg["m"], cfg["p"], cfg["q"], cfg["classes"]
    dev = torch.device("cuda", 0)
    ex = P.Executor(P.ExecSettings())
    with torch.cuda.stream(ex.stream):
        img1, lab = synthetic.blob_images_device(M, p, q, classes, seed=0, device=dev, start=0, stop=M)
        img2 = synthetic.second_view_device(img1, cfg["view2"], seed=1, executor=ex)
    ex.synchronize()
    layer_cfgs = [P.LayerConfig(L, P.PatchGeometry(l1, l2)) for L, l1, l2 in cfg["layers"]]
    enc = P.EncoderConfig(*cfg["block"])
    eng = E.Engine(ex)
    plan, groups, featlen = eng.feature_geometry(p, q, [E.DeviceLayer(c.geom, True, c.filters, None, None, None,
                                                                      None, None) for c in layer_cfgs], enc)
    kind = E.count_kind(plan.bpc)
    h1, h2 = img1.cpu().pin_memory(), img2.cpu().pin_memory()
    del img1, img2
    torch.cuda.empty_cache()
    host_counts = torch.empty((M, featlen), dtype=torch.int16 if kind == 2 else torch.uint8).pin_memory()
    ds = P.ViewPairDataset.shard(h1, h2, lab.astype(np.int64), 0, M, classes)
    net = P.NetworkConfig(tuple(layer_cfgs), batch=P.BatchSpec(128))
    pcfg = type("Cfg", (), {"net": net, "encoder": enc})()

    def step():
        bank = P.train_network(ds, net, ex)
        P.compute_feature_counts(ds, bank, pcfg, ex, host_out=host_counts)
        ds._device_state = None
        return bank

    step()
    torch.cuda.synchronize()
    # host-side duration of each public call (a call that blocks on the device shows up here)
    for _ in range(2):
        t = time.perf_counter()
        bank = P.train_network(ds, net, ex)
        t1 = time.perf_counter()
        P.compute_feature_counts(ds, bank, pcfg, ex, host_out=host_counts)
        t2 = time.perf_counter()
        ds._device_state = None
        t3 = time.perf_counter()
        print(f"host: train_network {1e3 * (t1 - t):.1f} ms, compute_feature_counts {1e3 * (t2 - t1):.1f} ms, "
              f"release {1e3 * (t3 - t2):.1f} ms")
    torch.cuda.synchronize()
    marks = []
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                            torch.profiler.ProfilerActivity.CPU]) as prof:
        for _ in range(steps):
            marks.append(time.perf_counter())
            step()
        torch.cuda.synchronize()
        marks.append(time.perf_counter())
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    kern, h2d, d2h = [], [], []
    for e in ev:
        iv = (e.time_range.start / 1e3, e.time_range.end / 1e3)  # ms
        n = e.name.lower()
        if "memcpy" in n and ("htod" in n or "host to device" in n):
            h2d.append(iv)
        elif "memcpy" in n and ("dtoh" in n or "device to host" in n):
            d2h.append(iv)
        elif "memcpy" not in n and "memset" not in n:
            kern.append(iv)
    t0 = min(a for a, _ in kern + h2d + d2h)
    t1 = max(b for _, b in kern + h2d + d2h)
    print(f"{steps} steps: span {t1 - t0:.1f} ms = {(t1 - t0) / steps:.1f} ms/step")
    for name, iv in (("kernels", kern), ("H2D", h2d), ("D2H", d2h)):
        print(f"  {name:8s} busy {union(iv):8.1f} ms ({len(iv)} ops)")
    both = []
    for a, b in d2h:
        for c, d in kern:
            lo, hi = max(a, c), min(b, d)
            if lo < hi:
                both.append((lo, hi))
    print(f"  D2H overlapped with kernels {union(both):.1f} ms")
    # coarse timeline: 10 ms bins, which engines are busy
    nb = int((t1 - t0) // 10) + 1
    line = {"K": np.zeros(nb), "U": np.zeros(nb), "D": np.zeros(nb)}
    for key, iv in (("K", kern), ("U", h2d), ("D", d2h)):
        for a, b in iv:
            for k in range(int((a - t0) // 10), int((b - t0) // 10) + 1):
                lo, hi = max(a, t0 + 10 * k), min(b, t0 + 10 * k + 10)
                if hi > lo:
                    line[key][k] += hi - lo
    for key in ("K", "U", "D"):
        print(key, "".join("#" if v > 7 else ("+" if v > 3 else ("." if v > 0 else " ")) for v in line[key]))
    # host marks (profiler clock is not the perf_counter clock: print relative spacing only)
    print("host step starts (ms from first):", [round(1e3 * (m - marks[0]), 1) for m in marks])
    for name, iv in (("K", kern), ("U", h2d), ("D", d2h)):
        segs = []
        for a, b in sorted(iv):
            if segs and a - segs[-1][1] < 2.0:
                segs[-1][1] = max(segs[-1][1], b)
            else:
                segs.append([a, b])
        print(name, "segments (ms):", [(round(a - t0, 1), round(b - t0, 1)) for a, b in segs if b - a > 1.0][:12])


if __name__ == "__main__":
    main()
