"""Time the oracle port (oracle/, the bench's CPU baseline) against the UNMODIFIED reference on the same sample.

Runs in the build container (the reference lives at /root/reference, read-only;
it is not on the GPU box, which is why the bench times the port there):

    python -B tools/port_vs_reference.py > profiles/round2_port_vs_reference.json

Same inputs (the bench's synthetic generator), same decomposition (batch per
thread), BLAS pinned to one thread per worker as the reference's run_bench
does (pipeline.py:282); fit = train_network, transform = compute_features.
"""
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))


def main():
    from threadpoolctl import threadpool_limits

    from make_golden import _import_reference
    import oracle as O
    from paper_2209_13027_b200 import synthetic

    dd = _import_reference()
    from ddccanet.pipeline import compute_features

    threads = min(8, os.cpu_count() or 1)
    out = {"host_cores": os.cpu_count(), "threads": threads, "runs": []}
    for workload, n in (("orl", 64), ("caltech256", 32)):
        cfg = synthetic.CONFIGS[workload]
        v1, v2, lab, _ = synthetic.make_corpus(workload, m=n)
        v1, v2 = v1.astype(np.float64), v2.astype(np.float32).astype(np.float64)
        batch = max(1, -(-n // threads))
        # reference
        samples = [dd.ViewPairSample(view1=a, view2=b, label=int(c)) for a, b, c in zip(v1, v2, lab)]
        ds = dd.ViewPairDataset(samples=samples, class_count=cfg["classes"])
        net = dd.NetworkConfig(layers=tuple(dd.LayerConfig(L, dd.PatchGeometry(l1, l2)) for L, l1, l2 in cfg["layers"]),
                               batch=dd.BatchSpec(batch))
        pcfg = type("Cfg", (), {"net": net, "encoder": dd.EncoderConfig(*cfg["block"])})()
        t_ref, t_port = [], []
        for _ in range(2):
            with threadpool_limits(1), dd.Executor(dd.ExecSettings(threads=threads)) as ex:
                t0 = time.perf_counter()
                bank = dd.train_network(ds, net, ex)
                f_ref = compute_features(ds, bank, pcfg, ex)
                t_ref.append(time.perf_counter() - t0)
            specs = [(L, O.Geometry(l1, l2), True) for L, l1, l2 in cfg["layers"]]
            with threadpool_limits(1), O.Pool(threads=threads) as pool:
                t0 = time.perf_counter()
                layers = O.train(v1, v2, lab, cfg["classes"], specs, batch=batch, pool=pool)
                f_port = O.features(v1, v2, layers, O.EncodeCfg(*cfg["block"]), batch=batch, pool=pool)
                t_port.append(time.perf_counter() - t0)
        rec = {"workload": workload, "images": n, "batch": batch, "reference_s": t_ref, "port_s": t_port,
               "reference_img_s": n / min(t_ref), "port_img_s": n / min(t_port),
               "port_over_reference_time": min(t_port) / min(t_ref),
               "features_identical_frac": float(np.mean(f_ref == f_port))}
        out["runs"].append(rec)
        print(json.dumps(rec), file=sys.stderr)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
