"""Throughput of the device NN classifier on count rows (diagnostic, also used for DESIGN numbers).

Usage: python tools/nn_bench.py [n_train] [n_query] [featlen]
Counts are random valid u8 histograms (16x16 blocks, 256 bins); time = one
predict_many over all queries (GEMM + epilogue + argmin), CUDA events.
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import engine as E  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 262144
enc = P.EncoderConfig(4, 4)  # bpc 16: u8 counts
plan = E.block_plan(enc, 64, 64, 8)
ex = P.Executor(P.ExecSettings())
g = torch.Generator(device="cuda").manual_seed(0)
tr = torch.randint(0, 17, (nt, dim), dtype=torch.uint8, device="cuda", generator=g)
qu = torch.randint(0, 17, (nq, dim), dtype=torch.uint8, device="cuda", generator=g)
labels = np.arange(nt) % 97
model = P.classify.fit(P.CountFeatures(tr, plan, enc), labels, executor=ex)
P.classify.predict_many(model, P.CountFeatures(qu[:64], plan, enc), ex)  # warm-up
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(ex.stream)
P.classify.predict_many(model, P.CountFeatures(qu, plan, enc), ex)
b.record(ex.stream)
b.synchronize()
ms = a.elapsed_time(b)
flop = 2.0 * nt * nq * dim
print(f"NN {nq} queries x {nt} train x {dim} features: {ms:.1f} ms, {flop / ms / 1e9:.1f} TFLOP/s (fp64 DFMA), "
      f"{nq / ms * 1e3:.0f} queries/s")
