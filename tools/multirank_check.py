"""Functional check of the multi-rank fit/transform on ONE GPU (gloo, host-side collectives).

Run: python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
         --master-port 29533 tools/multirank_check.py
Every rank runs train_network + compute_feature_counts on its batch shard (the
per-layer payload exchange goes through torch.distributed); rank 0 then repeats
the run as a world of one and checks that the filters are bitwise identical
(deterministic reduction) and that each rank's counts equal its rows of the
single-rank counts. No kernel waits on another rank, so sharing one GPU is safe;
timings from this are meaningless.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_13027_b200 as P  # noqa: E402
from paper_2209_13027_b200 import synthetic as S  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    solo = dist.new_group([0])
    imgs, labels = S.blob_images(1000, 24, 20, 7, seed=5)
    v1 = imgs.astype(np.float32)
    v2 = S.second_view(v1, labels, "channel", 7, seed=6).astype(np.float32)
    net = P.NetworkConfig((P.LayerConfig(6, P.PatchGeometry(5, 5)), P.LayerConfig(4, P.PatchGeometry(3, 3))),
                          batch=P.BatchSpec(64))
    cfg = type("Cfg", (), {"net": net, "encoder": P.EncoderConfig(6, 5)})()
    ok = True
    for det in (True, False):
        ex = P.Executor(P.ExecSettings(deterministic=det), device=0)
        assert ex.world_size == world
        ds = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
        bank = P.train_network(ds, net, ex)
        counts, _ = P.compute_feature_counts(ds, bank, cfg, ex)
        counts = counts.cpu()
        shard = ex.shard(-(-1000 // 64))
        s0, s1 = shard.start * 64, min(1000, shard.stop * 64)
        parts = [None] * world
        dist.all_gather_object(parts, (rank, s0, s1, counts.numpy(), [(l.filters1, l.filters2) for l in bank.layers]))
        if rank == 0:
            ex1 = P.Executor(P.ExecSettings(deterministic=det), device=0, process_group=solo)
            assert ex1.world_size == 1
            ds1 = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
            b1 = P.train_network(ds1, net, ex1)
            c1, _ = P.compute_feature_counts(ds1, b1, cfg, ex1)
            c1 = c1.cpu().numpy()
            # diagnostics: transform of the distributed bank / of the solo bank on fresh datasets
            ds2 = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
            c2, _ = P.compute_feature_counts(ds2, bank, cfg, ex1)
            c2 = c2.cpu().numpy()
            ds3 = P.ViewPairDataset.from_arrays(v1, v2, labels, class_count=7)
            c3, _ = P.compute_feature_counts(ds3, b1, cfg, ex1)
            c3 = c3.cpu().numpy()
            print(f"det={det}: solo cached vs fresh {np.mean(c1 == c3):.6f}; dist bank fresh vs solo "
                  f"{np.mean(c2 == c3):.6f}; rank0 dist vs fresh rows {np.mean(counts.numpy() == c2[s0:s1]):.6f}",
                  flush=True)
            for r, a, b, c, fl in parts:
                for (f1, f2), lay in zip(fl, b1.layers):
                    same = np.array_equal(f1, lay.filters1) and np.array_equal(f2, lay.filters2)
                    close = np.allclose(f1, lay.filters1, atol=1e-9) and np.allclose(f2, lay.filters2, atol=1e-9)
                    if det and not same:
                        ok = False
                        print(f"deterministic: rank {r} filters differ from the single-rank run")
                    if not close:
                        ok = False
                        print(f"det={det}: rank {r} filters not within 1e-9")
                eq = np.mean(c == c1[a:b]) if c.shape == c1[a:b].shape else 0.0
                if eq < (1.0 if det else 0.999):
                    ok = False
                    print(f"det={det}: rank {r} counts rows [{a},{b}) match {eq:.6f}")
            print(f"det={det}: ranks {world}, checked {'OK' if ok else 'FAILED'}", flush=True)
        dist.barrier()
    dist.destroy_process_group()
    if rank == 0 and not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
