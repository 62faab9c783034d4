"""Pinned host <-> device copy bandwidth on the box: one direction at a time and both at once
(the e2e step streams images up and counts down concurrently)."""
import time

import torch


def bw(n_bytes, up=True, down=True, reps=3):
    dev = torch.device("cuda:0")
    h_up = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    h_dn = torch.empty(n_bytes, dtype=torch.uint8, pin_memory=True)
    d_up = torch.empty(n_bytes, dtype=torch.uint8, device=dev)
    d_dn = torch.empty(n_bytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        if up:
            with torch.cuda.stream(s1):
                d_up.copy_(h_up, non_blocking=True)
        if down:
            with torch.cuda.stream(s2):
                h_dn.copy_(d_dn, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return n_bytes / best / 1e9


if __name__ == "__main__":
    n = 2 << 30
    print(f"H2D alone {bw(n, True, False):.1f} GB/s")
    print(f"D2H alone {bw(n, False, True):.1f} GB/s")
    print(f"both at once: {bw(n, True, True):.1f} GB/s per direction")
