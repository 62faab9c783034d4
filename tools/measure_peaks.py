"""Measured compute peaks of this B200 (FFMA, DFMA, DMMA, tcgen05 TF32 per-SM MMA rate) -> profiles/round2_peaks.json.

The driver's MEASURED_PEAKS.json carries HBM GB/s and cuBLAS bf16; the roofline
fractions of the FP32, FP64 and TF32 kernels are quoted against these instead
of figures derived from the datasheet. Run on a GPU box:

    python tools/measure_peaks.py
"""
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "tools" / "microbench" / "_bin"


def run(cmd):
    return subprocess.run(cmd, capture_output=True, text=True, timeout=300).stdout


class Clock:
    """Median NVML SM clock while a microbenchmark runs (the per-clock rate is what transfers)."""

    def __enter__(self):
        import threading

        import pynvml as nv

        nv.nvmlInit()
        h = nv.nvmlDeviceGetHandleByIndex(0)
        self.samples, self.halt = [], threading.Event()

        def poll():
            while not self.halt.wait(0.002):
                self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))

        self.t = threading.Thread(target=poll, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *exc):
        self.halt.set()
        self.t.join()
        s = sorted(x for x in self.samples if x > 500) or [1965]
        self.mhz = s[len(s) // 2]


def main():
    out = {"source": "tools/measure_peaks.py (tools/microbench/peaks.cu, dmma_dfma.cu, tc_probe.cu t)"}
    best = {}
    for _ in range(3):  # best of 3 runs, each with the SM clock it ran at
        with Clock() as clk:
            p = run([str(BIN / "peaks")])
        for key, pat in (("ffma", r"FFMA: ([\d.]+)"), ("dfma", r"DFMA: ([\d.]+)")):
            m = re.search(pat, p)
            if m:
                per_clk = float(m.group(1)) * 1e12 / (148 * clk.mhz * 1e6)  # flop per clock per SM
                if per_clk > best.get(key, (0, 0, 0))[0]:
                    best[key] = (per_clk, float(m.group(1)), clk.mhz)
    out["peaks_raw"] = p.strip().splitlines()
    for key in ("ffma", "dfma"):
        if key in best:
            out[f"{key}_flop_per_clk_per_sm"], tf, mhz = best[key]
            out[f"{key}_tflops_measured"], out[f"{key}_sm_mhz"] = tf, mhz
            out[f"{key}_tflops"] = best[key][0] * 148 * 1965e6 / 1e12  # at the max clock
    d = run([str(BIN / "dmma_dfma")])
    out["dmma_dfma_raw"] = d.strip().splitlines()
    vals = [float(x) for x in re.findall(r"mode 1 \(dmma\): [\d.]+ ms, ([\d.]+) TFLOP", d)]
    out["dmma_tflops"] = max(vals) if vals else None
    t = run([str(BIN / "tc_probe"), "t"])
    out["tc_probe_raw"] = t.strip().splitlines()
    m = re.search(r"uniform N=256 mma\s*:\s*([\d.]+) cycles per step of 6 ops", t)
    if m:
        cyc = float(m.group(1)) / 6.0  # cycles per M128 N256 K8 tf32 MMA on one SM
        out["tf32_mma_m128n256k8_cycles"] = cyc
        out["tf32_flop_per_clk_per_sm"] = 2 * 128 * 256 * 8 / cyc
    (ROOT / "profiles" / "round2_peaks.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps({k: v for k, v in out.items() if not k.endswith("_raw")}))


if __name__ == "__main__":
    sys.exit(main())
