"""Busy warps over time from a supernodal per-task trace (tools/sn_probe.py
with SN_TRACE_DUMP=...): per 1 ms bin, the mean number of warps executing a
task (after its waits) and of warps waiting.  Diagnostics only.

    python tools/sn_occupancy.py trace.npz [--bin-us 1000]
"""
import argparse

import numpy as np


def main():
    p = argparse.ArgumentParser()
    p.add_argument("trace")
    p.add_argument("--bin-us", type=float, default=1000.0)
    a = p.parse_args()
    tr = np.load(a.trace)["trace"].astype(np.float64) * 1e-2  # us
    span = tr[:, 3].max()
    nb = int(np.ceil(span / a.bin_us))
    busy = np.zeros(nb)
    wait = np.zeros(nb)
    for lo, hi, acc in ((tr[:, 2], tr[:, 3], busy), (tr[:, 0], tr[:, 2], wait)):
        # overlap of [lo, hi) with each bin, summed (warp-us per bin)
        edges = np.arange(nb + 1) * a.bin_us
        for b in range(nb):
            acc[b] = np.clip(np.minimum(hi, edges[b + 1]) - np.maximum(lo, edges[b]), 0, None).sum()
    print(f"span {span:.0f} us; per {a.bin_us:.0f}-us bin: mean warps executing / waiting")
    for b in range(nb):
        print(f"{b * a.bin_us / 1e3:6.1f} ms  exec {busy[b] / a.bin_us:7.1f}  wait {wait[b] / a.bin_us:7.1f}")


if __name__ == "__main__":
    main()
