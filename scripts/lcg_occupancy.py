"""LCG body throughput vs warps per SM and chains per thread (microbench.cu
k_lcg_peak): where does the executor's compute_bound body saturate an SM?"""
import json
import sys

sys.path.insert(0, ".")
from paper_2508_16522_b200 import roofline as RF  # noqa: E402

L = RF._lib()
out = {}
for chains in (2, 4, 8):
    for wps in (1, 2, 3, 4, 6, 7, 8, 12, 16, 32):
        # one 32-thread CTA per warp: wps CTAs per SM
        r = L.td_mb_compute_peak(0, chains, 148 * wps, 32, 1 << 14, 3)
        out[f"c{chains}_w{wps}"] = r / 148 / 1.965e9  # lane-updates per clock per SM
        print(chains, wps, round(out[f"c{chains}_w{wps}"], 2), flush=True)
print(json.dumps(out))
