"""Spread of the mailbox-hop microbenchmark (L_level of the latency roofline)
over the spacing of the ping-pong words and the pair count:
python scripts/hop_probe.py"""
import ctypes as C
import json
import sys

sys.path.insert(0, ".")
from paper_2508_16522_b200 import roofline as R  # noqa: E402

L = R._lib()
out = {}
for stride in (4, 32, 64, 128, 256, 384, 512, 1024, 4096, 4099, 8191):
    for pairs in (16, 74):
        mn = C.c_double()
        med = L.td_mb_mailbox_hop_strided(0, pairs, 20000, C.byref(mn), 0, stride)
        out[f"stride{stride}_pairs{pairs}"] = [round(med, 1), round(mn.value, 1)]
print(json.dumps(out))
