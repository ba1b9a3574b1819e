"""Stage breakdown of the decode GEMM (gemm_decode.cu) from a PPOEXP_GEMM_TRACE dump.

    PPOEXP_GEMM_TRACE=/tmp/g.bin python tools/profile_decode.py --new 24
    python tools/gemm_trace.py /tmp/g.bin

Stamps (CTA (0,0), clock64 converted at 1.965 GHz): 0 entry, 1 setup done, 2 PDL wait released,
3 first activation tile landed, 4 accumulator complete, 5 partial parked +
pushed, 6 peers' slices landed, 7 reduce + epilogue stored, 8 cluster exit.
"""
import collections
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
n = int(np.frombuffer(raw[:4], np.int32)[0])
meta = np.frombuffer(raw[4:4 + n * 16], np.int32).reshape(n, 4)
st = np.frombuffer(raw[4 + n * 16:], np.uint64).astype(np.int64).reshape(n, 16).copy()
names = ["setup", "pdl wait", "X landed", "MMA done", "park+push", "peers in", "reduce+store", "cluster exit"]
groups = collections.defaultdict(list)
for i in range(n):
    if st[i, 0] == 0 or st[i, 6] == 0:
        continue
    for k in (7, 8):  # direct push: no reduce/exit stamps -> zero-length stages
        if st[i, k] == 0:
            st[i, k] = st[i, k - 1]
    groups[tuple(meta[i])].append(st[i])
sub = ["drain(4-9)", "sync(9-10)", "clwait(10-11)", "push+x(11-5)"]
print(f"{'N,K,epi,S':22s} " + " ".join(f"{x:>14s}" for x in sub))
for key, rows in sorted(groups.items()):
    r = np.array(rows)
    if (r[:, 9] == 0).all():
        continue
    d = [(r[:, 9] - r[:, 4]), (r[:, 10] - r[:, 9]), (r[:, 11] - r[:, 10]), (r[:, 5] - r[:, 11])]
    print(f"{str(tuple(int(x) for x in key)):22s} " + " ".join(f"{np.median(x) / 1.965e3:14.2f}" for x in d))
print(f"{'N,K,epi,S':22s} {'n':>4s} " + " ".join(f"{x:>12s}" for x in names) + f" {'total':>8s}")
for key, rows in sorted(groups.items()):
    r = np.array(rows)
    d = np.diff(r[:, :9], axis=1) / 1.965e3
    med = np.median(d, axis=0)
    print(f"{str(key):22s} {len(rows):4d} " + " ".join(f"{x:12.2f}" for x in med) +
          f" {np.median((r[:, 8] - r[:, 0]) / 1.965e3):8.2f}")
