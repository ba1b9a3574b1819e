"""Phase breakdown of the persistent decode kernel from a PPOEXP_MEGA_TRACE dump.

    PPOEXP_MEGA_TRACE=/tmp/t.bin python tools/profile_decode.py --graphs 0 --new 24
    python tools/mega_trace.py /tmp/t.bin --layers 12 --grid 148

Per phase (averaged over layers): median / max per-CTA work (own release →
own arrival), barrier latency (last arrival → last release) and release
skew (first → last release), from %globaltimer stamps.
"""
import argparse

import numpy as np

PH = ["ln1", "qkv", "attn", "o_proj", "ln2", "up", "gelu", "down"]
ap = argparse.ArgumentParser()
ap.add_argument("path")
ap.add_argument("--layers", type=int, default=12)
ap.add_argument("--grid", type=int, default=148)
a = ap.parse_args()
L, G, P = a.layers, a.grid, len(PH)
t = np.fromfile(a.path, dtype=np.uint64).astype(np.int64)[:P * L * G * 2].reshape(P * L, G, 2)
print(f"barrier 0 .. last release: {(t[-1, :, 1].max() - t[0, :, 0].min()) / 1e3:.1f} us")
acc = {p: np.zeros(4) for p in PH}
for k in range(1, P * L):
    arr, dep, prev = t[k, :, 0], t[k, :, 1], t[k - 1, :, 1]
    w = (arr - prev) / 1e3
    acc[PH[k % P]] += [np.median(w), w.max(), (dep.max() - arr.max()) / 1e3, (dep.max() - dep.min()) / 1e3]
print(f"{'phase':7s} {'med work':>9s} {'max work':>9s} {'barrier':>8s} {'skew':>6s}   (us per layer)")
tot = 0.0
for p in PH:
    m = acc[p] / L
    tot += m[1] + m[2]
    print(f"{p:7s} {m[0]:9.2f} {m[1]:9.2f} {m[2]:8.2f} {m[3]:6.2f}")
print(f"sum of (max work + barrier) per layer: {tot:.1f} us")
raw = np.fromfile(a.path, dtype=np.uint64).astype(np.int64)
o = P * L * G * 2
if raw.size > o:
    at = raw[o:o + L * G * 8 * 4].reshape(L, G, 8, 4)
    act = at[:, :, :, 3] > 0
    pro = (at[:, :, :, 1] - at[:, :, :, 0])[act] / 1.965e3
    loop = (at[:, :, :, 2] - at[:, :, :, 1])[act] / 1.965e3
    nt = at[:, :, :, 3][act]
    print(f"attention item (warp-level, SM clock): prologue med {np.median(pro):.2f} us, tile loop med {np.median(loop):.2f} us "
          f"over med {np.median(nt):.0f} tiles ({np.median(loop / nt):.2f} us/tile)")
