"""Bucket-size distribution of the canonical rows under (map, f0, sub) keys,
sub = min(f1 - f0 - 1, S - 1) -- sizing the bucketed sort."""
import os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_2301_00806_b200 as wpm


def low(bits):
    nz = bits != 0
    w0 = np.argmax(nz, axis=1)
    ar = np.arange(bits.shape[0])
    x = bits[ar, w0]
    lb = x & (~x + np.uint64(1))
    f = w0 * 64 + np.round(np.log2(lb.astype(np.float64))).astype(np.int64)
    bits[ar, w0] = x & (x - np.uint64(1))
    return np.where(nz.any(axis=1), f, -1)


for n in [int(x) for x in sys.argv[1:]]:
    with wpm.Plan.orbits(n) as p:
        p.run()
        r = p.fetch()
    b = np.array(r.bits, dtype=np.uint64)
    mp = np.repeat(np.arange(len(r.counts)), r.counts)
    f0 = low(b)
    f1 = low(b)
    f2 = low(b)
    d = np.where(f1 >= 0, f1 - f0 - 1, 0)
    e = np.where(f2 >= 0, f2 - f1 - 1, 0)
    s1 = np.minimum(d, 7)
    s2 = np.where(s1 < 7, np.minimum(e, 7), 0)
    k = mp * (1 << 40) + f0 * (1 << 21) + s1 * 8 + s2
    _, inv, c = np.unique(k, return_inverse=True, return_counts=True)
    sz = c[inv]  # bucket size of every row
    print("n", n, "rows", len(k), "buckets", len(c), "max", int(c.max()), "row-weighted mean size", round(float(sz.mean()), 1),
          "rows in buckets <=32/64/128/256/512/1024:", [round(float((sz <= t).mean()), 3) for t in (32, 64, 128, 256, 512, 1024)], flush=True)
    for S in ():
        k = mp * (1 << 40) + f0 * (1 << 21) + np.minimum(d, S - 1)
        _, c = np.unique(k, return_counts=True)
        c = np.sort(c)[::-1]
        print("n", n, "rows", len(k), "S", S, "buckets", len(c), "max", c[:5].tolist(), ">1024:", int((c > 1024).sum()),
              "rows in >1024:", int(c[c > 1024].sum()), ">2048:", int((c > 2048).sum()), flush=True)
