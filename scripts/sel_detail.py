"""Per-item selection sub-phases of one traced step (debug, run under gpurun)."""
import sys
import numpy as np
t = np.load(sys.argv[1]).astype(np.int64)
t0 = t[0, 0].min()
r = (t - t0) / 1e3
names = [(2, "epi_wake"), (8, "c_prefix"), (9, "c_keys"), (10, "c_done"), (12, "r_wake"), (6, "r_loaded"), (11, "r_digit"),
         (15, "r_scan"), (4, "r_ranked"), (14, "e_scan"), (13, "e_done")]
for l in [int(x) for x in sys.argv[2:]]:
    ctas = [c for c in range(t.shape[2]) if t[l, 10, c] > t0]
    print("layer", l, "items on ctas", ctas[0], "..", ctas[-1])
    for e, n in names:
        v = r[l, e, ctas]
        print(f"  {n:10s} min {v.min():7.1f} med {np.median(v):7.1f} max {v.max():7.1f}")
