"""Summarise an attention timeline trace (tools/build_trace.sh, CT_TC_TRACE_OUT):
per tile, median softmax duration, hand-off latencies and block period (SM clocks)."""
import sys
import numpy as np

for f in sys.argv[1:]:
    d = np.loadtxt(f, dtype=np.int64)
    d = d[d[:, 2] > 0]
    t0 = d[:, 5].min()
    ss, se, pv, si = (d[:, k] - t0 for k in (2, 3, 4, 5))
    print(f, "blocks", d[:, 0].max() + 1)
    for x in (0, 1):
        m = d[:, 1] == x
        sl = slice(5, None)
        print(f"  tile {x}: softmax {np.median((se - ss)[m][sl]):.0f}"
              f"  S-commit->softmax {np.median((ss - si)[m][sl]):.0f}"
              f"  softmax-end->PV {np.median((pv - se)[m][sl]):.0f}"
              f"  PV->next S commit {np.median((si[m][1:] - pv[m][:-1])[5:]):.0f}"
              f"  period {np.median(np.diff(ss[m])[5:]):.0f}")
