#!/usr/bin/env python
"""tcgen05.mma 128 x N x 256 rate (mode 0 SS, 1 SS 16 issues + commit, 2 no commit,
3/4 MN-major, 5 TS = A in TMEM as the rollout's head / hidden MMA) on B200 (diagnostic for the rollout's per-step MMA)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_16592_b200 import engine  # noqa: E402

L = engine.lib()
for n in (16, 32, 128, 256):
    for mode in ((0, 1, 2, 5) if n < 128 else (0, 1, 2, 3, 4, 5)):
        for grid in (1,):
            reps = 2000
            out = np.zeros(grid, dtype=np.int64)
            rc = L.gfnx_test_mma_rate(n, reps, mode, grid, out.ctypes.data)
            assert rc == 0, engine.lib().gfnx_last_error(None)
            cyc = out.mean() / reps
            macs = 128 * n * 256
            print(f"N={n} mode={mode} grid={grid}: {cyc:8.1f} cycles/MMA  {macs / cyc:7.0f} MAC/clk/SM")
