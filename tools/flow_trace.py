"""Summarise a dataflow tree-launch trace (HM_FLOW_TRACE builds, $HM_FLOW_TRACE_FILE):
per level, the window of its pair tasks and the mean time of each task phase
(wait for the children / parent flags, stage the coefficient blocks, DMMA, signal).

    python tools/flow_trace.py gpurun_out/.../flow_c4.bin
"""
import struct
import sys

import numpy as np


def main(path):
    with open(path, "rb") as f:
        L, DL, grid, tasks = struct.unpack("4i", f.read(16))
        tr = np.frombuffer(f.read(), dtype=np.uint64).reshape(tasks, 6).astype(np.int64)
    t0 = tr[:, 0].min()
    n_up = (1 << L) - 1 if L >= 1 else 0
    rows = []
    for t in range(tasks):
        if t < n_up:
            v = (1 << L) - t
            l = int(v - 1).bit_length()
            kind = "up"
        else:
            u = t - n_up
            l = int(u + 1).bit_length()
            kind = "down"
        rows.append((kind, l))
    print(f"L={L} DL={DL} grid={grid} tasks={tasks}, span {(tr[:, 4].max() - t0) / 1e3:.1f} us")
    print(f"{'sweep':5s} {'lvl':>3s} {'pairs':>5s} {'first start':>11s} {'last end':>9s} "
          f"{'wait':>6s} {'stage':>6s} {'dmma':>6s} {'signal':>6s}  (us; phases: mean per task)")
    keys = sorted(set(rows), key=lambda r: (r[0] != "up", -r[1] if r[0] == "up" else r[1]))
    for kind, l in keys:
        idx = [i for i, r in enumerate(rows) if r == (kind, l)]
        a = tr[idx]
        print(f"{kind:5s} {l:3d} {len(idx):5d} {(a[:, 0].min() - t0) / 1e3:11.2f} {(a[:, 4].max() - t0) / 1e3:9.2f} "
              f"{np.mean(a[:, 1] - a[:, 0]) / 1e3:6.2f} {np.mean(a[:, 2] - a[:, 1]) / 1e3:6.2f} "
              f"{np.mean(a[:, 3] - a[:, 2]) / 1e3:6.2f} {np.mean(a[:, 4] - a[:, 3]) / 1e3:6.2f}")


if __name__ == "__main__":
    main(sys.argv[1])
