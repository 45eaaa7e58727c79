"""Slot-engine schedule simulation: 148 CTAs x 32 slots pull pixels in queue
order; a tick costs the same whatever the number of active slots (optionally:
proportional to the 8-slot column blocks holding an active pixel).  Reports the
makespan in ticks against the ideal (total iterations / slots).

    python tools/tail_sim.py gpurun_out/iters_admm.npy
"""
import sys

import numpy as np


def simulate(it, ctas=148, slots=32, blockskip=False, order=None):
    it = it if order is None else it[order]
    P = len(it)
    rem = np.zeros((ctas, slots), dtype=np.int64)
    q = 0
    # initial fill, CTA-interleaved like the atomic queue
    for s in range(slots):
        for c in range(ctas):
            if q < P:
                rem[c, s] = max(int(it[q]), 1)
                q += 1
    t = np.zeros(ctas)
    busy_cols = 0
    while True:
        active = rem > 0
        if not active.any():
            break
        # advance to the next retirement event of any slot (vectorised over ticks)
        step = int(rem[active].min())
        nblk = active.reshape(ctas, slots // 8, 8).any(axis=2).sum(axis=1) if blockskip else (active.any(axis=1) * (slots // 8))
        t += step * nblk / (slots // 8)
        busy_cols += step * active.sum()
        rem[active] -= step
        done = active & (rem == 0)
        for c, s in zip(*np.nonzero(done)):
            if q < P:
                rem[c, s] = max(int(it[q]), 1)
                q += 1
    ideal = it.sum() / (ctas * slots)
    return t.max(), ideal


if __name__ == "__main__":
    it = np.load(sys.argv[1])
    for bs in (False, True):
        mk, ideal = simulate(it, blockskip=bs)
        print(f"{sys.argv[1]}: blockskip={bs}: makespan {mk:.0f} ticks, ideal {ideal:.0f}, efficiency {ideal / mk:.3f}")
