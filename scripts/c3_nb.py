"""Derive the C3 borrower pool size from an oracle metadata run (calls only
oracle/ and workloads/): NB = ceil(1.2 x peak blocks owned before the burst
starts, under unlimited-memory FCFS) -- DESIGN.md "Input recipe", C3.

    python scripts/c3_nb.py  ->  prints the NB used by tests and bench.py
"""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import sim  # noqa: E402
from workloads import burst_trace  # noqa: E402

tr = burst_trace(seed=1)
t_burst = tr[24][1]
r = sim.run(tr, sim.SimConfig(NB=100_000, policy="fcfs", host_slots=1))
peak = max(b for t, b in r.timeline if t < t_burst)
print(f"requests={len(tr)} burst_start={t_burst:.3f}s pre_burst_peak_blocks={peak} "
      f"NB={math.ceil(1.2 * peak)} overall_peak_blocks={max(b for _, b in r.timeline)}")
