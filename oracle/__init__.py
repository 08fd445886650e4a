"""CPU oracle for the Aqua preempt/resume KV-paging hot path (arXiv 2407.21255).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything in this package.  The product (``paper_2407_21255_b200``: the C-ABI
library ``libaqua.so`` and its Python binding) never imports it, and this
package never imports the product: the two share no code, headers, tables or
helpers.  The only shared module is ``workloads`` (seeded random inputs, none
of the method's arithmetic).

Plain, slow, obviously-correct Python + NumPy.  Every function cites the
passage it follows: ``P:n`` = line n of the paper text, ``S:n`` =
line n of SPEC.md; the paper's section is named beside it.  Where the paper is
silent, the reading taken is numbered R1..R21 in DESIGN.md ("Readings").

Modules
  kvpool   -- paged KV pool, block allocator, lender/host arenas, swap_out,
              swap_in, free, query (C-1..C-7; paper Sec. 6, Sec. 7
              "Efficient context switching" P:840-853, Sec. 8)
  cfs      -- CFS batch partitioning + reschedule rule + FCFS baseline
              (Sec. 7; SPEC sched S:248-339)
  sim      -- metadata-mode trace driver: CFS + pool bookkeeping over a
              bursty trace on a virtual clock (Sec. 9)
  pattern  -- closed-form synthetic KV content (splitmix64 words), C-11
  bwfit    -- saturating bandwidth curve B(s)=peak*s/(s+half) (SPEC S:50-66,
              fitted to the paper's two A100 points P:846-848)

Parity status: every function here is pinned by a ``-m "not gpu"`` test
against something other than itself (worked examples, closed forms,
brute force, invariants); see DESIGN.md "Oracle pins".  None is unpinned.
"""
