"""Does compute-sanitizer initcheck see bytes written by TMA bulk copies
(cp.async.bulk, the async proxy)?  One swap_out into a FRESH arena
(torch.empty: never written) with a given engine, then the arena is copied
to the host.  Under initcheck, a copy of bytes the tool believes unwritten
is reported.  Run once per engine:

    compute-sanitizer --tool initcheck python scripts/initcheck_probe.py tma
    compute-sanitizer --tool initcheck python scripts/initcheck_probe.py ldst
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_21255_b200 import aqua  # noqa: E402

eng = sys.argv[1] if len(sys.argv) > 1 else "tma"
L, bs, H, D, NB, n = 2, 16, 2, 64, 8, 4
S = bs * H * D * 2
U = 2 * L * S
layers = [torch.full((2 * NB * S,), 7, dtype=torch.uint8, device="cuda") for _ in range(L)]
arena = torch.empty(n * U, dtype=torch.uint8, device="cuda")          # never written by anyone else
ctx = aqua.Ctx(0, L, bs, H, D, 2, NB, [t.data_ptr() for t in layers])
ctx.set_option(aqua.OPT_KERNEL, aqua.KERNEL_TMA if eng == "tma" else aqua.KERNEL_LDST)
ctx.lend(0, arena.data_ptr(), n * U)
ctx.alloc_blocks(1, n)
ctx.swap_out([1])
torch.cuda.synchronize()
h = arena.cpu()
print(eng, "arena bytes all written by the swap:", bool((h == 7).all()))
ctx.close()
