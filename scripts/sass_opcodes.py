"""Opcode counts per kernel from cuobjdump -sass of libaqua.so (no GPU
needed) -> JSON on stdout: the evidence that the product swap kernel moves
payload with TMA bulk copies (UBLKCP) and claims batches with a
non-aggregated atom.inc, with no 128-bit LDG/STG of payload.

    python scripts/sass_opcodes.py > profiles/r01_sass_opcodes.json
"""
import json
import os
import re
import shutil
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WATCH = ("UBLKCP", "SYNCS", "LDG", "STG", "ATOMG", "UTMA", "SHFL")


def kernels(lib=os.path.join(ROOT, "paper_2407_21255_b200", "libaqua.so")):
    cob = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    txt = subprocess.run([cob, "-sass", lib], capture_output=True, text=True, check=True).stdout
    out = {}
    for f in re.split(r"\n\s*Function : ", txt)[1:]:
        name = f.split("\n", 1)[0].strip()
        short = re.sub(r"^_ZN4aqua\w+?_aqua_kernels_cu_\w{8}\d+", "", name)
        ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
        c = Counter(ops)
        out[short] = {k: v for k, v in sorted(c.items()) if k.startswith(WATCH)}
        out[short]["total_instructions"] = len(ops)
    return out


if __name__ == "__main__":
    ks = kernels(*sys.argv[1:])
    print(json.dumps({"source": "cuobjdump -sass paper_2407_21255_b200/libaqua.so (sm_100a); opcode counts per "
                                "kernel (scripts/sass_opcodes.py)", "kernels": ks}, indent=1))
