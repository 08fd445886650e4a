"""Summarise ncu reports (run here, no GPU): per-launch time, DRAM bytes
read/written and throughput for the swap kernels -> JSON on stdout.

    python scripts/ncu_summarize.py gpurun_out/r01_prof_tma_final.ncu-rep [...]
"""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread"]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte/s": 1e12, "Gbyte/s": 1e9}


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for w in WANT:
            if w in h:
                i = h.index(w)
                v = float(r[i].replace(",", ""))
                u = units[i]
                if u in SCALE:
                    v *= SCALE[u]
                    u = "B/s" if "/s" in units[i] else "B"
                elif u == "ms":
                    v, u = v * 1e-3, "s"
                elif u == "us":
                    v, u = v * 1e-6, "s"
                d[w] = v
        d["traffic_bytes"] = d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        out.append(d)
    return out


if __name__ == "__main__":
    print(json.dumps({p: summarize(p) for p in sys.argv[1:]}, indent=1))
