"""Mutation check of the oracle's pins (test infrastructure).

The oracle must be pinned to something other than itself, "chosen so that a
plausible mistake anywhere in it (a dropped term, a wrong sign or index, a
transposed operand) fails one of them".  This script makes that claim
checkable: each MUTANT below is one such plausible mistake, written as a
textual edit of one oracle file.  For every mutant the script copies the
oracle, the seeded input generators and the oracle pin tests into a scratch
directory, applies the edit there (the repo is never modified) and runs ONLY
the oracle pin tests (`tests/test_oracle_*.py`, all `-m "not gpu"`): the
tests that compare the oracle with the paper's worked examples, closed forms,
brute force and invariants -- never with the CUDA path or the native host
library.  A mutant is "killed" when at least one pin fails.

    python scripts/oracle_mutants.py [--jobs 8] [--out profiles/r02_oracle_mutants.json]

`tests/test_oracle_mutants.py` checks (fast, no pytest runs) that every
mutant's text still occurs in the oracle exactly as many times as it says, so
this list cannot silently rot when the oracle changes.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import shutil
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PIN_TESTS = ["tests/test_oracle_cfs.py", "tests/test_oracle_kvpool.py", "tests/test_oracle_misc.py"]

# (name, file, [(old, new, occurrence)][, equivalence]): occurrence = the
# 0-based index of the match to replace, or None when `old` must be unique.
# Each names the paper passage / reading the mutated line implements.  An
# `equivalence` note marks a mutant that cannot change any result (argued in
# the note and checked by a random-trace comparison); it is run and reported
# but not counted as a surviving gap.
MUTANTS = [
    # ---- kvpool.py: byte definitions (R1, R3) ----------------
    ("S drops the element size e (C-1)", "kvpool.py",
     [("return self.bs * self.H * self.D * self.e", "return self.bs * self.H * self.D", None)]),
    ("U counts K or V only (U = L*S)", "kvpool.py",
     [("return 2 * self.L * self.S", "return self.L * self.S", None)]),
    ("chunk(): K/V plane and block strides transposed (R1)", "kvpool.py",
     [("off = kv * lay.P_kv + b * lay.P_b", "off = kv * lay.P_b + b * lay.P_kv", None)]),
    ("chunk(): V plane read from the K plane", "kvpool.py",
     [("off = kv * lay.P_kv + b * lay.P_b", "off = b * lay.P_b", None)]),
    ("swap_out image: (l, kv) chunk index 2l+kv -> l+kv (collides)", "kvpool.py",
     [("off = s * lay.U + (2 * l + kv) * lay.S", "off = s * lay.U + (l + kv) * lay.S", 0)]),
    ("image layout kv-major (kv*L + l) on both swap_out and swap_in (R3)", "kvpool.py",
     [("off = s * lay.U + (2 * l + kv) * lay.S", "off = s * lay.U + (kv * lay.L + l) * lay.S", 0),
      ("off = s * lay.U + (2 * l + kv) * lay.S", "off = s * lay.U + (kv * lay.L + l) * lay.S", 0)]),
    ("swap_out image: slot stride S instead of U", "kvpool.py",
     [("off = s * lay.U + (2 * l + kv) * lay.S", "off = s * lay.S + (2 * l + kv) * lay.S", 0)]),
    ("swap_in scatters the slots in reverse order", "kvpool.py",
     [("for j, (b, s) in enumerate(zip(new, p.slots)):", "for j, (b, s) in enumerate(zip(new, p.slots[::-1])):", None)]),
    # ---- kvpool.py: allocator and placement (R4, R5)
    ("fresh blocks: highest free ids first (R4)", "kvpool.py",
     [("ids = sorted(self.free)[:n]", "ids = sorted(self.free, reverse=True)[:n]", None)]),
    ("placement: lender needs strictly more than n_p free slots", "kvpool.py",
     [("if peer_free is not None and len(peer_free) >= n:", "if peer_free is not None and len(peer_free) > n:", None)]),
    ("placement: host before the lender (P:749-753 reversed)", "kvpool.py",
     [("if peer_free is not None and len(peer_free) >= n:",
       "if peer_free is not None and len(peer_free) >= n and (host_free is None or len(host_free) < n):", None)]),
    ("placement: highest lender slots first", "kvpool.py",
     [("peer_free = sorted(self.peer.free) if self.peer else None",
       "peer_free = sorted(self.peer.free, reverse=True) if self.peer else None", None)]),
    ("swap_out keeps the source blocks allocated (A4)", "kvpool.py",
     [("            self.free.update(p.blocks)\n            p.blocks = []", "            p.blocks = []", None)]),
    ("swap_out accepts a pid listed twice", "kvpool.py",
     [("raise AquaError(E_INVAL, \"duplicate pid\")", "pass", 0)]),
    ("swap_in: off-by-one pool capacity check", "kvpool.py",
     [("if need > len(self.free):", "if need >= len(self.free):", None)]),
    ("swap_in keeps the lender slots (A7)", "kvpool.py",
     [("            if p.slots:\n                ar.free.update(p.slots)\n            p.state, p.location, p.slots, p.blocks",
       "            p.state, p.location, p.slots, p.blocks", None)]),
    ("free_prompt of a swapped prompt keeps its slots (P:754-756)", "kvpool.py",
     [("        elif p.slots:\n            self.arena(p.location).free.update(p.slots)", "        elif False:\n            pass", None)]),
    # ---- kvpool.py: NEXT-1 / NEXT-2 --------------------------------------
    ("migrate copies from the destination slot index", "kvpool.py",
     [("= ar_s.data[s_old * lay.U:(s_old + 1) * lay.U]", "= ar_s.data[s_new * lay.U:(s_new + 1) * lay.U]", None)]),
    ("reclaim leaves the lender attached (P:758-768)", "kvpool.py",
     [("        self.peer = None\n        return list(zip(pids, moved))", "        return list(zip(pids, moved))", None)]),
    ("prefix_store persists the LAST n blocks", "kvpool.py",
     [("for b, s in zip(p.blocks[:n], slots):", "for b, s in zip(p.blocks[len(p.blocks) - n:], slots):", None)]),
    ("prefix_load consumes the cached image (copy, not move)", "kvpool.py",
     [("        p.blocks.extend(new)\n        return new", "        p.blocks.extend(new)\n        self.prefix_drop(fid)\n        return new", None)]),
    ("adopt_blocks accepts ids that are not free", "kvpool.py",
     [("                or any(b not in self.free for b in ids):", "                or False:", None)]),
    ("adopt_blocks sorts the caller's ids (block-table order lost)", "kvpool.py",
     [("        p.blocks.extend(ids)\n\n    # ---", "        p.blocks.extend(sorted(ids))\n\n    # ---", None)]),
    ("lend: capacity rounds a partial slot up", "kvpool.py",
     [("nslots = nbytes // self.lay.U", "nslots = -(-nbytes // self.lay.U)", None)]),
    ("migrate: capacity check off by one", "kvpool.py",
     [("if need > len(ar_d.free):", "if need >= len(ar_d.free):", None)]),
    ("reclaim moves prompts in descending pid order", "kvpool.py",
     [("moved = self._move([self.prompts[p] for p in pids], LOC_HOST)",
       "pids = pids[::-1]\n        moved = self._move([self.prompts[p] for p in pids], LOC_HOST)", None)]),
    ("reclaim moves prefixes before prompts", "kvpool.py",
     [("        moved = self._move([self.prompts[p] for p in pids], LOC_HOST)\n        self._move([self.prefixes[f] for f in fids], LOC_HOST)",
       "        self._move([self.prefixes[f] for f in fids], LOC_HOST)\n        moved = self._move([self.prompts[p] for p in pids], LOC_HOST)", None)]),
    ("prefix_store placement: lender needs more than n free slots", "kvpool.py",
     [("if self.peer is not None and len(self.peer.free) >= n:", "if self.peer is not None and len(self.peer.free) > n:", None)]),
    ("query of a swapped prompt reports its (empty) block table", "kvpool.py",
     [("ids = p.blocks if p.state == RESIDENT else p.slots", "ids = p.blocks", None)]),
    ("Pool accepts S not a multiple of 16 bytes", "kvpool.py",
     [("        if layout.S % 16 != 0:\n            raise AquaError(E_INVAL, \"S must be a multiple of 16 bytes\")",
       "        if False:\n            raise AquaError(E_INVAL, \"S must be a multiple of 16 bytes\")", None)]),
    ("adopt_blocks accepts out-of-range ids", "kvpool.py",
     [("or any(not (0 <= b < self.lay.NB) for b in ids) \\", "or False \\", None)],
     "equivalent: an id outside [0, NB) is never in the free set, so the free-and-distinct test that follows "
     "rejects it with the same code (E_INVAL) and no change"),
    ("alloc_blocks accepts n < 0", "kvpool.py",
     [("        if n < 0:\n            raise AquaError(E_INVAL, \"n < 0\")", "        if False:\n            pass", None)]),
    ("swap_out of a swapped prompt allowed", "kvpool.py",
     [("            if p is None or p.state != RESIDENT:\n                raise AquaError(E_STATE, f\"pid {pid} not resident\")",
       "            if p is None:\n                raise AquaError(E_STATE, f\"pid {pid} not resident\")", None)]),
    ("swap_in of a resident prompt allowed", "kvpool.py",
     [("            if p is None or p.state != SWAPPED:\n                raise AquaError(E_STATE, f\"pid {pid} not swapped\")",
       "            if p is None:\n                raise AquaError(E_STATE, f\"pid {pid} not swapped\")", None)]),
    ("migrate to the arena the image is already in allowed", "kvpool.py",
     [("if p is None or p.state != SWAPPED or p.location == dst:", "if p is None or p.state != SWAPPED:", None)]),
    ("prefix_store reuses a prefix id in use", "kvpool.py",
     [("        if int(fid) in self.prefixes:\n            raise AquaError(E_INVAL, \"prefix id in use\")",
       "        if False:\n            raise AquaError(E_INVAL, \"prefix id in use\")", None)]),
    ("prefix_load: capacity check off by one", "kvpool.py",
     [("        if len(f.slots) > len(self.free):", "        if len(f.slots) >= len(self.free):", None)]),
    ("reclaim: host capacity check off by one", "kvpool.py",
     [("if need and (self.host is None or need > len(self.host.free)):", "if need and (self.host is None or need >= len(self.host.free)):", None)]),
    # ---- cfs.py: batch partitioning ---------------
    ("decode order: most tokens generated first (P:833)", "cfs.py",
     [("key=lambda r: (r.g, r.arrival, r.id)", "key=lambda r: (-r.g, r.arrival, r.id)", None)]),
    ("prefill order: arrival only (least prefill done dropped)", "cfs.py",
     [("key=lambda r: (r.f, r.arrival, r.id)", "key=lambda r: (r.arrival, r.id)", None)]),
    ("ties broken by id, not (arrival, id) (R9)", "cfs.py",
     [("key=lambda r: (r.g, r.arrival, r.id)", "key=lambda r: (r.g, r.id)", None),
      ("key=lambda r: (r.f, r.arrival, r.id)", "key=lambda r: (r.f, r.id)", None)]),
    ("need(): floor instead of ceil blocks (R11)", "cfs.py",
     [("return -(-(r.ctx + t) // bs)", "return (r.ctx + t) // bs", None)]),
    ("need(): this iteration's tokens ignored (R11)", "cfs.py",
     [("return -(-(r.ctx + t) // bs)", "return -(-(r.ctx + 1) // bs)", None)]),
    ("step 1: d = C, not min(b, C)", "cfs.py",
     [("    d = min(b, C)\n", "    d = C\n", None)]),
    ("step 1: counts decode prompts before prefill (R16)", "cfs.py",
     [("for r in pre + dec:", "for r in dec + pre:", None)]),
    ("step 2: a prompt gets p tokens regardless of its remaining prefill", "cfs.py",
     [("alloc = min(p_rem, r.P - r.f)", "alloc = p_rem", None)]),
    ("step 3: one decode prompt too many (|D| <= d)", "cfs.py",
     [("if len(D) >= d:", "if len(D) > d:", None)]),
    ("step 3: a decode prompt that does not fit is skipped, not a stop (R12)", "cfs.py",
     [("        n = need(r, 1, bs)\n        if used + n > NB:\n            break\n        used += n\n        D.append(r.id)",
       "        n = need(r, 1, bs)\n        if used + n > NB:\n            continue\n        used += n\n        D.append(r.id)", None)]),
    ("step 4: extra tokens ignore the step-2 allocation", "cfs.py",
     [("extra = min(left, r.P - r.f - alloc)", "extra = min(left, r.P - r.f)", None)]),
    ("step 4: R21 branch dropped (p = 0 leaves slots unused)", "cfs.py",
     [("if not chosen and left > 0:", "if False:", None)]),
    ("step 5: memory test skipped for extra tokens", "cfs.py",
     [("while extra > 0 and used - need(r, alloc, bs) + need(r, alloc + extra, bs) > NB:",
       "while False:", None)]),
    ("fcfs_plan: decode list not capped at b", "cfs.py",
     [("if r.phase == DECODE][:b]", "if r.phase == DECODE]", None)]),
    # ---- sim.py: reschedule and iteration semantics
    ("reschedule every k+1 iterations (P:836)", "sim.py",
     [("i - last >= cfg.k or finished_prev", "i - last >= cfg.k + 1 or finished_prev", None)]),
    ("no reschedule when a request completes (P:837)", "sim.py",
     [("i - last >= cfg.k or finished_prev", "i - last >= cfg.k", None)]),
    ("page lists sorted by id, not (arrival, id)", "sim.py",
     [("key = lambda pid: (run_set[pid].arrival, pid)", "key = lambda pid: pid", None)]),
    ("page_out keeps resident prompts that left the plan (R13)", "sim.py",
     [("page_out = sorted((pid for pid in run_set if resident(pid) and pid not in in_plan), key=key)",
       "page_out = []", None)]),
    ("iteration cost drops the per-token term (S:233)", "sim.py",
     [("t += cfg.t_base + cfg.t_token * total", "t += cfg.t_base", None)]),
    ("decode stores no KV for its token (R15)", "sim.py",
     [("                r.ctx += 1\n                r.g += 1", "                r.g += 1", None)]),
    ("a prompt finishes one token late", "sim.py",
     [("if r.phase == DECODE and r.g >= r.O:", "if r.phase == DECODE and r.g > r.O:", None)]),
    ("FCFS overflow evicts the earliest arrival (R18)", "sim.py",
     [("victim = max(victims, key=lambda x: (run_set[x].arrival, x))",
       "victim = min(victims, key=lambda x: (run_set[x].arrival, x))", None)]),
    ("FCFS admission off by one (projection must fit NB)", "sim.py",
     [("if proj + n > lay.NB:", "if proj + n >= lay.NB:", None)]),
    ("fits(): this iteration's tokens ignored for resident prompts (R11)", "sim.py",
     [("tot += cfs.need(run_set[pid], tok.get(pid, 0), lay.bs)", "tot += cfs.need(run_set[pid], 0, lay.bs)", None)]),
    ("fits(): prompts to be paged in not counted (R11)", "sim.py",
     [("            if not resident(pid):\n                tot += cfs.need(run_set[pid], tt, lay.bs)",
       "            if False:\n                pass", None)],
     "equivalent: the old plan's prompts are all resident when fits() re-checks it (page-ins happen at the "
     "replan, a planned prefill gets its first blocks in its first iteration), and in FCFS the admission "
     "projection already bounds every admitted prompt's need; 600 random traces give identical logs"),
    ("prefill work not clipped to the tokens left", "sim.py",
     [("out.append((pid, min(a, r.P - r.f)))", "out.append((pid, a))", None)]),
    ("re-offer moves back the highest pids first (NEXT-1)", "sim.py",
     [("for pid in sorted(pid for pid, p in pool.prompts.items()\n                                  if p.state == SWAPPED and p.location == LOC_HOST):",
       "for pid in sorted((pid for pid, p in pool.prompts.items()\n                                  if p.state == SWAPPED and p.location == LOC_HOST), reverse=True):", None)]),
    ("re-offer skips a prompt that does not fit instead of stopping", "sim.py",
     [("                    if k > room:\n                        break", "                    if k > room:\n                        continue", None)]),
    ("fallback admits residents in id order, not arrival", "sim.py",
     [("admitted_fcfs[:] = [pid for pid in sorted(run_set, key=lambda x: (run_set[x].arrival, x))",
       "admitted_fcfs[:] = [pid for pid in sorted(run_set)", None)],
     "equivalent: admitted_fcfs is only read as a set (projection sum, resident filter, victim = max by "
     "(arrival, id)); fcfs_plan re-sorts by (arrival, id); 600 random traces give identical logs"),
    ("a prefill prompt's first token is not counted (g stays 0)", "sim.py",
     [("r.phase, r.g = DECODE, 1", "r.phase, r.g = DECODE, 0", None)]),
    # ---- pattern.py: closed-form KV words (C-11) --------------------------
    ("pack(): kv shifted onto l's bits", "pattern.py",
     [("(u(kv) << u(17))", "(u(kv) << u(18))", None)]),
    ("splitmix64 (vectorised): wrong second shift", "pattern.py",
     [("z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)",
       "z = (z ^ (z >> np.uint64(28))) * np.uint64(0x94D049BB133111EB)", None)]),
    ("write_tokens: token row ignores the head count", "pattern.py",
     [("row = i * lay.H * lay.D * 2\n                ch[row:row + lay.H * lay.D * 2] = w.reshape(-1).view(np.uint8)",
       "row = i * lay.D * 2\n                ch[row:row + lay.H * lay.D * 2] = w.reshape(-1).view(np.uint8)", None)]),
    ("write_token_range: the run of rows in a block starts at the block's row 0", "pattern.py",
     [("                ch[i * row:(i + n) * row] = w[tt - t0:tt - t0 + n].reshape(-1)",
       "                ch[0:n * row] = w[tt - t0:tt - t0 + n].reshape(-1)", None)]),
    ("splitmix64 (scalar): wrong increment", "pattern.py",
     [("    z = (x + 0x9E3779B97F4A7C15) & M64", "    z = (x + 0x9E3779B97F4A7C16) & M64", None)]),
    ("token_words keeps the high 16 bits", "pattern.py",
     [("    return (z & np.uint64(0xFFFF)).astype(np.uint16)", "    return (z >> np.uint64(48)).astype(np.uint16)", None)]),
    # ---- bwfit.py: saturating bandwidth curve -------
    ("B(s) = peak*s/(s+half) with half added twice", "bwfit.py",
     [("return peak * s / (s + half)", "return peak * s / (s + 2 * half)", None)]),
    ("calibrate: peak from the wrong point", "bwfit.py",
     [("peak = b1 * (s1 + half) / s1", "peak = b1 * (s2 + half) / s1", None)]),
    ("fit: half = slope / peak", "bwfit.py",
     [("return peak, slope * peak", "return peak, slope / peak", None)]),
    ("transfer_time: one buffer's time, not nbuf", "bwfit.py",
     [("return nbuf * (lat + s / effective_bandwidth(peak, half, s))",
       "return (lat + s / effective_bandwidth(peak, half, s))", None)]),
]


def apply(text: str, edits) -> str:
    for old, new, occ in edits:
        n = text.count(old)
        if occ is None:
            if n != 1:
                raise ValueError(f"{old[:60]!r}: {n} matches, expected exactly 1")
            text = text.replace(old, new)
        else:
            if n <= occ:
                raise ValueError(f"{old[:60]!r}: {n} matches, occurrence {occ} missing")
            i = -1
            for _ in range(occ + 1):
                i = text.index(old, i + 1)
            text = text[:i] + new + text[i + len(old):]
    return text


def check_all_apply() -> None:
    """Every mutant applies to the current oracle and changes it."""
    for name, fname, edits, *_ in MUTANTS:
        src = open(os.path.join(ROOT, "oracle", fname)).read()
        out = apply(src, edits)
        assert out != src, name


def run_one(idx: int) -> dict:
    name, fname, edits, *eq = MUTANTS[idx]
    tmp = tempfile.mkdtemp(prefix="mut_")
    try:
        shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(tmp, "oracle"),
                        ignore=shutil.ignore_patterns("__pycache__"))
        shutil.copytree(os.path.join(ROOT, "workloads"), os.path.join(tmp, "workloads"),
                        ignore=shutil.ignore_patterns("__pycache__"))
        os.makedirs(os.path.join(tmp, "tests"))
        shutil.copytree(os.path.join(ROOT, "tests", "golden"), os.path.join(tmp, "tests", "golden"))
        for f in ["tests/conftest.py"] + PIN_TESTS:
            shutil.copy(os.path.join(ROOT, f), os.path.join(tmp, f))
        p = os.path.join(tmp, "oracle", fname)
        with open(p) as f:
            src = f.read()
        with open(p, "w") as f:
            f.write(apply(src, edits))
        t0 = time.time()
        r = subprocess.run([sys.executable, "-m", "pytest", *PIN_TESTS, "-x", "-q", "-m", "not gpu",
                            "-p", "no:cacheprovider", "--timeout", "300"],
                           cwd=tmp, capture_output=True, text=True, timeout=900)
        out = r.stdout.strip().splitlines()
        failed = [ln.split(" - ")[0] for ln in out if ln.startswith("FAILED") or ln.startswith("ERROR")]
        return {"mutant": name, "file": f"oracle/{fname}", "killed": r.returncode != 0,
                "equivalent": eq[0] if eq else None,
                "first_failing_pin": failed[0] if failed else None,
                "summary": out[-1] if out else "", "seconds": round(time.time() - t0, 1)}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--jobs", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_oracle_mutants.json"))
    args = ap.parse_args()
    check_all_apply()
    with cf.ThreadPoolExecutor(args.jobs) as ex:
        res = list(ex.map(run_one, range(len(MUTANTS))))
    killed = sum(r["killed"] for r in res)
    equiv = sum(1 for r in res if not r["killed"] and r["equivalent"])
    doc = {"what": "oracle mutation check: each mutant is one plausible mistake in oracle/; killed = a "
                   "-m 'not gpu' oracle pin test (tests/test_oracle_*.py: paper examples, closed forms, "
                   "brute force, invariants; never the CUDA path) fails",
           "pin_tests": PIN_TESTS, "mutants": len(res), "killed": killed, "equivalent_unkilled": equiv,
           "survived": len(res) - killed - equiv,
           "results": res}
    with open(args.out, "w") as f:
        json.dump(doc, f, indent=1)
    for r in res:
        tag = "KILLED  " if r["killed"] else ("EQUIV   " if r["equivalent"] else "SURVIVED")
        print(tag, r["mutant"], "|", r["first_failing_pin"])
    print(f"{killed}/{len(res)} killed, {equiv} equivalent, {len(res) - killed - equiv} survived -> {args.out}")


if __name__ == "__main__":
    main()
