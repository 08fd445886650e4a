"""Mutation check of the parity tests against the PRODUCT (test infrastructure).

scripts/oracle_mutants.py shows the oracle's pins catch plausible mistakes in
the oracle.  This script shows the parity tests catch plausible mistakes in
the product: each MUTANT is a one-line edit of libaqua's sources (the sm_100a
kernels or the C++ host library).  For each one the script copies the package,
the headers, the oracle, the seeded generators and the tests into
build/mutants/mNN/, applies the edit there (the repo is never modified) and
builds that copy's libaqua.so with the product's own build (nvcc, sm_100a).
Then, for each mutant, it runs that copy's parity tests:

  kind "cpu": the dry-run parity tests (`tests/test_dryrun_parity.py`, host
              library vs oracle, no GPU) -- run here;
  kind "gpu": the GPU parity tests (`tests/test_gpu_parity.py -m gpu`: whole
              buffers vs the oracle) -- run on the B200 via gpurun.

A mutant is "killed" when a parity test fails (or the run errors / times out).

    python scripts/product_mutants.py prepare [--kind cpu|gpu|all] [--jobs 8]
    python scripts/product_mutants.py run --kind cpu|gpu [--out FILE]

No mutant can hang the GPU: none touches an mbarrier, a ring depth or a loop
bound, and every run is under `timeout`.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import shutil
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT_DIR = os.environ.get("AQUA_MUTANT_DIR") or os.path.join(ROOT, "build", "mutants")
PKG = "paper_2407_21255_b200"

CPU_TESTS = ["tests/test_dryrun_parity.py", "tests/test_multiproc.py", "tests/test_idset.py", "-m", "not gpu"]
GPU_TESTS = ["tests/test_gpu_parity.py", "tests/test_gpu_peer.py", "-m", "gpu"]

# (name, file under csrc/ (or a .py file of the package), [(old, new, occurrence)], kind)
MUTANTS = [
    # ---- kernels (aqua_kernels.cu): address arithmetic of A3 / A6 (R1, R3)
    ("image side: piece offset dropped", "aqua_kernels.cu",
     [("uint8_t* img = reinterpret_cast<uint8_t*>(base) + slot * p.U + int64_t(c) * p.S + off;",
       "uint8_t* img = reinterpret_cast<uint8_t*>(base) + slot * p.U + int64_t(c) * p.S;", None)], "gpu"),
    ("image side: chunk index c -> c/2 (K and V collide)", "aqua_kernels.cu",
     [("uint8_t* img = reinterpret_cast<uint8_t*>(base) + slot * p.U + int64_t(c) * p.S + off;",
       "uint8_t* img = reinterpret_cast<uint8_t*>(base) + slot * p.U + int64_t(c >> 1) * p.S + off;", None)], "gpu"),
    ("pool side: K/V plane stride replaced by the block stride", "aqua_kernels.cu",
     [("uint8_t* pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + l)) + kv * p.P_kv +",
       "uint8_t* pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + l)) + kv * p.P_b +", None)], "gpu"),
    ("last piece of a chunk copies a whole piece (ragged tail overrun)", "aqua_kernels.cu",
     [("bytes = static_cast<uint32_t>(rem < p.piece ? rem : p.piece);",
       "bytes = static_cast<uint32_t>(p.piece);", None)], "gpu"),
    ("TMA ring, static ranges: CTA range rounds down twice (items lost)", "aqua_kernels.cu",
     [("    i1 = p.nitems * (b + 1) / G;", "    i1 = p.nitems * (b + 1) / G - (b + 1 == G ? 1 : 0);", None)], "gpu"),
    ("TMA ring, claimed batches: the first batch skips its first item", "aqua_kernels.cu",
     [("    i0 = b * p.batch;\n", "    i0 = b * p.batch + (p.batch > 1 ? 1 : 0);\n", None)], "gpu"),
    ("TMA ring: grouped pool-side loads use the piece size, not S", "aqua_kernels.cu",
     [("      if (lane == 0) mbar_expect_tx(&bars[lstage], static_cast<uint32_t>(p.S) * k);\n      __syncwarp();\n"
       "      for (int t = lane; t < k; t += 32) {\n        item_addrs<D>(p, d, lu.c + t, 0, src, dst, bytes);\n"
       "        bulk_g2s(buf + size_t(t) * bytes, src, bytes, &bars[lstage], pol);",
       "      if (lane == 0) mbar_expect_tx(&bars[lstage], static_cast<uint32_t>(p.S) * k);\n      __syncwarp();\n"
       "      for (int t = lane; t < k; t += 32) {\n        item_addrs<D>(p, d, lu.c + ((t ^ 1) < k ? (t ^ 1) : t), 0, src, dst, bytes);\n"
       "        bulk_g2s(buf + size_t(t) * bytes, src, bytes, &bars[lstage], pol);", None)], "gpu"),
    ("LDST engine: stores one vector past the item", "aqua_kernels.cu",
     [("      if (idx < nvec) st_stream(dst + size_t(idx) * 16, v[u]);\n    }\n  };\n  int4 a[UNROLL], b[UNROLL];",
       "      if (idx <= nvec) st_stream(dst + size_t(idx) * 16, v[u]);\n    }\n  };\n  int4 a[UNROLL], b[UNROLL];",
       None)], "gpu"),
    ("small-chunk kernel: V chunk read from the K plane", "aqua_kernels.cu",
     [("        pool = const_cast<uint8_t*>(D == kOut ? src : dst) + p.P_kv;",
       "        pool = const_cast<uint8_t*>(D == kOut ? src : dst);", None)], "gpu"),
    ("small-chunk kernel: the last partial round is dropped", "aqua_kernels.cu",
     [("  const int64_t nrounds = (p.nitems + k - 1) / k;", "  const int64_t nrounds = p.nitems / k;", None)], "gpu"),
    ("register warps (hybrid): packed chunks land at the wrong offset", "aqua_kernels.cu",
     [("            const size_t vo = size_t((u * 32) % nvec_s + lane) * 16;\n            v[u] = ld_stream(src + vo);\n            dp[u] += vo;",
       "            const size_t vo = size_t((u * 32) % nvec_s + lane) * 16;\n            v[u] = ld_stream(src + vo);\n            dp[u] += vo ^ 16;",
       None)], "gpu"),
    # ---- host library: stream ordering (A4 / A7, R7) -- only a GPU can show a race
    ("alloc_blocks reuses a block without waiting for the swap that read it (A4)", "aqua_host.cpp",
     [("  for (int32_t b : ids) ts.push_back(c->btick[b]);\n  if (aqua_status s = wait_all(c, ts, reinterpret_cast<cudaStream_t>(stream))) return s;",
       "  for (int32_t b : ids) ts.push_back(c->btick[b]);", None)], "gpu"),
    ("launch: no wait for the last use of the call's blocks and slots (R7)", "aqua_host.cpp",
     [("  if (aqua_status s = wait_all(c, ts, st)) return s;\n  return enqueue_copy(c, ds, dir, st, layer_group, group_tickets, ticket);",
       "  return enqueue_copy(c, ds, dir, st, layer_group, group_tickets, ticket);", None)], "gpu"),
    ("free: the caller's stream is not recorded on the freed blocks (R7)", "aqua_host.cpp",
     [("      if (aqua_status s = record(c, st, &t)) return s;\n    }\n    for (int32_t b : p.ids) {",
       "    }\n    for (int32_t b : p.ids) {", None)], "gpu"),
    ("swap_in: the read slots are not tagged with its ticket (A7)", "aqua_host.cpp",
     [("    a->free.insert_all(ps[i]->ids.data(), ps[i]->ids.size());\n    uint64_t* st_tick = a->tick.data();\n    for (int32_t s : ps[i]->ids) st_tick[s] = ticket;",
       "    a->free.insert_all(ps[i]->ids.data(), ps[i]->ids.size());\n    uint64_t* st_tick = a->tick.data();\n    (void)st_tick;", None)], "gpu"),
    ("copy-engine host path: the last slot of a contiguous run is not copied to DRAM", "aqua_host.cpp",
     [("          CK(c, cudaMemcpy2DAsync(img, c->U, t, per, per, r, cudaMemcpyDefault, st));",
       "          CK(c, cudaMemcpy2DAsync(img, c->U, t, per, per, r > 1 ? r - 1 : r, cudaMemcpyDefault, st));", None)], "gpu"),
    ("copy-engine host path: the staging buffer is reused without waiting for its last user", "aqua_host.cpp",
     [("  if (aqua_status s = wait_all(c, {c->ce_tick[di]}, st)) return s;   // the buffer's last user\n",
       "", None)], "gpu"),
    ("layer-wise swaps: each layer group misses its last chunk", "aqua_host.cpp",
     [("    if (aqua_status s = run_copy(c, ds, dir, st, &regions, 2 * l0, 2 * (l1 - l0), dd)) return s;",
       "    if (aqua_status s = run_copy(c, ds, dir, st, &regions, 2 * l0, 2 * (l1 - l0) - 1, dd)) return s;", None)], "gpu"),
    ("migration kernel: the source image's arena bit is ignored", "aqua_kernels.cu",
     [("    const uint64_t sbase = (sb >> 31) ? p.arena_base[1] : p.arena_base[0];",
       "    const uint64_t sbase = p.arena_base[0];", None)], "gpu"),
    ("migration: the source slots are not tagged with its ticket (R7)", "aqua_host.cpp",
     [("      as->free.insert(so);\n      as->tick[so] = ticket;", "      as->free.insert(so);", None)], "gpu"),
    ("exchange: every resume piece waits only for the first preemption piece", "aqua_host.cpp",
     [("    parts[f == freed_by.end() ? 0 : f->second].push_back(d);", "    parts[0].push_back(d); (void)f;", None)], "gpu"),
    ("prefix_store: the source blocks are not tagged with its ticket (R7)", "aqua_host.cpp",
     [("    c->btick[src.ids[j]] = ticket;     // last reader of the prompt's blocks\n", "", None)], "gpu"),
    ("prefix_load: the image slots are not tagged with its ticket (R7)", "aqua_host.cpp",
     [("    a->tick[img.ids[j]] = ticket;      // last reader of the image\n", "", None)], "gpu"),
    ("prefix_store copies the LAST n blocks of the prompt", "aqua_host.cpp",
     [("    ds.push_back(Desc{src.ids[j], static_cast<uint32_t>(sl) | bit});",
       "    ds.push_back(Desc{src.ids[src.ids.size() - n + j], static_cast<uint32_t>(sl) | bit});", None)], "gpu"),
    ("descriptor ring: a region is rewritten without waiting for its last user", "aqua_host.cpp",
     [("    const bool overlap = it->off < off + len && off < it->off + it->len;",
       "    const bool overlap = false && it->off < off + len && off < it->off + it->len;", None)], "gpu"),
    ("TMA ring: grouped pool-side STORES of a unit swapped pairwise (swap_in)", "aqua_kernels.cu",
     [("      for (int t = lane; t < k; t += 32) {\n        item_addrs<D>(p, d, su.c + t, 0, src, dst, bytes);\n        bulk_s2g(dst, buf + size_t(t) * bytes, bytes, pol);",
       "      for (int t = lane; t < k; t += 32) {\n        item_addrs<D>(p, d, su.c + ((t ^ 1) < k ? (t ^ 1) : t), 0, src, dst, bytes);\n        bulk_s2g(dst, buf + size_t(t) * bytes, bytes, pol);", None)], "gpu"),
    ("small-chunk kernel: next layer's K plane of block 0 read from block 1", "aqua_kernels.cu",
     [("        pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + (p.kv_merged ? c : c >> 1))) + boff;",
       "        pool = reinterpret_cast<uint8_t*>(__ldg(p.layer_base + (p.kv_merged ? c : c >> 1))) + (boff ? boff : p.P_b);", None)], "gpu"),
    ("claimed batches: the counter pair is not reset for the next launch", "aqua_kernels.cu",
     [("    ctr[0] = 0;\n    ctr[1] = 0;", "    ctr[1] = 0;", None)], "gpu"),
    # ---- AUTO launch policy (DESIGN 5.1, section 8 peer cap, NEXT-4 rate budget): shapes, not bytes
    ("AUTO: a launch touching a peer arena is not capped at AQUA_OPT_PEER_CTAS", "aqua_host.cpp",
     [("      if (c->peer_ctas > 0 && (cap == 0 || cap > c->peer_ctas)) cap = c->peer_ctas;\n", "", None)], "gpu"),
    ("AUTO: a peer arena whose bulk-copy probe failed still gets the TMA engine (R20)", "aqua_host.cpp",
     [("      if ((c->gpu.probe & 6) != 6 && engine == AQUA_KERNEL_TMA) engine = AQUA_KERNEL_LDST;\n", "", None)], "gpu"),
    ("AUTO: the paging budget maps to one SM too few (rounds down)", "aqua_host.cpp",
     [("      const int want = std::max(1, (c->rate_gbps + kSwapGBpsPerSm - 1) / kSwapGBpsPerSm);",
       "      const int want = std::max(1, c->rate_gbps / kSwapGBpsPerSm);", None)], "gpu"),
    ("AUTO: host-only launches are not capped (PCIe-bound)", "aqua_host.cpp",
     [("    if (all_host && (cap == 0 || cap > kHostCtas)) cap = kHostCtas;\n", "", None)], "gpu"),
    ("AUTO: a call with images in both arenas runs as one fused launch (not split)", "aqua_host.cpp",
     [("    if (!host_only && img_any_host && dir != aqua::kMig && !dev_desc) {",
       "    if (false) {", None)], "gpu"),
    ("AUTO: the split sends every image to the TMA kernel (host part lost)", "aqua_host.cpp",
     [("      return run_copy_ce_host(c, dh, dir, st, c0, nc);", "      return AQUA_OK;", None)], "gpu"),
    ("AUTO: layer-wise mixed calls keep the shared descriptor upload", "aqua_host.cpp",
     [("    if (any_host && any_gpu) fused = false;", "    (void)any_host;", None)], "gpu"),
    ("migration on the copy engines: a run ignores the destination slots", "aqua_host.cpp",
     [("static_cast<uint32_t>(ds[j + r].block) == s0 + r && ds[j + r].slot_arena == d0 + r)",
       "static_cast<uint32_t>(ds[j + r].block) == s0 + r)", None)], "gpu"),
    ("migration on the copy engines: a run ignores the source slots", "aqua_host.cpp",
     [("static_cast<uint32_t>(ds[j + r].block) == s0 + r && ds[j + r].slot_arena == d0 + r)",
       "ds[j + r].slot_arena == d0 + r)", None)], "gpu"),
    # ---- host library: bookkeeping (A1, A2, A5, A7; R4, R5) -- dry-run parity on CPU
    ("placement: lender needs strictly more than n_p free slots (R5)", "aqua_host.cpp",
     [("    if (gpu_left >= np) {", "    if (gpu_left > np) {", None)], "cpu"),
    ("placement: the host arena before the lender (R5)", "aqua_host.cpp",
     [("    if (gpu_left >= np) {", "    if (gpu_left >= np && host_left < np) {", None)], "cpu"),
    ("swap_out descriptors pair block k with slot k+1", "aqua_host.cpp",
     [("    for (int32_t k = 0; k < np; ++k) dp[k] = Desc{ids[k], static_cast<uint32_t>(sv[k]) | bit};",
       "    for (int32_t k = 0; k < np; ++k) dp[k] = Desc{ids[k], static_cast<uint32_t>(sv[(k + 1) % np]) | bit};",
       None)], "cpu"),
    ("swap_out keeps the prompt's blocks allocated (A4)", "aqua_host.cpp",
     [("    c->free_blocks.insert_all(ps[i]->ids.data(), ps[i]->ids.size());\n    uint64_t* bt_tick = c->btick.data();\n    for (int32_t b : ps[i]->ids) bt_tick[b] = ticket;\n    ps[i]->state = AQUA_ST_SWAPPED;",
       "    uint64_t* bt_tick = c->btick.data();\n    for (int32_t b : ps[i]->ids) bt_tick[b] = ticket;\n    ps[i]->state = AQUA_ST_SWAPPED;",
       None)], "cpu"),
    ("swap_in: capacity check off by one (NOBLOCKS with exactly enough)", "aqua_host.cpp",
     [("  if (need > static_cast<int64_t>(c->free_blocks.size())) return fail(c, AQUA_E_NOBLOCKS, \"pool exhausted\");",
       "  if (need >= static_cast<int64_t>(c->free_blocks.size()) && need > 0) return fail(c, AQUA_E_NOBLOCKS, \"pool exhausted\");",
       None)], "cpu"),
    ("swap_in keeps the lender slots (A7)", "aqua_host.cpp",
     [("    a->free.insert_all(ps[i]->ids.data(), ps[i]->ids.size());\n    uint64_t* st_tick = a->tick.data();\n    for (int32_t s : ps[i]->ids) st_tick[s] = ticket;\n    uint64_t* bt_tick = c->btick.data();\n    for (int32_t b : fresh[i]) {",
       "    uint64_t* st_tick = a->tick.data();\n    for (int32_t s : ps[i]->ids) st_tick[s] = ticket;\n    uint64_t* bt_tick = c->btick.data();\n    for (int32_t b : fresh[i]) {",
       None)], "cpu"),
    ("adopt_blocks accepts a block that is not free", "aqua_host.cpp",
     [("!seen.insert(b).second || !c->free_blocks.count(b))", "!seen.insert(b).second)", None)], "cpu"),
    ("swap_out accepts a pid listed twice", "aqua_host.cpp",
     [("    if (!seen.insert(pids[i]).second) return fail(c, AQUA_E_INVAL, \"duplicate pid\");\n  for (int32_t i = 0; i < n; ++i) {\n    auto it = c->prompts.find(pids[i]);\n    if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT)",
       "    seen.insert(pids[i]);\n  for (int32_t i = 0; i < n; ++i) {\n    auto it = c->prompts.find(pids[i]);\n    if (it == c->prompts.end() || it->second.state != AQUA_ST_RESIDENT)",
       None)], "cpu"),
    ("exchange: the blocks the preemptions free are not counted for the resume (NOBLOCKS)", "aqua_host.cpp",
     [("  if (need > static_cast<int64_t>(c->free_blocks.size()) + freed)",
       "  if (need > static_cast<int64_t>(c->free_blocks.size()) + 0 * freed)", None)], "cpu"),
    ("exchange: resume blocks planned before the preemption frees its blocks", "aqua_host.cpp",
     [("  // ---- preemption bookkeeping\n  for (int32_t i = 0; i < n_out; ++i) {\n    Arena* a = arena_of(c, loc[i]);\n    for (int32_t sl : slots[i]) a->free.erase(sl);\n    for (int32_t b : po[i]->ids) c->free_blocks.insert(b);\n  }",
       "  // ---- preemption bookkeeping\n  for (int32_t i = 0; i < n_out; ++i) {\n    Arena* a = arena_of(c, loc[i]);\n    for (int32_t sl : slots[i]) a->free.erase(sl);\n  }", None)], "cpu"),
    ("migrate: capacity check off by one", "aqua_host.cpp",
     [("  if (!ad->present || need > ad->free.size()) return fail(c, AQUA_E_NOSPACE, \"dst arena missing or full\");",
       "  if (!ad->present || need >= ad->free.size()) return fail(c, AQUA_E_NOSPACE, \"dst arena missing or full\");", None)], "cpu"),
    ("prefix_store: lender needs more than n free slots", "aqua_host.cpp",
     [("  if (c->gpu.present && c->gpu.free.size() >= n)", "  if (c->gpu.present && c->gpu.free.size() > n)", None)], "cpu"),
    ("prefix_load: capacity check off by one", "aqua_host.cpp",
     [("  if (n > c->free_blocks.size()) return fail(c, AQUA_E_NOBLOCKS, \"pool exhausted\");",
       "  if (n > 0 && n >= c->free_blocks.size()) return fail(c, AQUA_E_NOBLOCKS, \"pool exhausted\");", None)], "cpu"),
    ("reclaim: host capacity check off by one", "aqua_host.cpp",
     [("  if (need > 0 && (!c->host.present || need > c->host.free.size()))",
       "  if (need > 0 && (!c->host.present || need >= c->host.free.size()))", None)], "cpu"),
    ("reclaim moves cached prefixes before prompts", "aqua_host.cpp",
     [("  for (uint64_t p : pids) ps.push_back(&c->prompts[p]);\n  for (uint64_t f : fids) ps.push_back(&c->prefixes[f]);",
       "  for (uint64_t f : fids) ps.push_back(&c->prefixes[f]);\n  for (uint64_t p : pids) ps.push_back(&c->prompts[p]);", None)], "cpu"),
    # ---- Python side of the product: pairing and the trace driver
    ("pairing: maximises the SUM instead of the minimum pair bandwidth", "pairing.py",
     [("            key = (min(vals) if vals else float(\"inf\"), [-x for x in part])\n            if best_key is None or key > best_key:\n                best, best_key = list(part), key",
       "            key = (sum(vals) if vals else float(\"inf\"), [-x for x in part])\n            if best_key is None or key > best_key:\n                best, best_key = list(part), key", None)], "cpu"),
    ("pairing: a pair's bandwidth taken one way only", "pairing.py",
     [("        vals = [min(bw[b][l], bw[l][b]) for b, l in zip(borrowers, perm)]",
       "        vals = [bw[b][l] for b, l in zip(borrowers, perm)]", None)], "cpu"),
    ("driver: the re-offer skips an image that does not fit instead of stopping (R22)", "driver.py",
     [("                    if k > room:\n                        break", "                    if k > room:\n                        continue", None)], "cpu"),
    ("free-id bitmap: a bulk insert does not lower the scan start (lowest-first lost)", "aqua_idset.h",
     [("        cnt += __builtin_popcountll(add);\n        if (wd < lo) lo = wd;", "        cnt += __builtin_popcountll(add);", None)], "cpu"),
    ("free-id bitmap: a bulk erase counts every id, present or not", "aqua_idset.h",
     [("      const uint64_t del = m & w[wd];\n      w[wd] &= ~del;\n      cnt -= __builtin_popcountll(del);",
       "      const uint64_t del = m & w[wd];\n      w[wd] &= ~del;\n      cnt -= __builtin_popcountll(m);", None)], "cpu"),
    ("free-id bitmap: erase_lowest takes a whole word when fewer bits are wanted", "aqua_idset.h",
     [("      if (pc <= k) {                 // the whole word goes", "      if (pc <= k + 1) {             // the whole word goes", None)], "cpu"),
    # ---- native CFS scheduler (aqua_cfs.cpp, A0)
    ("CFS: reschedule every k+1 iterations (P:836)", "aqua_cfs.cpp",
     [("s->iter - s->last >= s->cfg.k", "s->iter - s->last > s->cfg.k", None)], "cpu"),
    ("CFS: no reschedule when a request completes (P:837)", "aqua_cfs.cpp",
     [("s->iter - s->last >= s->cfg.k || s->finished_prev ||", "s->iter - s->last >= s->cfg.k ||", None)], "cpu"),
    ("CFS step 3: one decode prompt too many", "aqua_cfs.cpp",
     [("    if (static_cast<int32_t>(pl.dec.size()) >= d) break;", "    if (static_cast<int32_t>(pl.dec.size()) > d) break;", None)], "cpu"),
    ("CFS order: decode prompts by most tokens generated", "aqua_cfs.cpp",
     [("    if (a->g != b->g) return a->g < b->g;", "    if (a->g != b->g) return a->g > b->g;", None)], "cpu"),
    ("CFS order: prefill prompts by arrival only", "aqua_cfs.cpp",
     [("    if (a->f != b->f) return a->f < b->f;\n", "", None)], "cpu"),
    ("CFS step 1: decode prompts counted before prefill (R16)", "aqua_cfs.cpp",
     [("    for (const Req* r : pass == 0 ? pre : dec) {", "    for (const Req* r : pass == 0 ? dec : pre) {", None)], "cpu"),
    ("CFS step 1: d = fit, not min(b, fit)", "aqua_cfs.cpp",
     [("  const int32_t d = std::min(b, fit);", "  const int32_t d = fit;", None)], "cpu"),
    ("CFS step 3: a decode prompt that does not fit is skipped (R12)", "aqua_cfs.cpp",
     [("    const int32_t n = blocks_for(s, *r, 1);\n    if (mem + n > NB) break;\n    mem += n;\n    pl.dec.push_back(r->id);",
       "    const int32_t n = blocks_for(s, *r, 1);\n    if (mem + n > NB) continue;\n    mem += n;\n    pl.dec.push_back(r->id);", None)], "cpu"),
    ("CFS R21 branch dropped", "aqua_cfs.cpp",
     [("  if (chosen.empty()) {", "  if (false) {", None)], "cpu"),
    ("CFS step 5: extra prefill tokens ignore memory", "aqua_cfs.cpp",
     [("    if (room_tokens < hi) hi = static_cast<int32_t>(std::max<int64_t>(room_tokens, 0));\n", "", None)], "cpu"),
    ("FCFS admission off by one (projection must fit NB)", "aqua_cfs.cpp",
     [("      if (proj + n > s->cfg.num_blocks) break;", "      if (proj + n >= s->cfg.num_blocks) break;", None)], "cpu"),
    ("FCFS plan: decode list not capped at b", "aqua_cfs.cpp",
     [("        if (r->phase == AQUA_PHASE_DECODE && static_cast<int32_t>(pl.dec.size()) < s->cfg.batch_tokens)",
       "        if (r->phase == AQUA_PHASE_DECODE)", None)], "cpu"),
    ("FCFS overflow evicts the earliest-arrived resident (R18)", "aqua_cfs.cpp",
     [("        if (r.where == kResident && (!victim || by_arrival(victim, &r))) victim = &r;",
       "        if (r.where == kResident && (!victim || by_arrival(&r, victim))) victim = &r;", None)], "cpu"),
    ("CFS: a prompt finishes one token late", "aqua_cfs.cpp",
     [("    if (r.phase == AQUA_PHASE_DECODE && r.g >= r.O) fin.push_back(r.id);",
       "    if (r.phase == AQUA_PHASE_DECODE && r.g > r.O) fin.push_back(r.id);", None)], "cpu"),
]


def apply(text: str, edits) -> str:
    for old, new, occ in edits:
        n = text.count(old)
        if occ is None:
            if n != 1:
                raise ValueError(f"{old[:70]!r}: {n} matches, expected exactly 1")
            text = text.replace(old, new)
        else:
            if n <= occ:
                raise ValueError(f"{old[:70]!r}: {n} matches, occurrence {occ} missing")
            i = -1
            for _ in range(occ + 1):
                i = text.index(old, i + 1)
            text = text[:i] + new + text[i + len(old):]
    return text


def _src(root: str, fname: str) -> str:
    return os.path.join(root, PKG, fname) if fname.endswith(".py") else os.path.join(root, PKG, "csrc", fname)


def check_all_apply() -> None:
    for name, fname, edits, _ in MUTANTS:
        src = open(_src(ROOT, fname)).read()
        assert apply(src, edits) != src, name


def _dir(i: int) -> str:
    return os.path.join(OUT_DIR, f"m{i:02d}")


def prepare_one(i: int) -> str:
    name, fname, edits, _ = MUTANTS[i]
    d = _dir(i)
    shutil.rmtree(d, ignore_errors=True)
    ign = shutil.ignore_patterns("__pycache__", "*.so", "*.so.tmp")
    for sub in (PKG, "include", "oracle", "workloads", "tests", "scripts"):
        shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub), ignore=ign)
    for f in ("bench.py", "__graft_entry__.py", "MEASURED_PEAKS.json", "BASELINE.json"):
        if os.path.exists(os.path.join(ROOT, f)):
            shutil.copy(os.path.join(ROOT, f), os.path.join(d, f))
    p = _src(d, fname)
    with open(p) as f:
        src = f.read()
    with open(p, "w") as f:
        f.write(apply(src, edits))
    with open(os.path.join(d, "MUTANT.txt"), "w") as f:
        f.write(name + "\n")
    r = subprocess.run([sys.executable, "-m", f"{PKG}.build", "--force"], cwd=d, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"mutant {i} ({name}) does not build:\n{r.stderr[-2000:]}")
    return d


def run_one(i: int, timeout: int) -> dict:
    name, fname, _, kind = MUTANTS[i]
    d = _dir(i)
    tests = CPU_TESTS if kind == "cpu" else GPU_TESTS
    t0 = time.time()
    try:
        r = subprocess.run([sys.executable, "-m", "pytest", *tests, "-x", "-q", "-p", "no:cacheprovider"],
                           cwd=d, capture_output=True, text=True, timeout=timeout)
        out = r.stdout.strip().splitlines()
        failed = [ln.split(" - ")[0] for ln in out if ln.startswith(("FAILED", "ERROR"))]
        killed, first, summary = r.returncode != 0, (failed[0] if failed else None), (out[-1] if out else "")
    except subprocess.TimeoutExpired:
        killed, first, summary = True, None, f"timeout after {timeout} s"
    return {"mutant": name, "file": os.path.relpath(_src(ROOT, fname), ROOT), "kind": kind, "killed": killed,
            "first_failing_test": first, "summary": summary, "seconds": round(time.time() - t0, 1)}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["prepare", "run", "check"])
    ap.add_argument("--kind", default="all", choices=["cpu", "gpu", "all"])
    ap.add_argument("--jobs", type=int, default=min(8, os.cpu_count() or 1))
    ap.add_argument("--timeout", type=int, default=900)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default="", help="comma-separated mutant names (substring match) to run")
    args = ap.parse_args()
    check_all_apply()
    if args.cmd == "check":
        print(f"{len(MUTANTS)} mutants apply")
        return
    sel = [i for i, m in enumerate(MUTANTS) if args.kind in ("all", m[3])]
    if args.only:
        keys = [k.strip() for k in args.only.split(",") if k.strip()]
        sel = [i for i in sel if any(k in MUTANTS[i][0] for k in keys)]
    if args.cmd == "prepare":
        with cf.ThreadPoolExecutor(args.jobs) as ex:
            for d in ex.map(prepare_one, sel):
                print("built", d)
        return
    # the unmutated library must pass the same tests first (else every "kill" is meaningless)
    for kind in sorted({MUTANTS[i][3] for i in sel}):
        tests = CPU_TESTS if kind == "cpu" else GPU_TESTS
        r = subprocess.run([sys.executable, "-m", "pytest", *tests, "-x", "-q", "-p", "no:cacheprovider"],
                           cwd=ROOT, capture_output=True, text=True, timeout=args.timeout)
        if r.returncode != 0:
            raise SystemExit(f"baseline {kind} tests fail on the unmutated library:\n{r.stdout[-3000:]}")
        print(f"baseline {kind}: {r.stdout.strip().splitlines()[-1]}")
    jobs = args.jobs if args.kind == "cpu" else 1            # one GPU: one mutant at a time
    with cf.ThreadPoolExecutor(jobs) as ex:
        res = list(ex.map(lambda i: run_one(i, args.timeout), sel))
    killed = sum(r["killed"] for r in res)
    doc = {"what": "product mutation check: one-line edits of libaqua's sources (kernels, host library, native "
                   "scheduler), each built for sm_100a and run against the parity tests (cpu: dry-run host library "
                   "vs oracle; gpu: whole-buffer GPU parity vs oracle); killed = a parity test fails",
           "kind": args.kind, "tests": CPU_TESTS if args.kind == "cpu" else GPU_TESTS,
           "mutants": len(res), "killed": killed, "survived": len(res) - killed, "results": res}
    out = args.out or os.path.join(ROOT, "profiles", f"r02_product_mutants_{args.kind}.json")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    for r in res:
        print("KILLED  " if r["killed"] else "SURVIVED", r["mutant"], "|", r["first_failing_test"] or r["summary"])
    print(f"{killed}/{len(res)} killed -> {out}")


if __name__ == "__main__":
    main()
