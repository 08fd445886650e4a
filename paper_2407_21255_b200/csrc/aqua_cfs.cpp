// Native CFS time-slice scheduler (include/aqua_cfs.h): decides which
// prompts run each iteration and which are paged out / in by libaqua.
//
// Paper, Sec. 7 "Aqua's batch partitioning algorithm" and the
// reschedule rule; FCFS baseline per SPEC S:297-305.  Readings
// R8-R18 in DESIGN.md.  Written independently of the CPU oracle (oracle/cfs.py,
// oracle/sim.py); tests compare the two call logs exactly.
#include "aqua_cfs.h"

#include <algorithm>
#include <cmath>
#include <unordered_map>
#include <utility>
#include <vector>

namespace {

enum Where { kNone = 0, kResident = 1, kSwapped = 2 };

struct Req {
  uint64_t id;
  double arrival;
  int32_t P, O;
  int32_t f = 0, g = 0, ctx = 0;
  int32_t phase = AQUA_PHASE_PREFILL;
  int32_t blocks = 0;  // blocks the caller holds for it (resident or swapped image)
  int where = kNone;
};

struct Plan {
  std::vector<uint64_t> dec;
  std::vector<std::pair<uint64_t, int32_t>> pre;
};

}  // namespace

struct aqua_cfs {
  aqua_cfs_config cfg;
  int32_t mode = AQUA_POLICY_CFS;    // current policy (cfg.policy, or FCFS during a fallback)
  std::unordered_map<uint64_t, Req> reqs;
  bool have_plan = false;
  Plan plan;
  int64_t iter = 0, last = 0;
  bool finished_prev = false;
  double vclock = 0.0;
  std::vector<aqua_cfs_work> work;   // planned by next(), applied by commit()
  bool work_pending = false;
  std::vector<uint64_t> admitted;    // FCFS admission order
};

namespace {

int32_t blocks_for(const aqua_cfs* s, const Req& r, int32_t t) {
  const int64_t tok = int64_t(r.ctx) + t;
  return static_cast<int32_t>((tok + s->cfg.block_tokens - 1) / s->cfg.block_tokens);
}

bool by_arrival(const Req* a, const Req* b) {
  return a->arrival != b->arrival ? a->arrival < b->arrival : a->id < b->id;
}

// "prefill prompts having the least number of prefill tokens
// computed ... decode prompts with the least number of tokens generated";
// ties by (arrival, id) (R9).
void orders(const aqua_cfs* s, std::vector<const Req*>* pre, std::vector<const Req*>* dec) {
  for (const auto& kv : s->reqs) (kv.second.phase == AQUA_PHASE_DECODE ? dec : pre)->push_back(&kv.second);
  std::sort(pre->begin(), pre->end(), [](const Req* a, const Req* b) {
    if (a->f != b->f) return a->f < b->f;
    return by_arrival(a, b);
  });
  std::sort(dec->begin(), dec->end(), [](const Req* a, const Req* b) {
    if (a->g != b->g) return a->g < b->g;
    return by_arrival(a, b);
  });
}

Plan partition(const aqua_cfs* s) {
  const int32_t b = s->cfg.batch_tokens, NB = s->cfg.num_blocks;
  std::vector<const Req*> pre, dec;
  orders(s, &pre, &dec);
  // d = upper bound: prompts that fit (each current KV + 1 token), walked
  // in fill order (prefill first, R16), stopping at the first misfit (R12)
  int64_t mem = 0;
  int32_t fit = 0;
  for (int pass = 0; pass < 2; ++pass) {
    bool stop = false;
    for (const Req* r : pass == 0 ? pre : dec) {
      const int32_t n = blocks_for(s, *r, 1);
      if (mem + n > NB) {
        stop = true;
        break;
      }
      mem += n;
      ++fit;
    }
    if (stop) break;
  }
  const int32_t d = std::min(b, fit);
  Plan pl;
  std::vector<int32_t> alloc;
  std::vector<const Req*> chosen;
  mem = 0;
  int32_t p_left = b - d;
  for (const Req* r : pre) {
    if (p_left == 0) break;
    const int32_t a = std::min(p_left, r->P - r->f);
    const int32_t n = blocks_for(s, *r, a);
    if (mem + n > NB) break;
    mem += n;
    chosen.push_back(r);
    alloc.push_back(a);
    p_left -= a;
  }
  for (const Req* r : dec) {
    if (static_cast<int32_t>(pl.dec.size()) >= d) break;
    const int32_t n = blocks_for(s, *r, 1);
    if (mem + n > NB) break;
    mem += n;
    pl.dec.push_back(r->id);
  }
  // leftover decode slots become extra prefill tokens (R10), still within memory
  int32_t spare = d - static_cast<int32_t>(pl.dec.size());
  if (chosen.empty()) {
    // R21: no prompt chosen above (p = b - d = 0 once >= b prompts fit): the
    // spare decode slots go to prefill prompts in prefill order, walked as
    // above, so a run set of prefill-phase prompts never gets an empty plan
    for (const Req* r : pre) {
      if (spare == 0) break;
      const int32_t a = std::min(spare, r->P - r->f);
      const int32_t n = blocks_for(s, *r, a);
      if (mem + n > NB) break;
      mem += n;
      chosen.push_back(r);
      alloc.push_back(a);
      spare -= a;
    }
  }
  for (size_t i = 0; i < chosen.size() && spare > 0; ++i) {
    const Req* r = chosen[i];
    const int64_t base = mem - blocks_for(s, *r, alloc[i]);
    // largest extra <= min(spare, remaining prompt) whose blocks still fit
    int32_t hi = std::min(spare, r->P - r->f - alloc[i]);
    const int64_t room_tokens = (int64_t(NB) - base) * s->cfg.block_tokens - r->ctx - alloc[i];
    if (room_tokens < hi) hi = static_cast<int32_t>(std::max<int64_t>(room_tokens, 0));
    if (hi > 0) {
      mem = base + blocks_for(s, *r, alloc[i] + hi);
      alloc[i] += hi;
      spare -= hi;
    }
  }
  for (size_t i = 0; i < chosen.size(); ++i) pl.pre.emplace_back(chosen[i]->id, alloc[i]);
  return pl;
}

std::vector<aqua_cfs_work> work_of(const aqua_cfs* s, const Plan& pl) {
  std::vector<aqua_cfs_work> w;
  for (uint64_t id : pl.dec) {
    auto it = s->reqs.find(id);
    if (it != s->reqs.end() && it->second.phase == AQUA_PHASE_DECODE)
      w.push_back(aqua_cfs_work{id, it->second.ctx, 1, 0, AQUA_PHASE_DECODE});
  }
  for (const auto& pa : pl.pre) {
    auto it = s->reqs.find(pa.first);
    if (it != s->reqs.end() && it->second.phase == AQUA_PHASE_PREFILL)
      w.push_back(aqua_cfs_work{pa.first, it->second.ctx, std::min(pa.second, it->second.P - it->second.f), 0,
                                AQUA_PHASE_PREFILL});
  }
  return w;
}

bool fits(const aqua_cfs* s, const std::vector<aqua_cfs_work>& w) {
  std::unordered_map<uint64_t, int32_t> tok;
  for (const auto& x : w) tok[x.pid] = x.tokens;
  int64_t total = 0;
  for (const auto& kv : s->reqs) {
    const Req& r = kv.second;
    auto it = tok.find(r.id);
    if (r.where == kResident)
      total += blocks_for(s, r, it == tok.end() ? 0 : it->second);
    else if (it != tok.end())
      total += blocks_for(s, r, it->second);
  }
  return total <= s->cfg.num_blocks;
}

std::vector<uint64_t> sorted_by_arrival(const aqua_cfs* s, std::vector<uint64_t> ids) {
  std::sort(ids.begin(), ids.end(), [s](uint64_t a, uint64_t b) {
    return by_arrival(&s->reqs.at(a), &s->reqs.at(b));
  });
  return ids;
}

}  // namespace

extern "C" {

aqua_status aqua_cfs_create(const aqua_cfs_config* cfg, aqua_cfs** out) {
  if (!cfg || !out) return AQUA_E_INVAL;
  *out = nullptr;
  if (cfg->batch_tokens <= 0 || cfg->k <= 0 || cfg->block_tokens <= 0 || cfg->num_blocks <= 0 ||
      (cfg->policy != AQUA_POLICY_CFS && cfg->policy != AQUA_POLICY_FCFS))
    return AQUA_E_INVAL;
  aqua_cfs* s = new aqua_cfs();
  s->cfg = *cfg;
  s->mode = cfg->policy;
  *out = s;
  return AQUA_OK;
}

aqua_status aqua_cfs_destroy(aqua_cfs* s) {
  delete s;
  return AQUA_OK;
}

aqua_status aqua_cfs_add(aqua_cfs* s, uint64_t pid, double arrival, int32_t P, int32_t O) {
  if (!s || P < 1 || O < 1 || s->reqs.count(pid)) return AQUA_E_INVAL;
  Req r;
  r.id = pid;
  r.arrival = arrival;
  r.P = P;
  r.O = O;
  s->reqs.emplace(pid, r);
  return AQUA_OK;
}

aqua_status aqua_cfs_set_state(aqua_cfs* s, uint64_t pid, int32_t phase, int32_t f, int32_t g, int32_t ctx) {
  if (!s) return AQUA_E_INVAL;
  auto it = s->reqs.find(pid);
  if (it == s->reqs.end()) return AQUA_E_STATE;
  if (f < 0 || f > it->second.P || g < 0 || ctx < 0) return AQUA_E_INVAL;
  it->second.phase = phase;
  it->second.f = f;
  it->second.g = g;
  it->second.ctx = ctx;
  if (ctx > 0 && it->second.where == kNone) {
    // a restarted request with KV: the caller holds it as a swapped image
    // (placed with aqua_swap_out), so the next plan pages it in
    it->second.where = kSwapped;
    it->second.blocks = static_cast<int32_t>((int64_t(ctx) + s->cfg.block_tokens - 1) / s->cfg.block_tokens);
  }
  return AQUA_OK;
}

aqua_status aqua_cfs_partition(aqua_cfs* s, uint64_t* dec, int32_t* n_dec, uint64_t* pre, int32_t* pre_tok,
                               int32_t* n_pre, int32_t cap) {
  if (!s || !n_dec || !n_pre) return AQUA_E_INVAL;
  Plan pl = partition(s);
  if (static_cast<int32_t>(pl.dec.size()) > cap || static_cast<int32_t>(pl.pre.size()) > cap) return AQUA_E_INVAL;
  *n_dec = static_cast<int32_t>(pl.dec.size());
  *n_pre = static_cast<int32_t>(pl.pre.size());
  for (size_t i = 0; i < pl.dec.size(); ++i) dec[i] = pl.dec[i];
  for (size_t i = 0; i < pl.pre.size(); ++i) {
    pre[i] = pl.pre[i].first;
    pre_tok[i] = pl.pre[i].second;
  }
  return AQUA_OK;
}

aqua_status aqua_cfs_next(aqua_cfs* s, int32_t* rescheduled, uint64_t* page_out, int32_t* n_out,
                          uint64_t* page_in, int32_t* n_in, aqua_cfs_work* work, int32_t* n_work, int32_t cap) {
  if (!s || !rescheduled || !n_out || !n_in || !n_work) return AQUA_E_INVAL;
  if (s->work_pending) return AQUA_E_STATE;   // commit the previous iteration first
  *rescheduled = *n_out = *n_in = *n_work = 0;
  if (s->reqs.empty()) {
    s->have_plan = false;   // idle: the next non-empty runnable set replans
    return AQUA_OK;
  }
  std::vector<uint64_t> outs, ins;
  std::vector<aqua_cfs_work> w;
  // every failure below leaves the scheduler as it was on entry: the
  // residency flips are undone (outs were resident, ins swapped; a prompt
  // paged in and out again in one FCFS call ends swapped), and the
  // admitted set, plan and cadence are restored
  const std::vector<uint64_t> saved_admitted = s->admitted;
  const Plan saved_plan = s->plan;
  const bool saved_have = s->have_plan;
  const int64_t saved_last = s->last;
  auto fail = [&](aqua_status st) {
    for (uint64_t id : outs) s->reqs.at(id).where = kResident;
    for (uint64_t id : ins) s->reqs.at(id).where = kSwapped;
    s->admitted = saved_admitted;
    s->plan = saved_plan;
    s->have_plan = saved_have;
    s->last = saved_last;
    *rescheduled = *n_out = *n_in = *n_work = 0;
    return st;
  };
  if (s->mode == AQUA_POLICY_FCFS) {
    // admission in arrival order while the full projections fit
    int64_t proj = 0;
    for (uint64_t id : s->admitted) {
      const Req& r = s->reqs.at(id);
      proj += (int64_t(r.P) + r.O + s->cfg.block_tokens - 1) / s->cfg.block_tokens;
    }
    std::vector<const Req*> all;
    for (const auto& kv : s->reqs) all.push_back(&kv.second);
    std::sort(all.begin(), all.end(), by_arrival);
    for (const Req* r : all) {
      if (std::find(s->admitted.begin(), s->admitted.end(), r->id) != s->admitted.end()) continue;
      const int64_t n = (int64_t(r->P) + r->O + s->cfg.block_tokens - 1) / s->cfg.block_tokens;
      if (proj + n > s->cfg.num_blocks) break;
      proj += n;
      s->admitted.push_back(r->id);
      if (r->where == kSwapped) ins.push_back(r->id);      // paged in when admitted
    }
    for (uint64_t id : ins) s->reqs.at(id).where = kResident;
    auto fcfs_plan = [s]() {
      std::vector<const Req*> adm;
      for (uint64_t id : s->admitted) adm.push_back(&s->reqs.at(id));
      std::sort(adm.begin(), adm.end(), by_arrival);
      Plan pl;
      for (const Req* r : adm)
        if (r->phase == AQUA_PHASE_DECODE && static_cast<int32_t>(pl.dec.size()) < s->cfg.batch_tokens)
          pl.dec.push_back(r->id);
      int32_t left = s->cfg.batch_tokens - static_cast<int32_t>(pl.dec.size());
      for (const Req* r : adm) {
        if (r->phase != AQUA_PHASE_PREFILL || left == 0) continue;
        const int32_t t = std::min(left, r->P - r->f);
        pl.pre.emplace_back(r->id, t);
        left -= t;
      }
      return pl;
    };
    s->plan = fcfs_plan();
    s->have_plan = true;
    w = work_of(s, s->plan);
    // after a fallback the inherited residents may outgrow the pool: page out
    // the latest-arrived admitted resident until the iteration fits (R18)
    while (!w.empty() && !fits(s, w)) {
      const Req* victim = nullptr;
      for (uint64_t id : s->admitted) {
        const Req& r = s->reqs.at(id);
        if (r.where == kResident && (!victim || by_arrival(victim, &r))) victim = &r;
      }
      if (!victim) break;
      const uint64_t vid = victim->id;
      s->admitted.erase(std::find(s->admitted.begin(), s->admitted.end(), vid));
      s->reqs.at(vid).where = kSwapped;
      outs.push_back(vid);
      s->plan = fcfs_plan();
      w = work_of(s, s->plan);
    }
    if (w.empty()) return fail(AQUA_E_NOBLOCKS);   // head-of-line prompt can never fit
  } else {
    if (s->have_plan) w = work_of(s, s->plan);
    if (!s->have_plan || s->iter - s->last >= s->cfg.k || s->finished_prev || w.empty() || !fits(s, w)) {
      s->plan = partition(s);
      s->have_plan = true;
      s->last = s->iter;
      *rescheduled = 1;
      std::vector<uint64_t> in_plan(s->plan.dec);
      for (const auto& pa : s->plan.pre) in_plan.push_back(pa.first);
      std::sort(in_plan.begin(), in_plan.end());
      for (const auto& kv : s->reqs) {
        const bool planned = std::binary_search(in_plan.begin(), in_plan.end(), kv.first);
        if (kv.second.where == kResident && !planned) outs.push_back(kv.first);
        if (kv.second.where == kSwapped && planned) ins.push_back(kv.first);
      }
      outs = sorted_by_arrival(s, outs);
      ins = sorted_by_arrival(s, ins);
      for (uint64_t id : outs) s->reqs.at(id).where = kSwapped;
      for (uint64_t id : ins) s->reqs.at(id).where = kResident;
      w = work_of(s, s->plan);
      if (w.empty()) return fail(AQUA_E_NOBLOCKS);   // nothing fits: pool smaller than one prompt
    }
  }
  const int32_t nmax = static_cast<int32_t>(std::max({outs.size(), ins.size(), w.size()}));
  if (nmax > cap) return fail(AQUA_E_INVAL);
  for (auto& x : w) {
    Req& r = s->reqs.at(x.pid);
    const int32_t need = blocks_for(s, r, x.tokens);
    x.grow = std::max(0, need - r.blocks);
    r.blocks += x.grow;
    if (x.grow > 0 || r.where == kNone) r.where = kResident;
  }
  for (size_t i = 0; i < outs.size(); ++i) page_out[i] = outs[i];
  for (size_t i = 0; i < ins.size(); ++i) page_in[i] = ins[i];
  for (size_t i = 0; i < w.size(); ++i) work[i] = w[i];
  *n_out = static_cast<int32_t>(outs.size());
  *n_in = static_cast<int32_t>(ins.size());
  *n_work = static_cast<int32_t>(w.size());
  s->work = std::move(w);
  s->work_pending = true;
  return AQUA_OK;
}

aqua_status aqua_cfs_commit(aqua_cfs* s, uint64_t* finished, int32_t* n_fin, int32_t cap, double* vclock) {
  if (!s || !n_fin) return AQUA_E_INVAL;
  if (!s->work_pending) return AQUA_E_STATE;
  // count the finishes first, so a too-small `finished` array changes nothing
  int32_t n_done = 0;
  for (const auto& x : s->work) {
    const Req& r = s->reqs.at(x.pid);
    const bool decode_after = r.phase == AQUA_PHASE_DECODE || r.f + x.tokens == r.P;
    const int32_t g_after = r.phase == AQUA_PHASE_DECODE ? r.g + 1 : 1;
    n_done += decode_after && g_after >= r.O;
  }
  if (n_done > cap) return AQUA_E_INVAL;
  int64_t tokens = 0;
  for (const auto& x : s->work) tokens += x.tokens;
  s->vclock += s->cfg.t_base + s->cfg.t_token * static_cast<double>(tokens);
  std::vector<uint64_t> fin;
  for (const auto& x : s->work) {
    Req& r = s->reqs.at(x.pid);
    if (r.phase == AQUA_PHASE_PREFILL) {
      r.f += x.tokens;
      r.ctx += x.tokens;
      if (r.f == r.P) {
        r.phase = AQUA_PHASE_DECODE;
        r.g = 1;   // the first token is emitted at the end of the last prefill chunk
      }
    } else {
      r.ctx += 1;
      r.g += 1;
    }
    if (r.phase == AQUA_PHASE_DECODE && r.g >= r.O) fin.push_back(r.id);
  }
  for (size_t i = 0; i < fin.size(); ++i) {
    finished[i] = fin[i];
    s->reqs.erase(fin[i]);
    auto it = std::find(s->admitted.begin(), s->admitted.end(), fin[i]);
    if (it != s->admitted.end()) s->admitted.erase(it);
  }
  *n_fin = static_cast<int32_t>(fin.size());
  s->finished_prev = !fin.empty();
  s->iter += 1;
  s->work.clear();
  s->work_pending = false;
  if (vclock) *vclock = s->vclock;
  return AQUA_OK;
}

aqua_status aqua_cfs_set_policy(aqua_cfs* s, int32_t policy) {
  if (!s || (policy != AQUA_POLICY_CFS && policy != AQUA_POLICY_FCFS)) return AQUA_E_INVAL;
  if (s->work_pending) return AQUA_E_STATE;
  if (policy == s->mode) return AQUA_OK;
  s->mode = policy;
  s->admitted.clear();
  if (policy == AQUA_POLICY_FCFS) {
    // the prompts already on the GPU are the admitted ones, in arrival order
    std::vector<const Req*> res;
    for (const auto& kv : s->reqs)
      if (kv.second.where == kResident) res.push_back(&kv.second);
    std::sort(res.begin(), res.end(), by_arrival);
    for (const Req* r : res) s->admitted.push_back(r->id);
  } else {
    s->have_plan = false;    // replan at once
  }
  return AQUA_OK;
}

aqua_status aqua_cfs_vclock(aqua_cfs* s, double* v) {
  if (!s || !v) return AQUA_E_INVAL;
  *v = s->vclock;
  return AQUA_OK;
}

aqua_status aqua_cfs_advance_to(aqua_cfs* s, double v) {
  if (!s || v < s->vclock) return AQUA_E_INVAL;
  s->vclock = v;
  return AQUA_OK;
}

aqua_status aqua_cfs_stats(aqua_cfs* s, int32_t* runnable, int32_t* resident, int64_t* iterations) {
  if (!s) return AQUA_E_INVAL;
  if (runnable) *runnable = static_cast<int32_t>(s->reqs.size());
  if (resident) {
    int32_t n = 0;
    for (const auto& kv : s->reqs) n += kv.second.where == kResident;
    *resident = n;
  }
  if (iterations) *iterations = s->iter;
  return AQUA_OK;
}

}  // extern "C"
