// Unit test of the host library's free-id bitmap (csrc/aqua_idset.h) against
// a plain std::set model: random mixes of single and bulk inserts / erases
// (ids present or absent, duplicates, sorted runs and scattered ids),
// erase_lowest and the lowest-first scan.  Prints "ok <ops>" or the first
// mismatch.  Built and run by tests/test_idset.py (g++, no CUDA).
#include <cstdio>
#include <random>
#include <set>
#include <vector>

#include "aqua_idset.h"

static bool same(aqua::IdSet& s, const std::set<int32_t>& m, int n) {
  if (s.size() != static_cast<int32_t>(m.size())) return false;
  for (int i = 0; i < n; ++i)
    if (s.count(i) != (m.count(i) == 1)) return false;
  std::vector<int32_t> got;
  for (auto it = s.begin(); !it.at_end(); ++it) got.push_back(*it);
  if (got != std::vector<int32_t>(m.begin(), m.end())) return false;
  std::vector<int32_t> f(m.size() + 3, -1);
  aqua::IdSet::Scan sc = s.scan();
  const int32_t k = aqua::IdSet::fill(sc, static_cast<int32_t>(m.size()) + 3, f.data());
  if (k != static_cast<int32_t>(m.size())) return false;
  return std::equal(m.begin(), m.end(), f.begin());
}

int main() {
  std::mt19937 rng(7);
  long ops = 0;
  for (int trial = 0; trial < 300; ++trial) {
    const int n = 1 + static_cast<int>(rng() % 700);
    aqua::IdSet s;
    std::set<int32_t> m;
    const bool full = rng() & 1;
    s.init(n, full);
    if (full)
      for (int i = 0; i < n; ++i) m.insert(i);
    for (int step = 0; step < 60; ++step, ++ops) {
      const int kind = static_cast<int>(rng() % 5);
      std::vector<int32_t> ids(rng() % 80);
      const bool sorted = rng() & 1;
      int32_t base = static_cast<int32_t>(rng() % n);
      for (auto& x : ids) {
        x = sorted ? base : static_cast<int32_t>(rng() % n);
        if (sorted) base = std::min(n - 1, base + static_cast<int32_t>(rng() % 3));   // runs, repeats
      }
      if (kind == 0) {
        s.insert_all(ids.data(), ids.size());
        m.insert(ids.begin(), ids.end());
      } else if (kind == 1) {
        s.erase_all(ids.data(), ids.size());
        for (int32_t x : ids) m.erase(x);
      } else if (kind == 2) {
        for (int32_t x : ids) s.insert(x), m.insert(x);
      } else if (kind == 3) {
        for (int32_t x : ids) s.erase(x), m.erase(x);
      } else {
        const int32_t k = static_cast<int32_t>(rng() % (m.size() + 1));
        s.erase_lowest(k);
        for (int32_t i = 0; i < k; ++i) m.erase(m.begin());
      }
      if (!same(s, m, n)) {
        std::printf("mismatch trial %d step %d kind %d n %d\n", trial, step, kind, n);
        return 1;
      }
    }
  }
  std::printf("ok %ld\n", ops);
  return 0;
}
