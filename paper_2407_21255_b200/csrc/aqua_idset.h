// Free-id set for blocks and slots: a bitmap with lowest-first iteration
// (reading R4: allocations take the lowest free ids, ascending).  Replaces a
// node-based std::set: O(1) insert / erase and word-at-a-time scans keep the
// host cost of a 2048-block swap in the tens of microseconds.
#pragma once
#include <cstdint>
#include <vector>

namespace aqua {

class IdSet {
 public:
  void init(int32_t n, bool all_free) {
    n_ = n;
    w_.assign((static_cast<size_t>(n) + 63) / 64, all_free ? ~uint64_t(0) : 0);
    if (all_free && (n & 63)) w_.back() = (uint64_t(1) << (n & 63)) - 1;
    count_ = all_free ? n : 0;
    lo_ = 0;
  }
  int32_t size() const { return count_; }
  bool count(int32_t id) const { return (w_[id >> 6] >> (id & 63)) & 1; }
  void insert(int32_t id) {
    uint64_t& x = w_[id >> 6];
    const uint64_t b = uint64_t(1) << (id & 63);
    if (!(x & b)) {
      x |= b;
      ++count_;
      if ((id >> 6) < lo_) lo_ = id >> 6;
    }
  }
  void erase(int32_t id) {
    uint64_t& x = w_[id >> 6];
    const uint64_t b = uint64_t(1) << (id & 63);
    if (x & b) {
      x &= ~b;
      --count_;
    }
  }

  // Ascending iteration over the free ids.
  class iterator {
   public:
    iterator(const IdSet* s, int32_t word) : s_(s), word_(word), bits_(0) {
      if (word_ < static_cast<int32_t>(s_->w_.size())) bits_ = s_->w_[word_];
      advance();
    }
    int32_t operator*() const { return cur_; }
    iterator& operator++() {
      bits_ &= bits_ - 1;
      advance();
      return *this;
    }
    iterator operator++(int) {
      iterator t = *this;
      ++*this;
      return t;
    }
    bool at_end() const { return cur_ < 0; }

   private:
    void advance() {
      const int32_t nw = static_cast<int32_t>(s_->w_.size());
      while (!bits_ && ++word_ < nw) bits_ = s_->w_[word_];
      cur_ = bits_ ? word_ * 64 + __builtin_ctzll(bits_) : -1;
    }
    const IdSet* s_;
    int32_t word_;
    uint64_t bits_;
    int32_t cur_ = -1;
  };

  iterator begin() {
    const int32_t nw = static_cast<int32_t>(w_.size());
    while (lo_ < nw && !w_[lo_]) ++lo_;
    return iterator(this, lo_);
  }

  // Bulk insert / erase of n ids (same semantics as n single calls).  Ids
  // are taken in runs that fall in one bitmap word (slots and fresh blocks
  // come sorted, so runs are long): each run is one read-modify-write of its
  // word and a popcount, not one dependent update per id.
  void insert_all(const int32_t* ids, size_t n) {
    uint64_t* w = w_.data();
    int32_t cnt = count_, lo = lo_;
    size_t i = 0;
    while (i < n) {
      const int32_t wd = ids[i] >> 6;
      uint64_t m = 0;
      do m |= uint64_t(1) << (ids[i] & 63);
      while (++i < n && (ids[i] >> 6) == wd);
      const uint64_t add = m & ~w[wd];
      if (add) {
        w[wd] |= add;
        cnt += __builtin_popcountll(add);
        if (wd < lo) lo = wd;
      }
    }
    count_ = cnt;
    lo_ = lo;
  }
  void erase_all(const int32_t* ids, size_t n) {
    uint64_t* w = w_.data();
    int32_t cnt = count_;
    size_t i = 0;
    while (i < n) {
      const int32_t wd = ids[i] >> 6;
      uint64_t m = 0;
      do m |= uint64_t(1) << (ids[i] & 63);
      while (++i < n && (ids[i] >> 6) == wd);
      const uint64_t del = m & w[wd];
      w[wd] &= ~del;
      cnt -= __builtin_popcountll(del);
    }
    count_ = cnt;
  }

  // Ascending scan over the free ids that leaves the set unchanged; fill()
  // writes the next k ids (fewer if the set runs out) with the scan state in
  // locals, a few cycles per id.
  struct Scan {
    const uint64_t* w;
    int32_t nw, word;
    uint64_t bits;
  };
  Scan scan() {
    const int32_t nw = static_cast<int32_t>(w_.size());
    while (lo_ < nw && !w_[lo_]) ++lo_;
    return Scan{w_.data(), nw, lo_, lo_ < nw ? w_[lo_] : 0};
  }
  static int32_t fill(Scan& s, int32_t k, int32_t* out) {
    const uint64_t* w = s.w;
    int32_t word = s.word, got = 0;
    uint64_t bits = s.bits;
    while (got < k) {
      while (!bits) {
        if (++word >= s.nw) {
          s.word = word;
          s.bits = 0;
          return got;
        }
        bits = w[word];
      }
      out[got++] = word * 64 + __builtin_ctzll(bits);
      bits &= bits - 1;
    }
    s.word = word;
    s.bits = bits;
    return got;
  }

  // Remove the k lowest free ids (k <= size()).
  void erase_lowest(int32_t k) {
    const int32_t nw = static_cast<int32_t>(w_.size());
    while (k > 0 && lo_ < nw) {
      uint64_t& x = w_[lo_];
      const int32_t pc = __builtin_popcountll(x);
      if (pc <= k) {                 // the whole word goes
        x = 0;
        k -= pc;
        count_ -= pc;
        ++lo_;
      } else {                       // the lowest k bits of this word
        count_ -= k;
        while (k > 0) {
          x &= x - 1;
          --k;
        }
      }
    }
  }

 private:
  std::vector<uint64_t> w_;
  int32_t n_ = 0, count_ = 0, lo_ = 0;   // lo_: no set bit in words below it
};

}  // namespace aqua
