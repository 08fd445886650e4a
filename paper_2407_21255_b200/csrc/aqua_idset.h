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

  // Remove the k lowest free ids (k <= size()).
  void erase_lowest(int32_t k) {
    const int32_t nw = static_cast<int32_t>(w_.size());
    while (k > 0 && lo_ < nw) {
      uint64_t& x = w_[lo_];
      while (x && k > 0) {
        x &= x - 1;
        --k;
        --count_;
      }
      if (!x) ++lo_;
    }
  }

 private:
  std::vector<uint64_t> w_;
  int32_t n_ = 0, count_ = 0, lo_ = 0;   // lo_: no set bit in words below it
};

}  // namespace aqua
