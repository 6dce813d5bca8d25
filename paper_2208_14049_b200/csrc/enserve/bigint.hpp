// Minimal arbitrary-precision unsigned integer for the matrix-space size
// ((B+1)^D - 1)^M, which overflows 128 bits already at 8 devices x 12 models
// (~5.0e74).  The reference uses boost::multiprecision::cpp_int for this
// (/root/reference/proj/include/enserve/opt/optimizer.hpp:9,15); this build has
// no boost dependency.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace enserve {

class BigUInt {
 public:
  BigUInt() = default;
  BigUInt(std::uint64_t v) {  // NOLINT(implicit): small literals read naturally
    for (; v; v >>= 32) words_.push_back(static_cast<std::uint32_t>(v));
  }

  static BigUInt parse(const std::string& digits) {
    BigUInt r;
    for (char ch : digits) {
      if (ch < '0' || ch > '9') throw std::invalid_argument("BigUInt: not a decimal digit");
      r = r.mul_small(10);
      r = r + BigUInt(static_cast<std::uint64_t>(ch - '0'));
    }
    return r;
  }

  bool fits_u64() const { return words_.size() <= 2; }
  std::uint64_t to_u64() const {
    std::uint64_t v = 0;
    for (std::size_t i = std::min<std::size_t>(words_.size(), 2); i-- > 0;) v = (v << 32) | words_[i];
    return v;
  }

  std::string str() const {
    if (words_.empty()) return "0";
    std::string out;
    BigUInt t = *this;
    while (!t.words_.empty()) out.push_back(static_cast<char>('0' + t.divmod_small(10)));
    std::reverse(out.begin(), out.end());
    return out;
  }

  BigUInt mul_small(std::uint32_t k) const {
    BigUInt r;
    std::uint64_t carry = 0;
    for (std::uint32_t w : words_) {
      std::uint64_t cur = static_cast<std::uint64_t>(w) * k + carry;
      r.words_.push_back(static_cast<std::uint32_t>(cur));
      carry = cur >> 32;
    }
    if (carry) r.words_.push_back(static_cast<std::uint32_t>(carry));
    r.normalize();
    return r;
  }

  friend BigUInt operator*(const BigUInt& a, const BigUInt& b) {
    BigUInt r;
    if (a.words_.empty() || b.words_.empty()) return r;
    r.words_.assign(a.words_.size() + b.words_.size(), 0u);
    for (std::size_t i = 0; i < a.words_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < b.words_.size() || carry; ++j) {
        std::uint64_t cur = r.words_[i + j] + carry +
                            (j < b.words_.size() ? static_cast<std::uint64_t>(a.words_[i]) * b.words_[j] : 0);
        r.words_[i + j] = static_cast<std::uint32_t>(cur);
        carry = cur >> 32;
      }
    }
    r.normalize();
    return r;
  }

  friend BigUInt operator+(const BigUInt& a, const BigUInt& b) {
    BigUInt r;
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < std::max(a.words_.size(), b.words_.size()) || carry; ++i) {
      std::uint64_t cur = carry + (i < a.words_.size() ? a.words_[i] : 0u) +
                          (i < b.words_.size() ? b.words_[i] : 0u);
      r.words_.push_back(static_cast<std::uint32_t>(cur));
      carry = cur >> 32;
    }
    r.normalize();
    return r;
  }

  // a - b for a >= b.
  friend BigUInt operator-(const BigUInt& a, const BigUInt& b) {
    if (a < b) throw std::domain_error("BigUInt: negative result");
    BigUInt r = a;
    std::uint64_t borrow = 0;
    for (std::size_t i = 0; i < r.words_.size(); ++i) {
      std::uint64_t sub = borrow + (i < b.words_.size() ? b.words_[i] : 0u);
      std::uint64_t cur = static_cast<std::uint64_t>(r.words_[i]);
      borrow = cur < sub ? 1 : 0;
      r.words_[i] = static_cast<std::uint32_t>(cur + (borrow << 32) - sub);
    }
    r.normalize();
    return r;
  }

  friend BigUInt pow(BigUInt base, unsigned exp) {
    BigUInt acc(1);
    for (; exp; exp >>= 1) {
      if (exp & 1u) acc = acc * base;
      if (exp > 1) base = base * base;
    }
    return acc;
  }

  friend int cmp(const BigUInt& a, const BigUInt& b) {
    if (a.words_.size() != b.words_.size()) return a.words_.size() < b.words_.size() ? -1 : 1;
    for (std::size_t i = a.words_.size(); i-- > 0;)
      if (a.words_[i] != b.words_[i]) return a.words_[i] < b.words_[i] ? -1 : 1;
    return 0;
  }
  friend bool operator==(const BigUInt& a, const BigUInt& b) { return cmp(a, b) == 0; }
  friend bool operator<(const BigUInt& a, const BigUInt& b) { return cmp(a, b) < 0; }
  friend bool operator>(const BigUInt& a, const BigUInt& b) { return cmp(a, b) > 0; }

 private:
  std::uint32_t divmod_small(std::uint32_t k) {
    std::uint64_t rem = 0;
    for (std::size_t i = words_.size(); i-- > 0;) {
      std::uint64_t cur = (rem << 32) | words_[i];
      words_[i] = static_cast<std::uint32_t>(cur / k);
      rem = cur % k;
    }
    normalize();
    return static_cast<std::uint32_t>(rem);
  }
  void normalize() {
    while (!words_.empty() && words_.back() == 0) words_.pop_back();
  }
  std::vector<std::uint32_t> words_;  // little-endian, base 2^32
};

}  // namespace enserve
