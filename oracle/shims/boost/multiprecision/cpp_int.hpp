// ORACLE BUILD SHIM — test infrastructure only, never linked into the product.
//
// The reference includes <boost/multiprecision/cpp_int.hpp>
// (/root/reference/proj/include/enserve/opt/optimizer.hpp:9) but does not vendor
// boost (/root/reference/proj/.gitignore:2).  Only count_total_matrices /
// for_each_matrix use it (src/opt/optimizer.cpp:105-163): pow, subtraction of 1,
// comparisons, str() and convert_to<uint64_t>().  This header supplies exactly
// that surface as an arbitrary-precision unsigned integer so the reference
// compiles unmodified from its own sources (oracle/Makefile).
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  cpp_int() = default;
  template <typename I, typename = std::enable_if_t<std::is_integral_v<I>>>
  cpp_int(I v) {  // NOLINT(implicit)
    if constexpr (std::is_signed_v<I>) {
      if (v < 0) throw std::domain_error("shim cpp_int is unsigned");
    }
    unsigned long long u = static_cast<unsigned long long>(v);
    while (u) {
      limbs_.push_back(static_cast<std::uint32_t>(u));
      u >>= 32;
    }
  }
  explicit cpp_int(const char* s) { parse(s); }
  explicit cpp_int(const std::string& s) { parse(s.c_str()); }

  std::string str() const {
    if (limbs_.empty()) return "0";
    std::vector<std::uint32_t> t = limbs_;
    std::string out;
    while (!t.empty()) {
      std::uint64_t rem = 0;
      for (std::size_t i = t.size(); i-- > 0;) {
        std::uint64_t cur = (rem << 32) | t[i];
        t[i] = static_cast<std::uint32_t>(cur / 10);
        rem = cur % 10;
      }
      out.push_back(static_cast<char>('0' + rem));
      while (!t.empty() && t.back() == 0) t.pop_back();
    }
    std::reverse(out.begin(), out.end());
    return out;
  }

  template <typename T>
  T convert_to() const {
    unsigned long long u = 0;
    for (std::size_t i = limbs_.size(); i-- > 0;) u = (u << 32) | limbs_[i];
    return static_cast<T>(u);
  }

  friend cpp_int operator*(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    if (a.limbs_.empty() || b.limbs_.empty()) return r;
    r.limbs_.assign(a.limbs_.size() + b.limbs_.size(), 0);
    for (std::size_t i = 0; i < a.limbs_.size(); ++i) {
      std::uint64_t carry = 0;
      for (std::size_t j = 0; j < b.limbs_.size(); ++j) {
        std::uint64_t cur = static_cast<std::uint64_t>(a.limbs_[i]) * b.limbs_[j] +
                            r.limbs_[i + j] + carry;
        r.limbs_[i + j] = static_cast<std::uint32_t>(cur);
        carry = cur >> 32;
      }
      std::size_t k = i + b.limbs_.size();
      while (carry) {
        std::uint64_t cur = static_cast<std::uint64_t>(r.limbs_[k]) + carry;
        r.limbs_[k++] = static_cast<std::uint32_t>(cur);
        carry = cur >> 32;
      }
    }
    r.trim();
    return r;
  }
  friend cpp_int operator+(const cpp_int& a, const cpp_int& b) {
    cpp_int r;
    std::size_t n = std::max(a.limbs_.size(), b.limbs_.size());
    std::uint64_t carry = 0;
    for (std::size_t i = 0; i < n || carry; ++i) {
      std::uint64_t cur = carry;
      if (i < a.limbs_.size()) cur += a.limbs_[i];
      if (i < b.limbs_.size()) cur += b.limbs_[i];
      r.limbs_.push_back(static_cast<std::uint32_t>(cur));
      carry = cur >> 32;
    }
    r.trim();
    return r;
  }
  friend cpp_int operator-(const cpp_int& a, const cpp_int& b) {
    if (a < b) throw std::domain_error("shim cpp_int underflow");
    cpp_int r = a;
    std::int64_t borrow = 0;
    for (std::size_t i = 0; i < r.limbs_.size(); ++i) {
      std::int64_t cur = static_cast<std::int64_t>(r.limbs_[i]) - borrow -
                         (i < b.limbs_.size() ? b.limbs_[i] : 0);
      borrow = cur < 0 ? 1 : 0;
      if (cur < 0) cur += (std::int64_t(1) << 32);
      r.limbs_[i] = static_cast<std::uint32_t>(cur);
    }
    r.trim();
    return r;
  }
  template <typename I, typename = std::enable_if_t<std::is_integral_v<I>>>
  friend cpp_int operator-(const cpp_int& a, I b) { return a - cpp_int(b); }

  friend int compare(const cpp_int& a, const cpp_int& b) {
    if (a.limbs_.size() != b.limbs_.size())
      return a.limbs_.size() < b.limbs_.size() ? -1 : 1;
    for (std::size_t i = a.limbs_.size(); i-- > 0;)
      if (a.limbs_[i] != b.limbs_[i]) return a.limbs_[i] < b.limbs_[i] ? -1 : 1;
    return 0;
  }
  friend bool operator==(const cpp_int& a, const cpp_int& b) { return compare(a, b) == 0; }
  friend bool operator!=(const cpp_int& a, const cpp_int& b) { return compare(a, b) != 0; }
  friend bool operator<(const cpp_int& a, const cpp_int& b) { return compare(a, b) < 0; }
  friend bool operator>(const cpp_int& a, const cpp_int& b) { return compare(a, b) > 0; }
  friend bool operator<=(const cpp_int& a, const cpp_int& b) { return compare(a, b) <= 0; }
  friend bool operator>=(const cpp_int& a, const cpp_int& b) { return compare(a, b) >= 0; }

 private:
  void trim() {
    while (!limbs_.empty() && limbs_.back() == 0) limbs_.pop_back();
  }
  void parse(const char* s) {
    limbs_.clear();
    for (; *s; ++s) {
      if (*s < '0' || *s > '9') throw std::invalid_argument("shim cpp_int: bad digit");
      *this = *this * cpp_int(10u) + cpp_int(static_cast<unsigned>(*s - '0'));
    }
  }
  std::vector<std::uint32_t> limbs_;  // little-endian base 2^32
};

inline cpp_int pow(const cpp_int& base, unsigned exp) {
  cpp_int result(1u), b = base;
  while (exp) {
    if (exp & 1u) result = result * b;
    exp >>= 1u;
    if (exp) b = b * b;
  }
  return result;
}

}  // namespace multiprecision
}  // namespace boost
