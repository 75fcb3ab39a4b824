// ORACLE BUILD SHIM — test infrastructure only, never linked into the product.
//
// Boost.Multiprecision is not installed in this image.  The reference's hot
// path touches BigInt only for integer order formulas
// (/root/reference/proj/src/solver.cpp:182-205,
//  /root/reference/proj/src/factorized.cpp:13-19,114,151-154), all of which
// fit an unsigned 128-bit integer for the inputs the parity suite uses
// (orders <= 2^62 are guarded by the reference itself).  This header
// provides exactly that subset so the reference sources compile unmodified
// from /root/reference.  Arithmetic saturates at 2^128-1 instead of growing,
// which only matters for formula-only paths the oracle never exercises.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

namespace boost {
namespace multiprecision {

class cpp_int {
 public:
  using u128 = unsigned __int128;
  static constexpr u128 kMax = ~static_cast<u128>(0);

  cpp_int() = default;
  template <class I, class = decltype(static_cast<u128>(I{}))>
  cpp_int(I v) : v_(v < I{} ? 0 : static_cast<u128>(v)) {}

  explicit operator std::size_t() const { return static_cast<std::size_t>(v_); }
  explicit operator unsigned long long() const { return static_cast<unsigned long long>(v_); }
  explicit operator double() const { return static_cast<double>(v_); }

  friend cpp_int operator+(cpp_int a, cpp_int b) {
    cpp_int r; r.v_ = (a.v_ > kMax - b.v_) ? kMax : a.v_ + b.v_; return r;
  }
  friend cpp_int operator-(cpp_int a, cpp_int b) {
    cpp_int r; r.v_ = a.v_ < b.v_ ? 0 : a.v_ - b.v_; return r;
  }
  friend cpp_int operator*(cpp_int a, cpp_int b) {
    cpp_int r;
    r.v_ = (a.v_ != 0 && b.v_ > kMax / a.v_) ? kMax : a.v_ * b.v_;
    return r;
  }
  friend cpp_int operator&(cpp_int a, cpp_int b) { cpp_int r; r.v_ = a.v_ & b.v_; return r; }
  friend cpp_int operator<<(cpp_int a, unsigned s) {
    cpp_int r;
    if (s >= 128 || (s > 0 && (a.v_ >> (128 - s)) != 0)) r.v_ = a.v_ == 0 ? 0 : kMax;
    else r.v_ = a.v_ << s;
    return r;
  }
  friend cpp_int operator<<(cpp_int a, int s) { return a << static_cast<unsigned>(s); }
  cpp_int& operator<<=(unsigned s) { *this = *this << s; return *this; }
  cpp_int& operator+=(cpp_int b) { *this = *this + b; return *this; }
  cpp_int& operator*=(cpp_int b) { *this = *this * b; return *this; }

  friend bool operator<(cpp_int a, cpp_int b) { return a.v_ < b.v_; }
  friend bool operator>(cpp_int a, cpp_int b) { return a.v_ > b.v_; }
  friend bool operator<=(cpp_int a, cpp_int b) { return a.v_ <= b.v_; }
  friend bool operator>=(cpp_int a, cpp_int b) { return a.v_ >= b.v_; }
  friend bool operator==(cpp_int a, cpp_int b) { return a.v_ == b.v_; }
  friend bool operator!=(cpp_int a, cpp_int b) { return a.v_ != b.v_; }

  std::string str() const {
    if (v_ == 0) return "0";
    std::string s;
    u128 v = v_;
    while (v) { s.insert(s.begin(), static_cast<char>('0' + static_cast<int>(v % 10))); v /= 10; }
    return s;
  }
  u128 raw() const { return v_; }

 private:
  u128 v_ = 0;
};

inline cpp_int pow(cpp_int base, unsigned e) {
  cpp_int r(1);
  while (e--) r = r * base;
  return r;
}

inline unsigned msb(const cpp_int& v) {
  unsigned b = 0;
  for (auto x = v.raw(); x > 1; x >>= 1) ++b;
  return b;
}

// Only named by proj/include/nn/bigint.hpp:9; the hot path never uses it.
struct cpp_rational {
  cpp_int num{0}, den{1};
};

}  // namespace multiprecision
}  // namespace boost
