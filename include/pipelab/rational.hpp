// pipelab drop-in: exact rational numbers for byte accounting.
//
// Source-compatible replacement for the reference's pipelab::Rat
// (reference: proj/include/pipelab/rational.hpp:15-98).  Values are kept as a
// reduced fraction of two int64 with a positive denominator; intermediate
// products are formed in 128-bit so the only failure mode is a reduced
// result that does not fit int64 (std::overflow_error).  Conversion to whole
// bytes happens only through ceil_int().
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace pipelab {

class Rat {
  using wide = __int128;

 public:
  constexpr Rat() = default;
  Rat(std::int64_t value) : num_(value) {}
  Rat(std::int64_t numerator, std::int64_t denominator) { *this = reduce(numerator, denominator); }

  std::int64_t num() const { return num_; }
  std::int64_t den() const { return den_; }
  bool is_integer() const { return den_ == 1; }
  double to_double() const { return double(num_) / double(den_); }

  // Smallest integer >= value; defined for non-negative values only.
  std::int64_t ceil_int() const {
    if (num_ < 0) throw std::domain_error("Rat::ceil_int: negative value");
    return num_ / den_ + (num_ % den_ != 0 ? 1 : 0);
  }

  std::string str() const {
    return den_ == 1 ? std::to_string(num_) : std::to_string(num_) + "/" + std::to_string(den_);
  }

  friend Rat operator+(const Rat& x, const Rat& y) {
    return reduce(wide(x.num_) * y.den_ + wide(y.num_) * x.den_, wide(x.den_) * y.den_);
  }
  friend Rat operator-(const Rat& x, const Rat& y) {
    return reduce(wide(x.num_) * y.den_ - wide(y.num_) * x.den_, wide(x.den_) * y.den_);
  }
  friend Rat operator*(const Rat& x, const Rat& y) {
    return reduce(wide(x.num_) * y.num_, wide(x.den_) * y.den_);
  }
  friend Rat operator/(const Rat& x, const Rat& y) {
    if (y.num_ == 0) throw std::domain_error("Rat: division by zero");
    return reduce(wide(x.num_) * y.den_, wide(x.den_) * y.num_);
  }
  Rat& operator+=(const Rat& y) { return *this = *this + y; }
  Rat& operator-=(const Rat& y) { return *this = *this - y; }
  Rat& operator*=(const Rat& y) { return *this = *this * y; }
  Rat& operator/=(const Rat& y) { return *this = *this / y; }

  friend bool operator==(const Rat& x, const Rat& y) { return x.num_ == y.num_ && x.den_ == y.den_; }
  friend bool operator!=(const Rat& x, const Rat& y) { return !(x == y); }
  friend bool operator<(const Rat& x, const Rat& y) { return wide(x.num_) * y.den_ < wide(y.num_) * x.den_; }
  friend bool operator>(const Rat& x, const Rat& y) { return y < x; }
  friend bool operator<=(const Rat& x, const Rat& y) { return !(y < x); }
  friend bool operator>=(const Rat& x, const Rat& y) { return !(x < y); }

 private:
  static Rat reduce(wide n, wide d) {
    if (d == 0) throw std::domain_error("Rat: zero denominator");
    if (d < 0) n = -n, d = -d;
    wide a = n < 0 ? -n : n, b = d;
    while (b != 0) {  // Euclid on magnitudes
      wide t = a % b;
      a = b;
      b = t;
    }
    if (a > 1) n /= a, d /= a;
    const wide lim = wide(INT64_MAX);
    if (n > lim || n < -lim - 1 || d > lim) throw std::overflow_error("Rat: value out of 64-bit range");
    Rat r;
    r.num_ = std::int64_t(n);
    r.den_ = std::int64_t(d);
    return r;
  }

  std::int64_t num_ = 0;
  std::int64_t den_ = 1;
};

}  // namespace pipelab
