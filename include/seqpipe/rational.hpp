// seqpipe::Rational — exact int64 fractions for costs, times and imbalance.
//
// Behavioural contract follows the reference header
// /root/reference/proj/core/include/seqpipe/rational.hpp:45-215: values are kept
// reduced with a positive denominator, every product goes through 128-bit
// integers, and narrowing back to 64 bits throws std::overflow_error rather
// than wrapping. parse() accepts "n", "n/d" and "x.y"; format_decimal rounds
// half away from zero.
#pragma once

#include <compare>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>

namespace seqpipe {
namespace detail {

using Int128 = __int128;

constexpr Int128 iabs(Int128 x) { return x < 0 ? -x : x; }

constexpr Int128 igcd(Int128 x, Int128 y) {
  x = iabs(x);
  y = iabs(y);
  while (y) {
    Int128 r = x % y;
    x = y;
    y = r;
  }
  return x;
}

inline std::int64_t to_i64(Int128 x) {
  constexpr Int128 kHi = static_cast<Int128>(INT64_MAX);
  constexpr Int128 kLo = static_cast<Int128>(INT64_MIN);
  if (x > kHi || x < kLo) throw std::overflow_error("rational overflow: value does not fit in int64");
  return static_cast<std::int64_t>(x);
}

// Decimal rendering of a 128-bit integer (std::to_string has no __int128 overload).
inline std::string int128_str(Int128 v) {
  if (v == 0) return "0";
  bool neg = v < 0;
  unsigned __int128 u = neg ? static_cast<unsigned __int128>(-(v + 1)) + 1u : static_cast<unsigned __int128>(v);
  char buf[48];
  int i = 47;
  buf[i] = 0;
  while (u) {
    buf[--i] = static_cast<char>('0' + static_cast<int>(u % 10));
    u /= 10;
  }
  if (neg) buf[--i] = '-';
  return std::string(buf + i);
}

}  // namespace detail

class Rational {
 public:
  constexpr Rational() = default;
  constexpr Rational(std::int64_t v) : n_(v), d_(1) {}  // NOLINT: implicit by design (as the reference)
  constexpr Rational(int v) : n_(v), d_(1) {}           // NOLINT
  Rational(std::int64_t num, std::int64_t den) { *this = reduce(num, den); }

  // Reduces a 128-bit fraction; throws domain_error on a zero denominator and
  // overflow_error when the reduced terms do not fit in int64.
  static Rational reduce(detail::Int128 num, detail::Int128 den) {
    if (den == 0) throw std::domain_error("rational: zero denominator");
    if (den < 0) {
      num = -num;
      den = -den;
    }
    detail::Int128 g = detail::igcd(num, den);
    if (g > 1) {
      num /= g;
      den /= g;
    }
    Rational out;
    out.n_ = detail::to_i64(num);
    out.d_ = detail::to_i64(den);
    return out;
  }
  // Reference spelling of reduce().
  static Rational from_parts(detail::Int128 num, detail::Int128 den) { return reduce(num, den); }

  static Rational parse(std::string_view text);

  std::int64_t numerator() const { return n_; }
  std::int64_t denominator() const { return d_; }
  bool is_zero() const { return n_ == 0; }
  bool is_integer() const { return d_ == 1; }
  bool is_negative() const { return n_ < 0; }
  bool is_positive() const { return n_ > 0; }
  double to_double() const { return static_cast<double>(n_) / static_cast<double>(d_); }
  std::string str() const { return d_ == 1 ? std::to_string(n_) : std::to_string(n_) + "/" + std::to_string(d_); }

  Rational operator-() const {
    Rational r;
    r.n_ = -n_;
    r.d_ = d_;
    return r;
  }
  friend Rational operator+(const Rational& x, const Rational& y) {
    using detail::Int128;
    return reduce(Int128(x.n_) * y.d_ + Int128(y.n_) * x.d_, Int128(x.d_) * y.d_);
  }
  friend Rational operator-(const Rational& x, const Rational& y) {
    using detail::Int128;
    return reduce(Int128(x.n_) * y.d_ - Int128(y.n_) * x.d_, Int128(x.d_) * y.d_);
  }
  friend Rational operator*(const Rational& x, const Rational& y) {
    using detail::Int128;
    return reduce(Int128(x.n_) * y.n_, Int128(x.d_) * y.d_);
  }
  friend Rational operator/(const Rational& x, const Rational& y) {
    using detail::Int128;
    if (y.n_ == 0) throw std::domain_error("rational: division by zero");
    return reduce(Int128(x.n_) * y.d_, Int128(x.d_) * y.n_);
  }
  Rational& operator+=(const Rational& o) { return *this = *this + o; }
  Rational& operator-=(const Rational& o) { return *this = *this - o; }
  Rational& operator*=(const Rational& o) { return *this = *this * o; }
  Rational& operator/=(const Rational& o) { return *this = *this / o; }

  friend bool operator==(const Rational& x, const Rational& y) { return x.n_ == y.n_ && x.d_ == y.d_; }
  friend std::strong_ordering operator<=>(const Rational& x, const Rational& y) {
    using detail::Int128;
    Int128 l = Int128(x.n_) * y.d_, r = Int128(y.n_) * x.d_;
    return l < r ? std::strong_ordering::less : (l > r ? std::strong_ordering::greater : std::strong_ordering::equal);
  }

 private:
  std::int64_t n_ = 0;
  std::int64_t d_ = 1;
};

inline Rational abs(const Rational& r) { return r.is_negative() ? -r : r; }

inline Rational Rational::parse(std::string_view text) {
  using detail::Int128;
  const std::string shown(text);
  auto bad = [&shown]() -> std::invalid_argument {
    return std::invalid_argument("cannot parse rational from '" + shown + "'");
  };
  std::size_t i = 0;
  bool neg = false;
  if (i < text.size() && (text[i] == '-' || text[i] == '+')) neg = text[i++] == '-';
  // Reads a run of digits; returns the digit count.
  auto digits = [&](Int128& v) {
    std::size_t start = i;
    v = 0;
    for (; i < text.size() && text[i] >= '0' && text[i] <= '9'; ++i) {
      v = v * 10 + (text[i] - '0');
      if (v > Int128(INT64_MAX) * 1000000) throw std::overflow_error("rational literal too large");
    }
    return i - start;
  };
  Int128 whole = 0;
  if (digits(whole) == 0) throw bad();
  Int128 num = whole, den = 1;
  if (i < text.size()) {
    char sep = text[i++];
    Int128 tail = 0;
    std::size_t nd = digits(tail);
    if (nd == 0 || i != text.size()) throw bad();
    if (sep == '/') {
      if (tail == 0) throw bad();
      den = tail;
    } else if (sep == '.') {
      for (std::size_t j = 0; j < nd; ++j) den *= 10;
      num = whole * den + tail;
    } else {
      throw bad();
    }
  }
  return reduce(neg ? -num : num, den);
}

// Fixed-point decimal with round-half-away-from-zero, e.g. format_decimal(2/3, 4) == "0.6667".
inline std::string format_decimal(const Rational& r, int digits) {
  using detail::Int128;
  if (digits < 0 || digits > 18) throw std::invalid_argument("format_decimal digits out of range");
  Int128 scale = 1;
  for (int i = 0; i < digits; ++i) scale *= 10;
  Int128 mag = detail::iabs(Int128(r.numerator()));
  Int128 den = r.denominator();
  Int128 q = (2 * mag * scale + den) / (2 * den);
  std::string out = (r.is_negative() && q != 0) ? "-" : "";
  out += std::to_string(static_cast<long long>(detail::to_i64(q / scale)));
  if (digits > 0) {
    std::string frac = std::to_string(static_cast<long long>(detail::to_i64(q % scale)));
    out += '.';
    out.append(static_cast<std::size_t>(digits) - frac.size(), '0');
    out += frac;
  }
  return out;
}

}  // namespace seqpipe
