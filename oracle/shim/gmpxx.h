// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Minimal stand-in for the GMP C++ interface that the reference's
// `stencilkit::Rational` (proj/include/stencilkit/rational.hpp:4-59,
// proj/src/rational.cpp:10-34) is written against. GMP's headers and
// libgmpxx are absent from this image (only the runtime libgmp.so.10 exists),
// so the reference cannot compile as shipped; this header lets the UNMODIFIED
// reference sources compile so they can serve as the parity oracle.
//
// This is an independent implementation on checked __int128 arithmetic (no
// GMP source is reproduced). It covers exactly the surface the reference
// library uses: mpz_class / mpq_class construction, canonical form, + - * /,
// comparisons, sgn, get_str, get_d, mpz_fac_ui and mpz_pow_ui. Every
// operation throws std::overflow_error instead of wrapping, so a result that
// would need more than ~126 bits fails loudly instead of silently differing
// from GMP. Hot-path rationals are tiny (weights <= 1607/24, products of a
// few small factorials), far inside that range.
//
// get_d() truncates toward zero, as GMP's mpq_get_d does: that is what the
// reference's `Rational::to_double` (rational.hpp:32) yields with real GMP and
// is the value `assemble` multiplies by h^s (grid.cpp:77-81). Integer and
// dyadic weights are exact either way; the non-dyadic 73-point weights differ
// by 1 ulp from round-to-nearest.
#ifndef SK_ORACLE_GMPXX_SHIM_H
#define SK_ORACLE_GMPXX_SHIM_H

#include <climits>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>

namespace sk_shim {

using i128 = __int128;

inline i128 checked_add(i128 a, i128 b) {
  i128 r;
  if (__builtin_add_overflow(a, b, &r)) throw std::overflow_error("gmpxx shim: int128 overflow (add)");
  return r;
}
inline i128 checked_sub(i128 a, i128 b) {
  i128 r;
  if (__builtin_sub_overflow(a, b, &r)) throw std::overflow_error("gmpxx shim: int128 overflow (sub)");
  return r;
}
inline i128 checked_mul(i128 a, i128 b) {
  i128 r;
  if (__builtin_mul_overflow(a, b, &r)) throw std::overflow_error("gmpxx shim: int128 overflow (mul)");
  return r;
}
inline i128 iabs(i128 a) {
  const i128 lowest = static_cast<i128>(static_cast<unsigned __int128>(1) << 127);
  if (a == lowest) throw std::overflow_error("gmpxx shim: int128 overflow (abs)");
  return a < 0 ? -a : a;
}
inline i128 gcd(i128 a, i128 b) {
  a = iabs(a);
  b = iabs(b);
  while (b != 0) {
    i128 t = a % b;
    a = b;
    b = t;
  }
  return a;
}
inline int bitlen(i128 a) {  // a >= 0
  int n = 0;
  while (a > 0) {
    a >>= 1;
    ++n;
  }
  return n;
}
inline std::string to_str(i128 v) {
  if (v == 0) return "0";
  bool neg = v < 0;
  unsigned __int128 u = neg ? (unsigned __int128)(-(v + 1)) + 1 : (unsigned __int128)v;
  std::string s;
  while (u > 0) {
    s.insert(s.begin(), char('0' + int(u % 10)));
    u /= 10;
  }
  return neg ? "-" + s : s;
}
inline i128 parse(const std::string& s) {
  size_t i = 0;
  bool neg = false;
  if (i < s.size() && (s[i] == '-' || s[i] == '+')) neg = s[i++] == '-';
  if (i == s.size()) throw std::invalid_argument("gmpxx shim: not an integer");
  i128 v = 0;
  for (; i < s.size(); ++i) {
    if (s[i] < '0' || s[i] > '9') throw std::invalid_argument("gmpxx shim: not an integer");
    v = checked_add(checked_mul(v, 10), s[i] - '0');
  }
  return neg ? -v : v;
}

// num/den (den > 0) to double, truncated toward zero (mpq_get_d semantics).
inline double trunc_div_to_double(i128 num, i128 den) {
  if (num == 0) return 0.0;
  const bool neg = num < 0;
  i128 n = iabs(num);
  // shift so the integer quotient carries >= 54 significant bits, then drop
  // low bits: floor(floor(x*2^s)/2^j) == floor(x*2^(s-j)), so truncation is exact
  int s = 55 + bitlen(den) - bitlen(n);
  if (s < 0) s = 0;
  if (bitlen(n) + s > 126) throw std::overflow_error("gmpxx shim: get_d range");
  i128 q = (n << s) / den;
  int extra = bitlen(q) - 53;
  if (extra > 0) {
    q >>= extra;
    s -= extra;
  }
  double d = std::ldexp(static_cast<double>(static_cast<std::int64_t>(q)), -s);
  return neg ? -d : d;
}

}  // namespace sk_shim

struct sk_mpz_struct {
  __int128 v;
};
using mpz_ptr = sk_mpz_struct*;
using mpz_srcptr = const sk_mpz_struct*;

class mpz_class {
 public:
  mpz_class() : z_{0} {}
  mpz_class(int v) : z_{v} {}    // NOLINT
  mpz_class(long v) : z_{v} {}   // NOLINT
  mpz_class(long long v) : z_{v} {}  // NOLINT
  mpz_class(unsigned long v) : z_{(__int128)v} {}  // NOLINT
  explicit mpz_class(__int128 v) : z_{v} {}
  explicit mpz_class(const std::string& s) : z_{sk_shim::parse(s)} {}
  explicit mpz_class(const char* s) : z_{sk_shim::parse(s)} {}

  __int128 raw() const { return z_.v; }
  mpz_ptr get_mpz_t() { return &z_; }
  mpz_srcptr get_mpz_t() const { return &z_; }
  std::string get_str(int base = 10) const {
    if (base != 10) throw std::invalid_argument("gmpxx shim: base 10 only");
    return sk_shim::to_str(z_.v);
  }
  bool fits_slong_p() const { return z_.v >= LONG_MIN && z_.v <= LONG_MAX; }
  long get_si() const { return static_cast<long>(z_.v); }
  double get_d() const { return static_cast<double>(z_.v); }

  friend bool operator==(const mpz_class& a, const mpz_class& b) { return a.z_.v == b.z_.v; }
  friend bool operator!=(const mpz_class& a, const mpz_class& b) { return a.z_.v != b.z_.v; }
  friend bool operator<(const mpz_class& a, const mpz_class& b) { return a.z_.v < b.z_.v; }
  friend bool operator>(const mpz_class& a, const mpz_class& b) { return a.z_.v > b.z_.v; }
  friend bool operator==(const mpz_class& a, long b) { return a.z_.v == b; }
  friend bool operator!=(const mpz_class& a, long b) { return a.z_.v != b; }
  friend bool operator==(const mpz_class& a, int b) { return a.z_.v == b; }
  friend bool operator!=(const mpz_class& a, int b) { return a.z_.v != b; }
  friend mpz_class operator*(const mpz_class& a, const mpz_class& b) {
    return mpz_class(sk_shim::checked_mul(a.z_.v, b.z_.v));
  }
  friend mpz_class operator+(const mpz_class& a, const mpz_class& b) {
    return mpz_class(sk_shim::checked_add(a.z_.v, b.z_.v));
  }
  friend mpz_class operator-(const mpz_class& a, const mpz_class& b) {
    return mpz_class(sk_shim::checked_sub(a.z_.v, b.z_.v));
  }
  mpz_class operator-() const { return mpz_class(sk_shim::checked_sub(0, z_.v)); }

 private:
  sk_mpz_struct z_;
};

inline int sgn(const mpz_class& z) { return (z.raw() > 0) - (z.raw() < 0); }

inline void mpz_fac_ui(mpz_ptr r, unsigned long n) {
  __int128 f = 1;
  for (unsigned long k = 2; k <= n; ++k) f = sk_shim::checked_mul(f, (__int128)k);
  r->v = f;
}

inline void mpz_pow_ui(mpz_ptr r, mpz_srcptr b, unsigned long e) {
  __int128 p = 1;
  for (unsigned long k = 0; k < e; ++k) p = sk_shim::checked_mul(p, b->v);
  r->v = p;
}

class mpq_class {
 public:
  mpq_class() : num_(0), den_(1) {}
  mpq_class(int v) : num_(v), den_(1) {}   // NOLINT
  mpq_class(long v) : num_(v), den_(1) {}  // NOLINT
  mpq_class(const mpz_class& n, const mpz_class& d) : num_(n), den_(d) {}

  // Lowest terms, positive denominator.
  void canonicalize() {
    __int128 n = num_.raw(), d = den_.raw();
    if (d == 0) throw std::domain_error("gmpxx shim: zero denominator");
    if (d < 0) {
      n = sk_shim::checked_sub(0, n);
      d = sk_shim::checked_sub(0, d);
    }
    __int128 g = sk_shim::gcd(n, d);
    if (g > 1) {
      n /= g;
      d /= g;
    }
    num_ = mpz_class(n);
    den_ = mpz_class(d);
  }

  const mpz_class& get_num() const { return num_; }
  const mpz_class& get_den() const { return den_; }
  double get_d() const { return sk_shim::trunc_div_to_double(num_.raw(), den_.raw()); }

  friend mpq_class operator+(const mpq_class& a, const mpq_class& b) {
    using namespace sk_shim;
    __int128 g = gcd(a.den_.raw(), b.den_.raw());
    __int128 bd = b.den_.raw() / g;
    __int128 n = checked_add(checked_mul(a.num_.raw(), bd), checked_mul(b.num_.raw(), a.den_.raw() / g));
    return make(n, checked_mul(a.den_.raw(), bd));
  }
  friend mpq_class operator-(const mpq_class& a, const mpq_class& b) { return a + (-b); }
  friend mpq_class operator*(const mpq_class& a, const mpq_class& b) {
    using namespace sk_shim;
    __int128 g1 = gcd(a.num_.raw(), b.den_.raw()), g2 = gcd(b.num_.raw(), a.den_.raw());
    if (g1 == 0) g1 = 1;
    if (g2 == 0) g2 = 1;
    return make(checked_mul(a.num_.raw() / g1, b.num_.raw() / g2),
                checked_mul(a.den_.raw() / g2, b.den_.raw() / g1));
  }
  friend mpq_class operator/(const mpq_class& a, const mpq_class& b) {
    if (b.num_.raw() == 0) throw std::domain_error("gmpxx shim: division by zero");
    return a * mpq_class(b.den_, b.num_).canon();
  }
  mpq_class operator-() const { return mpq_class(-num_, den_); }
  mpq_class& operator+=(const mpq_class& o) { return *this = *this + o; }
  mpq_class& operator-=(const mpq_class& o) { return *this = *this - o; }
  mpq_class& operator*=(const mpq_class& o) { return *this = *this * o; }

  friend bool operator==(const mpq_class& a, const mpq_class& b) {
    return a.num_ == b.num_ && a.den_ == b.den_;
  }
  friend bool operator!=(const mpq_class& a, const mpq_class& b) { return !(a == b); }
  friend bool operator<(const mpq_class& a, const mpq_class& b) {
    using namespace sk_shim;
    return checked_mul(a.num_.raw(), b.den_.raw()) < checked_mul(b.num_.raw(), a.den_.raw());
  }
  friend bool operator>(const mpq_class& a, const mpq_class& b) { return b < a; }
  friend bool operator==(const mpq_class& a, int b) { return a.den_ == 1 && a.num_ == b; }
  friend bool operator!=(const mpq_class& a, int b) { return !(a == b); }

 private:
  static mpq_class make(__int128 n, __int128 d) {
    mpq_class q{mpz_class(n), mpz_class(d)};
    q.canonicalize();
    return q;
  }
  mpq_class canon() const {
    mpq_class q = *this;
    q.canonicalize();
    return q;
  }
  mpz_class num_, den_;
};

inline int sgn(const mpq_class& q) { return sgn(q.get_num()); }

#endif
