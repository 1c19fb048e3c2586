// TEST INFRASTRUCTURE — checks paper_2501_10714_b200/csrc/glibc_libm.cuh
// (the device restatement of glibc's __log_fma / __exp_fma / __log1p_fma /
// __cos_fma) against the live libm of this host, bit for bit.
// Built by tests/test_glibc_libm.py with -O2 -ffp-contract=off -fno-builtin.
// Usage: glibc_libm_check N seed  -> one line per function: "name tested mismatches"
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "glibc_libm.cuh"

using namespace fsmoe_libm;

static uint64_t bits(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}
static double from(uint64_t u) {
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
static bool same(double a, double b) {
  if (std::isnan(a) && std::isnan(b)) return true;
  return bits(a) == bits(b);
}

struct Tally {
  const char* name;
  long long n = 0, bad = 0;
  double first_x = 0;
  void check(double x, double want, double got) {
    ++n;
    if (!same(want, got)) {
      if (!bad) first_x = x;
      ++bad;
    }
  }
  void print() const {
    std::printf("%s %lld %lld %a\n", name, n, bad, first_x);
  }
};

int main(int argc, char** argv) {
  const long long N = argc > 1 ? std::atoll(argv[1]) : 1000000;
  std::mt19937_64 g(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1);
  auto u53 = [&]() { return (static_cast<double>(g() >> 11) + 0.5) * 0x1.0p-53; };  // workload.cpp:91
  auto uni = [&](double lo, double hi) { return lo + (hi - lo) * (static_cast<double>(g() >> 11) * 0x1.0p-53); };
  Tally tl{"log"}, te{"exp"}, t1{"log1p"}, tc{"cos"}, tn{"normal"}, ts{"softplus"};
  const double two_pi = 2.0 * 3.141592653589793238462643383279502884;
  for (long long i = 0; i < N; ++i) {
    // log: the gate's u1 domain, the near-1 window, arbitrary positive bit patterns
    double u1 = u53();
    tl.check(u1, std::log(u1), gl_log(u1));
    double xn = uni(0.9, 1.1);
    tl.check(xn, std::log(xn), gl_log(xn));
    double xb = from(g() & 0x7fffffffffffffffULL);
    tl.check(xb, std::log(xb), gl_log(xb));
    // cos: the gate's 2 pi u2 domain and wider ranges (every reduction branch)
    double u2 = u53();
    double a = two_pi * u2;
    tc.check(a, std::cos(a), gl_cos(a));
    double w = uni(-1e6, 1e6);
    tc.check(w, std::cos(w), gl_cos(w));
    double v = uni(-4.0, 4.0);
    tc.check(v, std::cos(v), gl_cos(v));
    double t = std::ldexp(uni(1.0, 2.0), static_cast<int>(g() % 60) - 40);
    tc.check(t, std::cos(t), gl_cos(t));
    // exp / log1p / softplus: logits-scale arguments and the full finite range
    double z = uni(-40.0, 40.0);
    te.check(z, std::exp(z), gl_exp(z));
    double zz = uni(-745.0, 710.0);
    te.check(zz, std::exp(zz), gl_exp(zz));
    double zt = std::ldexp(uni(-1.0, 1.0), -static_cast<int>(g() % 80));
    te.check(zt, std::exp(zt), gl_exp(zt));
    double e = std::exp(z);
    t1.check(e, std::log1p(e), gl_log1p(e));
    double q = uni(-0.999, 3.0);
    t1.check(q, std::log1p(q), gl_log1p(q));
    double qb = from(g() & 0x7fffffffffffffffULL);
    t1.check(qb, std::log1p(qb), gl_log1p(qb));
    double qs = std::ldexp(uni(-1.0, 1.0), -static_cast<int>(g() % 70));
    t1.check(qs, std::log1p(qs), gl_log1p(qs));
    ts.check(z, std::log1p(std::exp(z)), gl_softplus(z));
    // one normal draw exactly as workload.cpp:90-95
    double n_ref = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.141592653589793238462643383279502884 * u2);
    tn.check(u1, n_ref, gl_normal(u1, u2));
  }
  // edge arguments
  const double edges[] = {0.0, -0.0, 1.0, -1.0, 0x1p-1074, 0x1p-1022, 0x1.fffffffffffffp-1, 0x1.0000000000001p0,
                          0.9375, 1.0644531249999998, 0x1p-27, 0x1p-28, 0.855469, 2.426265, 708.0, 709.78,
                          -708.0, -745.0, 512.0, -512.0, 1e-300, 1e300, INFINITY, -INFINITY, NAN};
  for (double x : edges) {
    tl.check(x, std::log(x), gl_log(x));
    te.check(x, std::exp(x), gl_exp(x));
    t1.check(x, std::log1p(x), gl_log1p(x));
    if (!(std::fabs(x) >= 105414350.0)) tc.check(x, std::cos(x), gl_cos(x));  // gl_cos's domain
  }
  tl.print();
  te.print();
  t1.print();
  tc.print();
  tn.print();
  ts.print();
  return 0;
}
