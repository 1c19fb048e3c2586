/* TEST INFRASTRUCTURE — the host libm (glibc) over arrays, multi-threaded,
 * for the device libm audit (tests/test_noise_exact_gpu.py). fn as
 * fsmoe_libm_eval: 0 log, 1 exp, 2 log1p, 3 cos, 4 normal draw, 5 softplus.
 * The normal draw and softplus are written exactly as the reference
 * (proj/src/workload.cpp:90-101). Built with -O2 -ffp-contract=off
 * -fno-builtin. */
#include <math.h>
#include <pthread.h>

typedef struct {
  int fn;
  const double *x, *x2;
  double* y;
  long lo, hi;
} job_t;

static void* run(void* p) {
  job_t* j = (job_t*)p;
  for (long i = j->lo; i < j->hi; ++i) {
    double a = j->x[i], r;
    switch (j->fn) {
      case 0: r = log(a); break;
      case 1: r = exp(a); break;
      case 2: r = log1p(a); break;
      case 3: r = cos(a); break;
      case 4: r = sqrt(-2.0 * log(a)) * cos(2.0 * 3.141592653589793238462643383279502884 * j->x2[i]); break;
      default: r = log1p(exp(a)); break;
    }
    j->y[i] = r;
  }
  return 0;
}

void host_libm_eval(int fn, const double* x, const double* x2, double* y, long n, int threads) {
  if (threads < 1) threads = 1;
  if (threads > 64) threads = 64;
  pthread_t th[64];
  job_t jb[64];
  for (int t = 0; t < threads; ++t) {
    jb[t].fn = fn;
    jb[t].x = x;
    jb[t].x2 = x2;
    jb[t].y = y;
    jb[t].lo = n * t / threads;
    jb[t].hi = n * (t + 1) / threads;
    pthread_create(&th[t], 0, run, &jb[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], 0);
}
