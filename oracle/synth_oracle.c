/*
 * TEST INFRASTRUCTURE (oracle/): host restatement of the counter-based
 * synthetic tensor generator, the checker for the device generator
 * (paper_1409_2383_b200/csrc/synth.cu, C ABI ntf_synth_dense) and the source
 * of the tensors the reference is run on by tests/golden/make_golden.py.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU legs load it.
 *
 * The generator stands in for the reference's synthetic protocol
 * (reference bench.py:34-46 and SURVEY 8(d): U[0,1) true factors from a
 * seed, X = [[A,B,C]] + i.i.d. Gaussian noise scaled to an SNR).  Element
 * (i,j,k) of the full I x J x K tensor, e = (i J + j) K + k:
 *   clean = sum_{r=0..R-1} (A[i,r] * B[j,r]) * C[k,r]     (r ascending)
 *   w1, w2 = SplitMix64 outputs 2e+1, 2e+2 of `key`
 *   u1 = ((w1 >> 11) + 1) 2^-53 in (0,1],  u2 = (w2 >> 11) 2^-53 in [0,1)
 *   z = sqrt(-2 ln u1) cos(2 pi u2)
 *   x = clean + sigma * z   (rounded to float for fp32 tensors)
 * ln and cos are fixed polynomials evaluated in IEEE double with separate
 * correctly rounded operations (built with -ffp-contract=off), so the device
 * kernel reproduces every byte.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 *        oracle/synth_oracle.c -o oracle/libsynth_oracle.so -lm
 */
#include <math.h>
#include <stdint.h>

static const uint64_t kGamma = 0x9E3779B97F4A7C15ull;
static const double kSqrt2 = 0x1.6a09e667f3bcdp+0;
static const double kPio2 = 0x1.921fb54442d18p+0;
static const double kLn2Hi = 0x1.62e42fee00000p-1;
static const double kLn2Lo = 0x1.a39ef35793c76p-33;
static const double kLn[12] = {0x1.0000000000000p+0, 0x1.5555555555555p-2, 0x1.999999999999ap-3,
                               0x1.2492492492492p-3, 0x1.c71c71c71c71cp-4, 0x1.745d1745d1746p-4,
                               0x1.3b13b13b13b14p-4, 0x1.1111111111111p-4, 0x1.e1e1e1e1e1e1ep-5,
                               0x1.af286bca1af28p-5, 0x1.8618618618618p-5, 0x1.642c8590b2164p-5};
static const double kCos[11] = {0x1.0000000000000p+0,  -0x1.0000000000000p-1, 0x1.5555555555555p-5,
                                -0x1.6c16c16c16c17p-10, 0x1.a01a01a01a01ap-16, -0x1.27e4fb7789f5cp-22,
                                0x1.1eed8eff8d898p-29,  -0x1.93974a8c07c9dp-37, 0x1.ae7f3e733b81fp-45,
                                -0x1.6827863b97d97p-53, 0x1.e542ba4020225p-62};
static const double kSin[11] = {0x1.0000000000000p+0,  -0x1.5555555555555p-3, 0x1.1111111111111p-7,
                                -0x1.a01a01a01a01ap-13, 0x1.71de3a556c734p-19, -0x1.ae64567f544e4p-26,
                                0x1.6124613a86d09p-33,  -0x1.ae7f3e733b81fp-41, 0x1.952c77030ad4ap-49,
                                -0x1.2f49b46814157p-57, 0x1.71b8ef6dcf572p-66};

static uint64_t splitmix(uint64_t key, uint64_t c) {
  uint64_t z = key + c * kGamma;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double synth_std_normal(uint64_t key, uint64_t e) {
  const uint64_t w1 = splitmix(key, 2 * e + 1);
  const uint64_t w2 = splitmix(key, 2 * e + 2);
  const double u1 = (double)((w1 >> 11) + 1) * 0x1p-53;
  int ex = 0;
  const double mant = frexp(u1, &ex);
  double m = mant * 2.0;
  int E = ex - 1;
  if (m > kSqrt2) {
    m = mant;
    E = ex;
  }
  const double s = (m - 1.0) / (m + 1.0);
  const double s2 = s * s;
  double p = kLn[11];
  for (int k = 10; k >= 0; --k) {
    p = p * s2;
    p = p + kLn[k];
  }
  const double lnm = (2.0 * s) * p;
  const double Ed = (double)E;
  const double t = Ed * kLn2Lo;
  const double ln = Ed * kLn2Hi + (t + lnm);
  const double rad = sqrt(-2.0 * ln);
  const uint64_t n2 = w2 >> 11;
  const int q = (int)(n2 >> 51);
  const uint64_t fi = n2 & ((1ull << 51) - 1);
  const int sw = fi > (1ull << 50);
  const double g = (double)(sw ? (1ull << 51) - fi : fi) * 0x1p-51;
  const double th = g * kPio2;
  const double t2 = th * th;
  double c = kCos[10], sn = kSin[10];
  for (int k = 9; k >= 0; --k) {
    c = c * t2;
    c = c + kCos[k];
    sn = sn * t2;
    sn = sn + kSin[k];
  }
  sn = th * sn;
  const double cq = sw ? sn : c, sq = sw ? c : sn;
  const double v = q == 0 ? cq : (q == 1 ? -sq : (q == 2 ? -cq : sq));
  return rad * v;
}

/* Box [lo, hi) of the full dims tensor, row-major, into out (float if
 * out_f32, else double).  A, B, C: full factors (dims[m] x R, row-major).
 * Returns 0, or -1 for R outside 1..4096. */
int synth_box(const double* A, const double* B, const double* C, const int64_t* dims,
               const int64_t* lo, const int64_t* hi, int R, double sigma, uint64_t key, int out_f32,
               void* out) {
  const int64_t bi = hi[0] - lo[0], bj = hi[1] - lo[1], bk = hi[2] - lo[2];
  const int64_t rows = bi * bj;
  if (R < 1 || R > 4096) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t rr = 0; rr < rows; ++rr) {
    const int64_t i = lo[0] + rr / bj, j = lo[1] + rr % bj;
    double pr[4096];
    for (int r = 0; r < R; ++r) pr[r] = A[i * R + r] * B[j * R + r];
    for (int64_t kk = 0; kk < bk; ++kk) {
      const int64_t k = lo[2] + kk;
      double acc = 0.0;
      for (int r = 0; r < R; ++r) {
        const double t = pr[r] * C[k * R + r];
        acc = acc + t;
      }
      const uint64_t e = (uint64_t)((i * dims[1] + j) * dims[2] + k);
      const double x = acc + sigma * synth_std_normal(key, e);
      if (out_f32)
        ((float*)out)[rr * bk + kk] = (float)x;
      else
        ((double*)out)[rr * bk + kk] = x;
    }
  }
  return 0;
}
