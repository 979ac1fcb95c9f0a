/* Host generator of the BASELINE dechirped-LFM operators -- TEST
 * INFRASTRUCTURE ONLY (bench.py's CPU-baseline / reference legs and tests).
 *
 * The same IEEE operation sequence as scenario.baseline_operator (NumPy) and
 * the device generator dechirp_kernel (kernels_dense.cuh): per entry
 *   tau  = (|tx - p_n| + |rx_m - p_n|) / c
 *   cyc  = (alpha tau) t_k + fc tau,  cyc -= floor(cyc)
 *   t    = cyc + u_n,                 t   -= floor(t)
 *   A    = (cos 2 pi t, sin 2 pi t)   via the portable octant/Taylor sincos
 * with every operation separately rounded (-ffp-contract=off), so all three
 * produce the same complex64 bits (tests/test_oracle_pins.py checks it).
 * Written in C with OpenMP because a config-3 sensor (8192 x 65536 entries)
 * takes minutes in NumPy and ~1 s here.  Output is column-major (pixel
 * columns contiguous), interleaved re/im float32.
 */
#include <math.h>
#include <stdint.h>

static const double kSin[8] = {-0.16666666666666666, 0.008333333333333333, -0.0001984126984126984,
                               2.7557319223985893e-06, -2.505210838544172e-08, 1.6059043836821613e-10,
                               -7.647163731819816e-13, 2.8114572543455206e-15};
static const double kCos[9] = {-0.5, 0.041666666666666664, -0.001388888888888889, 2.48015873015873e-05,
                               -2.755731922398589e-07, 2.08767569878681e-09, -1.1470745597729725e-11,
                               4.779477332387385e-14, -1.5619206968586225e-16};

static void sincos_turns(double t, double* c_out, double* s_out) {
  const double t8 = t * 8.0;
  const double o = floor(t8);
  const double f = t8 - o;
  const int oi = (int)o;
  const double h = (oi & 1) ? 1.0 - f : f;
  const double x = h * 0.7853981633974483;
  const double x2 = x * x;
  double p = kSin[7];
  for (int i = 6; i >= 0; --i) p = kSin[i] + x2 * p;
  const double sx = x + (x * x2) * p;
  double r = kCos[8];
  for (int i = 7; i >= 0; --i) r = kCos[i] + x2 * r;
  const double cx = 1.0 + x2 * r;
  const int sw = ((oi + 1) >> 1) & 1;
  const double sa = sw ? cx : sx, ca = sw ? sx : cx;
  *s_out = (oi >= 4) ? -sa : sa;
  *c_out = (oi >= 2 && oi <= 5) ? -ca : ca;
}

static double dist3(const double* a, const double* p) {
  const double d0 = a[0] - p[0], d1 = a[1] - p[1], d2 = a[2] - p[2];
  return sqrt((d0 * d0 + d1 * d1) + d2 * d2);
}

void baseline_operator_c64(int M, int K, int N, const double* pix, const double* tx, const double* rx,
                           const double* turns, double alpha, double fc, double t_step, double c_light, float* out) {
  const int64_t rows = (int64_t)M * K;
#pragma omp parallel for schedule(static)
  for (int n = 0; n < N; ++n) {
    const double* p = pix + 3 * (int64_t)n;
    const double dtx = dist3(tx, p);
    float* col = out + 2 * rows * (int64_t)n;
    for (int m = 0; m < M; ++m) {
      const double tau = (dtx + dist3(rx + 3 * m, p)) / c_light;
      const double at = alpha * tau, ft = fc * tau;
      for (int k = 0; k < K; ++k) {
        double cyc = at * ((double)k * t_step) + ft;
        cyc = cyc - floor(cyc);
        double t = cyc + turns[n];
        t = t - floor(t);
        double c, s;
        sincos_turns(t, &c, &s);
        col[2 * ((int64_t)m * K + k)] = (float)c;
        col[2 * ((int64_t)m * K + k) + 1] = (float)s;
      }
    }
  }
}
