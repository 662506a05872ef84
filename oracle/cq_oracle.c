/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the B200 backend.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker / the reported CPU baseline.
 *
 * A plain-C restatement of the reference's arithmetic for the BASELINE
 * workloads.  The reference (clusterq, pure Python) evaluates every cell with
 * eval_kernel (pkg/src/clusterq/kernel.py:291-331): depth-first, left to
 * right, one IEEE rounding per operator, reads clamped per axis to the buffer
 * extent (model.py:442-446).  Built with -ffp-contract=off so no operator is
 * fused; float variants round every operator to binary32 (SSE, no excess
 * precision) -- the definition of the new float32 element kind.
 *
 * N-body and matmul are not expressible in the reference DSL;
 * their restatement follows the reference's conventions (float64, fixed
 * left-to-right j / k order) and is "parity unpinned" by the reference.
 */
#include <math.h>
#include <stdint.h>

/* SAXPY body "alpha * x[i] + y[i]" (scenarios/saxpy.json:15). */
void oracle_saxpy_f64(double alpha, const double* x, const double* y, double* z, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double t = alpha * x[i];
    z[i] = t + y[i];
  }
}

void oracle_saxpy_f32(float alpha, const float* x, const float* y, float* z, int64_t n) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    float t = alpha * x[i];
    z[i] = t + y[i];
  }
}

static inline int64_t clampi(int64_t v, int64_t n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); }

/* One wave step over rows [r0, r1) of an H x W grid (SURVEY.md §8c body):
 *   out = ((k2*u) - upr) + (c * ((((uN + uS) + uW) + uE) - (k4*u)))
 * out may alias upr (each cell reads its own upr before writing). */
#define WAVE_BODY(T)                                                                   \
  _Pragma("omp parallel for schedule(static)") for (int64_t i = r0; i < r1; ++i) {     \
    const T* um = u + clampi(i - 1, H) * W;                                             \
    const T* uc = u + i * W;                                                            \
    const T* up = u + clampi(i + 1, H) * W;                                             \
    for (int64_t j = 0; j < W; ++j) {                                                   \
      T a = k2 * uc[j];                                                                 \
      T b = a - upr[i * W + j];                                                         \
      T s = um[j] + up[j];                                                              \
      s = s + uc[clampi(j - 1, W)];                                                     \
      s = s + uc[clampi(j + 1, W)];                                                     \
      T f = k4 * uc[j];                                                                 \
      T l = s - f;                                                                      \
      T g = c * l;                                                                      \
      out[i * W + j] = b + g;                                                           \
    }                                                                                   \
  }

void oracle_wave5_f64(const double* u, const double* upr, double* out, int64_t H, int64_t W,
                      int64_t r0, int64_t r1, double c, double k2, double k4) {
  WAVE_BODY(double)
}

void oracle_wave5_f32(const float* u, const float* upr, float* out, int64_t H, int64_t W,
                      int64_t r0, int64_t r1, float c, float k2, float k4) {
  WAVE_BODY(float)
}

/* N-body kick for bodies [i0, i1): double-precision accumulation over all j
 * in ascending order; pos rows (x, y, z, m) as float, result a_i (float64). */
void oracle_nbody_accel(const float* pos, int64_t n, int64_t i0, int64_t i1, double eps2,
                        double* acc /* [(i1-i0) x 3] */) {
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t i = i0; i < i1; ++i) {
    double px = pos[4 * i], py = pos[4 * i + 1], pz = pos[4 * i + 2];
    double ax = 0, ay = 0, az = 0;
    for (int64_t j = 0; j < n; ++j) {
      double dx = (double)pos[4 * j] - px, dy = (double)pos[4 * j + 1] - py, dz = (double)pos[4 * j + 2] - pz;
      double r2 = dx * dx + dy * dy + dz * dz + eps2;
      double inv = 1.0 / sqrt(r2);
      double s = (double)pos[4 * j + 3] * inv * inv * inv;
      ax += dx * s;
      ay += dy * s;
      az += dz * s;
    }
    acc[3 * (i - i0)] = ax;
    acc[3 * (i - i0) + 1] = ay;
    acc[3 * (i - i0) + 2] = az;
  }
}

/* Same as oracle_nbody_accel for an explicit list of i-bodies. */
void oracle_nbody_accel_idx(const float* pos, int64_t n, const int64_t* idx, int64_t count, double eps2,
                            double* acc) {
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t q = 0; q < count; ++q) {
    int64_t i = idx[q];
    double px = pos[4 * i], py = pos[4 * i + 1], pz = pos[4 * i + 2];
    double ax = 0, ay = 0, az = 0;
    for (int64_t j = 0; j < n; ++j) {
      double dx = (double)pos[4 * j] - px, dy = (double)pos[4 * j + 1] - py, dz = (double)pos[4 * j + 2] - pz;
      double r2 = dx * dx + dy * dy + dz * dz + eps2;
      double inv = 1.0 / sqrt(r2);
      double s = (double)pos[4 * j + 3] * inv * inv * inv;
      ax += dx * s;
      ay += dy * s;
      az += dz * s;
    }
    acc[3 * q] = ax;
    acc[3 * q + 1] = ay;
    acc[3 * q + 2] = az;
  }
}

/* C rows: c[r, :] = sum_k a[r, k] * b[k, :] in float64, k ascending; also
 * returns sum_k |a[r,k]| |b[k,:]| for the normalised error metric (cabs may be
 * NULL). */
void oracle_sgemm_rows(const float* a, const float* b, int64_t n, int64_t k, const int64_t* rows,
                       int64_t nrows, double* c, double* cabs) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nrows; ++q) {
    const float* ar = a + rows[q] * k;
    double* cr = c + q * n;
    double* ca = cabs ? cabs + q * n : 0;
    for (int64_t j = 0; j < n; ++j) {
      cr[j] = 0;
      if (ca) ca[j] = 0;
    }
    for (int64_t kk = 0; kk < k; ++kk) {
      double av = ar[kk];
      const float* br = b + kk * n;
      if (ca) {
        for (int64_t j = 0; j < n; ++j) {
          cr[j] += av * (double)br[j];
          ca[j] += fabs(av * (double)br[j]);
        }
      } else {  /* cabs == NULL: C rows only (bench.py's CPU timing) */
        for (int64_t j = 0; j < n; ++j) cr[j] += av * (double)br[j];
      }
    }
  }
}
