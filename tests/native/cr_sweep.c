/*
 * TEST HELPER (not product code): exhaustive correct-rounding sweep of the
 * ORACLE's f32 EXP and LOG (SURVEY §8(c) "EXP/LOG" pin; R6).
 *
 * For every f32 bit pattern in [lo, hi) the oracle's eager evaluation of the
 * one-instruction programs [LOAD0 EXP] / [LOAD0 LOG] (orc_eval, linked from
 * oracle/liboracle.so) is compared with the reference (float)expq(x) /
 * (float)logq(x) computed here in binary128 (libquadmath): 113 significand
 * bits, so rounding the quad value once more to binary32 is innocuous
 * (113 >= 2*24 + 2) unless exp/log(x) lies within 2^-112 relative of an f32
 * rounding midpoint, far closer than any f32 worst case.  NaN must pair with
 * NaN; everything else (infinities, zeros incl. sign, subnormals) bit-exact.
 * Shares no code with the oracle: it only calls its public entry point.
 *
 * Mode "quad" evaluates every reference in binary128.  Mode "filtered" first
 * evaluates expl / logl in x87 long double (64-bit significand; glibc's error
 * bound is a few ulp = ~2^-62 relative) and falls back to binary128 wherever
 * that value lies within 2^-50 relative of an f32 rounding midpoint or near
 * the ends of the f32 range (NaN, exact 0 / inf and values far outside the
 * range are decided directly): outside that band the long double value and the
 * exact value round to the same f32, so both modes decide every input the
 * same way; "filtered" is ~50x faster and runs in the default CPU suite.
 *
 * usage: cr_sweep EXP|LOG quad|filtered lo hi threads [stride]
 *   (stride s > 1: only the patterns lo, lo + s, lo + 2s, ... < hi)
 *   -> prints "checked N mismatches M quad_fallbacks Q" and up to 10
 *      mismatching inputs.
 */
#include <pthread.h>
#include <math.h>
#include <quadmath.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

int orc_eval(int type, uint64_t n, const void* const* operands, int n_operands,
             const void* scalars, int n_scalars, const int* ops, const int* args, int n_instr,
             void* out);

enum { F32 = 0, LOAD = 0, EXP = 6, LOG = 7 };
#define CHUNK (1u << 20)

static int g_op, g_quad;
static uint64_t g_lo, g_hi, g_stride = 1;
static uint64_t g_next;
static pthread_mutex_t g_mu = PTHREAD_MUTEX_INITIALIZER;
static uint64_t g_checked, g_bad, g_fallback;
static uint32_t g_first[10];

static float f_of(uint32_t b) { float f; memcpy(&f, &b, 4); return f; }
static uint32_t b_of(float f) { uint32_t b; memcpy(&b, &f, 4); return b; }

/* f32 rounding of the value v (given to ~2^-62 relative): returns 1 and the
 * rounded value if v is clear of every f32 rounding midpoint by 2^-50 |v|. */
static int clear_of_midpoint(long double v, float* out) {
  const long double a = v < 0 ? -v : v;
  if (v != v || a == 0 || a == (long double)INFINITY) {
    /* NaN (NaN input, log of a negative), exact zero (log(1); an exp whose
     * long double value underflowed to 0 is below 2^-16000: f32 +0), exact
     * infinities (exp(+inf), log(+inf), log(+-0)) */
    *out = (float)v;
    return 1;
  }
  if (a > 0x1.000001p128L) { *out = v < 0 ? -INFINITY : INFINITY; return 1; }  /* > 2^128: inf */
  if (a < 0x1.fffffep-151L) { *out = v < 0 ? -0.0f : 0.0f; return 1; }       /* < 2^-150: 0 */
  if (a > 0x1.fffffcp127L || a < 0x1.000002p-150L) return 0;  /* near the range ends */
  const float r = (float)v;
  const float up = nextafterf(r, INFINITY), dn = nextafterf(r, -INFINITY);
  const long double band = a * 0x1p-50L;
  const long double m1 = ((long double)r + (long double)up) / 2;  /* exact in x87 */
  const long double m2 = ((long double)r + (long double)dn) / 2;
  const long double d1 = v - m1 < 0 ? m1 - v : v - m1;
  const long double d2 = v - m2 < 0 ? m2 - v : v - m2;
  if (d1 <= band || d2 <= band) return 0;
  *out = r;
  return 1;
}

static void* worker(void* unused) {
  (void)unused;
  float* x = malloc(CHUNK * sizeof(float));
  float* y = malloc(CHUNK * sizeof(float));
  int ops[2] = {LOAD, g_op}, args[2] = {0, 0};
  for (;;) {
    pthread_mutex_lock(&g_mu);
    uint64_t b = g_next;
    g_next += CHUNK;
    pthread_mutex_unlock(&g_mu);
    if (b >= g_hi) break;
    /* this chunk: indices b .. e-1 of the sequence lo + k * stride */
    uint64_t e = b + CHUNK < g_hi ? b + CHUNK : g_hi;
    uint64_t n = e - b;
    for (uint64_t i = 0; i < n; ++i) x[i] = f_of((uint32_t)(g_lo + (b + i) * g_stride));
    const void* opnd[1] = {x};
    if (orc_eval(F32, n, opnd, 1, NULL, 0, ops, args, 2, y) != 0) {
      fprintf(stderr, "orc_eval failed\n");
      exit(2);
    }
    uint64_t bad = 0, fb = 0;
    uint32_t first[10];
    for (uint64_t i = 0; i < n; ++i) {
      float want;
      if (g_quad || !clear_of_midpoint(g_op == EXP ? expl((long double)x[i])
                                                   : logl((long double)x[i]), &want)) {
        __float128 q = (__float128)x[i];
        want = (float)(g_op == EXP ? expq(q) : logq(q));
        ++fb;
      }
      int ok = (want != want) ? (y[i] != y[i]) : (b_of(want) == b_of(y[i]));
      if (!ok) {
        if (bad < 10) first[bad] = b_of(x[i]);
        ++bad;
      }
    }
    pthread_mutex_lock(&g_mu);
    for (uint64_t k = 0; k < bad && g_bad + k < 10; ++k) g_first[g_bad + k] = first[k];
    g_bad += bad;
    g_fallback += fb;
    g_checked += n;
    pthread_mutex_unlock(&g_mu);
  }
  free(x);
  free(y);
  return NULL;
}

int main(int argc, char** argv) {
  if (argc != 6 && argc != 7) {
    fprintf(stderr, "usage: %s EXP|LOG quad|filtered lo hi threads\n", argv[0]);
    return 2;
  }
  g_op = strcmp(argv[1], "EXP") == 0 ? EXP : LOG;
  g_quad = strcmp(argv[2], "quad") == 0;
  g_lo = strtoull(argv[3], NULL, 0);
  if (argc == 7) g_stride = strtoull(argv[6], NULL, 0);
  if (g_stride == 0) g_stride = 1;
  /* the worker walks sequence positions [0, count) */
  g_hi = (strtoull(argv[4], NULL, 0) - g_lo + g_stride - 1) / g_stride;
  g_next = 0;
  int T = atoi(argv[5]);
  if (T < 1) T = 1;
  pthread_t th[256];
  for (int t = 0; t < T && t < 256; ++t) pthread_create(&th[t], NULL, worker, NULL);
  for (int t = 0; t < T && t < 256; ++t) pthread_join(th[t], NULL);
  printf("checked %llu mismatches %llu quad_fallbacks %llu", (unsigned long long)g_checked,
         (unsigned long long)g_bad, (unsigned long long)g_fallback);
  for (uint64_t k = 0; k < g_bad && k < 10; ++k) printf(" 0x%08x", g_first[k]);
  printf("\n");
  return 0;
}
