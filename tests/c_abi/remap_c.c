/* The C-ABI used from plain C (C99), the way a non-Python binding would: device fields, a
 * stencil from host arrays (an InterpolationWeights built elsewhere, interp.py:120-133),
 * sg_remap_apply (apply_remap, interp.py:206-228) and the host-buffer execute in gather mode,
 * checked bitwise against the reference's expression evaluated here in C
 * ((w0*a + w1*b) + w2*c, every op rounded: compile with -ffp-contract=off).  Then the N>1
 * entry points on a 2-rank toy decomposition emulated on one GPU (one launch over both ranks):
 * halo plans, signal words, the signalled exchange (halo_exchange, functionspace.py:107-118)
 * and the fused exchange + apply step (cli.py:138-144).  Then the error conventions:
 * ShapeMismatch as a domain error with the class-name prefix, invalid handle, double release,
 * and no leaked handles.  Exit code 0 = pass; prints the first failure. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "spheregrid_b200.h"

#define CHECK(cond, ...)                \
  do {                                  \
    if (!(cond)) {                      \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);     \
      fprintf(stderr, "\n");            \
      return 1;                         \
    }                                   \
  } while (0)
#define OK(call)                                                           \
  do {                                                                     \
    int32_t _s = (call);                                                   \
    if (_s != SG_OK) {                                                     \
      char _m[512];                                                        \
      sg_last_error(_m, sizeof _m);                                        \
      fprintf(stderr, "FAIL %s:%d: %s -> %d (%s)\n", __FILE__, __LINE__, #call, _s, _m); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static uint64_t next(void) {
  rng ^= rng << 13;
  rng ^= rng >> 7;
  rng ^= rng << 17;
  return rng;
}
static double unif(void) { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }

int main(void) {
  const int64_t n = 50000, m = 20000;
  const int32_t L = 137;
  int32_t ndev = 0;
  OK(sg_device_count(&ndev));
  CHECK(ndev >= 1, "no CUDA device");
  int64_t live0 = 0;
  OK(sg_registry_count(&live0));

  int64_t* nodes = malloc(sizeof(int64_t) * 3 * m);
  double* w = malloc(sizeof(double) * 3 * m);
  for (int64_t t = 0; t < m; ++t) {
    const int64_t base = (int64_t)(unif() * (n - 3000));
    nodes[3 * t] = base;
    nodes[3 * t + 1] = base + 1 + (int64_t)(unif() * 5);
    nodes[3 * t + 2] = base + 2000 + (int64_t)(unif() * 900);
    double a = unif(), b = unif(), c = unif(), s = (a + b) + c;
    w[3 * t] = a / s, w[3 * t + 1] = b / s, w[3 * t + 2] = c / s;
  }
  uint64_t src_h = 0, dst_h = 0;
  OK(sg_host_alloc(sizeof(double) * n * L, &src_h));
  OK(sg_host_alloc(sizeof(double) * m * L, &dst_h));
  double* src = (double*)(uintptr_t)src_h;
  double* dst = (double*)(uintptr_t)dst_h;
  for (int64_t i = 0; i < n * L; ++i) src[i] = unif() * 2.0 - 1.0;
  double* expect = malloc(sizeof(double) * m * L);
  for (int64_t t = 0; t < m; ++t)
    for (int32_t l = 0; l < L; ++l) {
      const double p0 = w[3 * t] * src[nodes[3 * t] * L + l];
      const double p1 = w[3 * t + 1] * src[nodes[3 * t + 1] * L + l];
      const double p2 = w[3 * t + 2] * src[nodes[3 * t + 2] * L + l];
      expect[t * L + l] = (p0 + p1) + p2;
    }

  uint64_t st = 0, fs = 0, ft = 0, fbad = 0;
  int64_t pitch = 0;
  OK(sg_stencil_create(0, nodes, w, m, n, &st));
  OK(sg_field_alloc(0, n, L, 8, &fs, &pitch, NULL));
  CHECK(pitch == L, "dense rows expected, pitch %lld", (long long)pitch);
  OK(sg_field_alloc(0, m, L, 8, &ft, NULL, NULL));
  OK(sg_field_h2d(fs, src, 0));
  OK(sg_remap_apply(st, &fs, &ft, 1, 0, 0));
  memset(dst, 0, sizeof(double) * m * L);
  OK(sg_field_d2h(ft, dst, 0));
  OK(sg_stream_synchronize(0, 0));
  CHECK(memcmp(dst, expect, sizeof(double) * m * L) == 0, "sg_remap_apply differs from the C expression");

  /* host buffers in / out, GPU gather of referenced rows (flags bit 2) */
  memset(dst, 0, sizeof(double) * m * L);
  int64_t moved = 0;
  OK(sg_remap_execute_host(st, &fs, &ft, 1, &src_h, &dst_h, 7, 0, 4, &moved));
  CHECK(memcmp(dst, expect, sizeof(double) * m * L) == 0, "gather execute differs");
  CHECK(moved > 0 && moved <= n, "rows moved %lld", (long long)moved);

  /* ---- N>1: two ranks of a banded toy decomposition on device 0 -------------------------
   * rank r owns global rows [r*no, (r+1)*no) as local rows [0, no); its ng ghosts are local rows
   * [no, no+ng): rank 0's are global [no, no+ng) (rank 1's first rows), rank 1's are global
   * [no-ng, no) (rank 0's last rows). */
  {
    enum { no = 3000, ng = 400, mr = 2500 };
    const int64_t nl = no + ng;
    double* gv = malloc(sizeof(double) * 2 * no * L);
    for (int64_t i = 0; i < 2 * no * L; ++i) gv[i] = unif() * 2.0 - 1.0;
    uint64_t plan[2], fsrc[2], fx[2], fdst[2], sig[2], stn[2], step[2], xch[2];
    uint64_t fptr[2], xptr[2], sptr[2];
    int64_t* rn = malloc(sizeof(int64_t) * 3 * mr);
    double* rw = malloc(sizeof(double) * 3 * mr);
    double* init = malloc(sizeof(double) * nl * L);
    double* got = malloc(sizeof(double) * nl * L);
    double* rexp = malloc(sizeof(double) * 2 * mr * L);
    for (int r = 0; r < 2; ++r) {
      /* global row of local row i */
#define GROW(r, i) ((i) < no ? (int64_t)(r) * no + (i) : ((r) == 0 ? no + ((i) - no) : no - ng + ((i) - no)))
      const int32_t peer = 1 - r;
      const int64_t sc = ng, rc = ng;
      int64_t* srows = malloc(sizeof(int64_t) * ng);
      int64_t* rrows = malloc(sizeof(int64_t) * ng);
      int64_t* rrem = malloc(sizeof(int64_t) * ng);
      for (int64_t j = 0; j < ng; ++j) {
        srows[j] = r == 0 ? no - ng + j : j; /* the peer's ghosts, in its order */
        rrows[j] = no + j;
        rrem[j] = r == 0 ? j : no - ng + j; /* owner row of my ghost j */
      }
      OK(sg_halo_plan_create(0, nl, 1, &peer, &sc, srows, &rc, rrows, rrem, &plan[r]));
      free(srows), free(rrows), free(rrem);
      OK(sg_field_alloc(0, nl, L, 8, &fsrc[r], NULL, &fptr[r]));
      OK(sg_field_alloc(0, nl, L, 8, &fx[r], NULL, &xptr[r]));
      OK(sg_field_alloc(0, mr, L, 8, &fdst[r], NULL, NULL));
      for (int64_t i = 0; i < nl; ++i)
        for (int32_t l = 0; l < L; ++l) init[i * L + l] = i < no ? gv[GROW(r, i) * L + l] : 0.0;
      OK(sg_field_h2d(fsrc[r], init, 0));
      OK(sg_field_h2d(fx[r], init, 0));
      for (int64_t t = 0; t < mr; ++t) { /* a third of the targets read a ghost row */
        const int64_t a = (int64_t)(unif() * (no - 1));
        rn[3 * t] = a;
        rn[3 * t + 1] = a + 1;
        rn[3 * t + 2] = t % 3 == 0 ? no + (int64_t)(unif() * ng) : (int64_t)(unif() * no);
        double x = unif(), y = unif(), z = unif(), q = (x + y) + z;
        rw[3 * t] = x / q, rw[3 * t + 1] = y / q, rw[3 * t + 2] = z / q;
        for (int32_t l = 0; l < L; ++l) {
          const double p0 = rw[3 * t] * gv[GROW(r, rn[3 * t]) * L + l];
          const double p1 = rw[3 * t + 1] * gv[GROW(r, rn[3 * t + 1]) * L + l];
          const double p2 = rw[3 * t + 2] * gv[GROW(r, rn[3 * t + 2]) * L + l];
          rexp[((int64_t)r * mr + t) * L + l] = (p0 + p1) + p2;
        }
      }
      OK(sg_stencil_create(0, rn, rw, mr, nl, &stn[r]));
      OK(sg_signal_create(0, 2, r, &sig[r]));
      OK(sg_signal_ptr(sig[r], &sptr[r]));
    }
    for (int r = 0; r < 2; ++r) {
      const int64_t pitch_l = L;
      OK(sg_exchange_create(plan[r], fx[r], sig[r], &xptr[1 - r], &pitch_l, &sptr[1 - r], &xch[r]));
      OK(sg_step_create(stn[r], plan[r], fsrc[r], fdst[r], sig[r], &fptr[1 - r], &pitch_l, &sptr[1 - r], &step[r]));
    }
    CHECK(sg_exchange_launch(xch, 2, 1, 0) == SG_INVALID_ARGUMENT, "a 2-rank launch on one GPU may not wait");
    OK(sg_exchange_launch(xch, 2, 0, 0));
    OK(sg_step_launch(step, 2, 0, 0));
    OK(sg_stream_synchronize(0, 0));
    for (int r = 0; r < 2; ++r) {
      OK(sg_field_d2h(fx[r], got, 0));
      OK(sg_stream_synchronize(0, 0));
      for (int64_t i = 0; i < nl; ++i)
        CHECK(memcmp(got + i * L, gv + GROW(r, i) * L, sizeof(double) * L) == 0, "rank %d row %lld after exchange",
              r, (long long)i);
      OK(sg_field_d2h(fdst[r], got, 0));
      OK(sg_stream_synchronize(0, 0));
      CHECK(memcmp(got, rexp + (int64_t)r * mr * L, sizeof(double) * mr * L) == 0, "rank %d fused step differs", r);
      uint64_t err = 9, epoch = 0;
      OK(sg_step_check(step[r], &err, &epoch));
      /* the exchange and the step share the rank's signal: two epochs */
      CHECK(err == 0 && epoch == 2, "rank %d signal words: error %llu epoch %llu", r, (unsigned long long)err,
            (unsigned long long)epoch);
    }
#undef GROW
    for (int r = 0; r < 2; ++r) {
      OK(sg_release(step[r]));
      OK(sg_release(xch[r]));
      OK(sg_release(sig[r]));
      OK(sg_release(stn[r]));
      OK(sg_release(plan[r]));
      OK(sg_release(fsrc[r]));
      OK(sg_release(fx[r]));
      OK(sg_release(fdst[r]));
    }
    free(gv), free(rn), free(rw), free(init), free(got), free(rexp);
  }

  /* ShapeMismatch: a target field with the wrong number of points (interp.py:208-217) */
  OK(sg_field_alloc(0, m + 1, L, 8, &fbad, NULL, NULL));
  int32_t s = sg_remap_apply(st, &fs, &fbad, 1, 0, 0);
  char msg[512];
  sg_last_error(msg, sizeof msg);
  CHECK(s == SG_DOMAIN_ERROR && strncmp(msg, "ShapeMismatch", 13) == 0, "status %d msg '%s'", s, msg);

  /* invalid handle, double release, leak probe */
  CHECK(sg_remap_apply(123456789, &fs, &ft, 1, 0, 0) == SG_INVALID_HANDLE, "bogus stencil handle accepted");
  OK(sg_release(fbad));
  CHECK(sg_release(fbad) == SG_INVALID_HANDLE, "double release accepted");
  OK(sg_release(st));
  OK(sg_release(fs));
  OK(sg_release(ft));
  int64_t live1 = 0;
  OK(sg_registry_count(&live1));
  CHECK(live1 == live0, "leaked handles: %lld -> %lld", (long long)live0, (long long)live1);
  OK(sg_host_free(src_h));
  OK(sg_host_free(dst_h));
  free(nodes), free(w), free(expect);
  printf("c-abi ok: %lld targets x %d levels, %lld source rows moved by the gather; 2-rank signalled "
         "exchange + fused step\n", (long long)m, L, (long long)moved);
  return 0;
}
