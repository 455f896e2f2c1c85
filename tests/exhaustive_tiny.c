/*
 * exhaustive_tiny.c -- AC1 (SURVEY 8(c) "what pins each part"):
 * every permutation of n <= 9 distinct keys and every {0,1}-array of n <= 16,
 * under several minruns, through all four oracle variants, checked against
 * the plain definition of the stable sort for these inputs:
 *   - a permutation of 0..n-1 sorts to 0..n-1, and the payload at output
 *     position v is the input position of v (the inverse permutation);
 *   - a {0,1}-array sorts stably to the input positions of its zeros, in
 *     order, followed by those of its ones (stable partition).
 * Plus, per input: every variant reports the same plan (Alg. 1 is the policy
 * of all of them), comparisons of A, B and C0 are equal (all merge left to
 * right), every variant writes exactly M merge outputs (reading R8), C's
 * staging is <= n and its moves <= C0's, and the moves of B and
 * C agree up to 3n (abstract).
 *
 * Test code (tests/ may link the oracle); compiled and run by
 * tests/test_oracle.py::test_exhaustive_tiny_c.  Prints one summary line,
 * exits non-zero on the first failure.
 */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle/vmps_oracle.h"

#define NV 4
static const int VARIANTS[NV] = {ORC_VARIANT_COPYMERGE, ORC_VARIANT_VM, ORC_VARIANT_PINGPONG,
                                 ORC_VARIANT_PINGPONG_PLAIN};
static long n_cases = 0;

static int fail(const char* what, const uint32_t* keys, int n, int mr, int var) {
  fprintf(stderr, "FAIL %s n=%d minrun=%d variant=%d keys:", what, n, mr, var);
  for (int i = 0; i < n; ++i) fprintf(stderr, " %u", keys[i]);
  fprintf(stderr, "\n");
  return 1;
}

/* expected payload order, computed from the input by the definition */
static int check_one(const uint32_t* keys, int n, int mr, const uint32_t* exp_keys, const uint32_t* exp_vals) {
  uint64_t rs[NV][20];
  uint8_t rk[NV][20];
  orc_merge_t mg[NV][20];
  orc_stats_t st[NV];
  for (int v = 0; v < NV; ++v) {
    uint32_t k[20], val[20];
    memcpy(k, keys, n * sizeof(uint32_t));
    for (int i = 0; i < n; ++i) val[i] = (uint32_t)i;
    int rc = orc_sort(ORC_U32, k, val, (uint64_t)n, VARIANTS[v], (uint32_t)mr, rs[v], rk[v], 20, mg[v], &st[v]);
    if (rc) return fail("rc", keys, n, mr, v);
    for (int i = 0; i < n; ++i)
      if (k[i] != exp_keys[i] || val[i] != exp_vals[i]) return fail("output", keys, n, mr, v);
    if (n >= 1 && st[v].moves_merge_out != st[v].merge_cost_M) return fail("writes != M", keys, n, mr, v);
  }
  for (int v = 1; v < NV; ++v) {
    if (st[v].runs != st[0].runs || st[v].merges != st[0].merges) return fail("plan size", keys, n, mr, v);
    if (memcmp(rs[v], rs[0], st[0].runs * 8) || memcmp(rk[v], rk[0], st[0].runs))
      return fail("runs", keys, n, mr, v);
    for (uint64_t m = 0; m < st[0].merges; ++m)
      if (mg[v][m].i != mg[0][m].i || mg[v][m].j != mg[0][m].j || mg[v][m].k != mg[0][m].k ||
          mg[v][m].power != mg[0][m].power)
        return fail("merges", keys, n, mr, v);
  }
  /* A = 0, B = 1, C = 2, C0 = 3 */
  if (st[0].comp_merge != st[1].comp_merge || st[0].comp_merge != st[3].comp_merge)
    return fail("comparisons A/B/C0", keys, n, mr, 0);
  if (st[2].moves_staging > (uint64_t)n) return fail("C staging > n", keys, n, mr, 2);
  uint64_t mB = st[1].moves_merge_out + st[1].moves_staging + st[1].moves_copy;
  uint64_t mC = st[2].moves_merge_out + st[2].moves_staging;
  uint64_t mC0 = st[3].moves_merge_out + st[3].moves_staging;
  if (mC > mC0) return fail("C moves > C0 moves", keys, n, mr, 2);
  if ((mB > mC ? mB - mC : mC - mB) > 3ull * (uint64_t)n) return fail("|moves B - C| > 3n", keys, n, mr, 2);
  ++n_cases;
  return 0;
}

static int next_perm(uint32_t* a, int n) {
  int i = n - 2;
  while (i >= 0 && a[i] >= a[i + 1]) --i;
  if (i < 0) return 0;
  int j = n - 1;
  while (a[j] <= a[i]) --j;
  uint32_t t = a[i]; a[i] = a[j]; a[j] = t;
  for (int l = i + 1, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
  return 1;
}

int main(int argc, char** argv) {
  int maxp = argc > 1 ? atoi(argv[1]) : 9;
  int maxb = argc > 2 ? atoi(argv[2]) : 16;
  const int mrs[4] = {1, 2, 3, 0};
  long perms = 0, bins = 0;
  for (int n = 0; n <= maxp; ++n) {
    for (int q = 0; q < 4; ++q) {
      uint32_t a[20], ek[20], ev[20];
      for (int i = 0; i < n; ++i) a[i] = (uint32_t)i;
      do {
        for (int i = 0; i < n; ++i) { ek[i] = (uint32_t)i; ev[a[i]] = (uint32_t)i; }
        if (check_one(a, n, mrs[q], ek, ev)) return 1;
        ++perms;
      } while (n > 0 && next_perm(a, n));
    }
  }
  for (int n = 0; n <= maxb; ++n) {
    for (int q = 0; q < 3; ++q) {
      const int mr = q == 2 ? 0 : q + 1;
      for (uint32_t bits = 0; bits < (1u << n); ++bits) {
        uint32_t a[20], ek[20], ev[20];
        int z = 0;
        for (int i = 0; i < n; ++i) a[i] = (bits >> i) & 1u;
        for (int i = 0; i < n; ++i) if (!a[i]) { ek[z] = 0; ev[z++] = (uint32_t)i; }
        for (int i = 0; i < n; ++i) if (a[i]) { ek[z] = 1; ev[z++] = (uint32_t)i; }
        if (check_one(a, n, mr, ek, ev)) return 1;
        ++bins;
      }
    }
  }
  printf("ok permutations(n<=%d)=%ld binary(n<=%d)=%ld cases=%ld\n", maxp, perms, maxb, bins, n_cases);
  return 0;
}
