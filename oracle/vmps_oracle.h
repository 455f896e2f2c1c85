/*
 * vmps_oracle.h -- plain, slow, single-threaded CPU oracle of Powersort
 * (arXiv 2605.27147, Alg. 1 "Abstract Powersort").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2605_27147_b200/, libvmps.so) never links,
 * imports or calls anything here, and shares no code with it.
 *
 * Every function cites the passage it follows; see vmps_oracle.c.
 */
#ifndef VMPS_ORACLE_H
#define VMPS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_U32 = 0, ORC_U64 = 1, ORC_F32 = 2 };
/* variants: A copy-merge (Fig. 1), B Virtual-Memory (Sec. 4), C Pingpong (Sec. 3)
 * with the last-pop right-to-left merge, C0 Pingpong without it */
enum { ORC_VARIANT_COPYMERGE = 0, ORC_VARIANT_VM = 1, ORC_VARIANT_PINGPONG = 2, ORC_VARIANT_PINGPONG_PLAIN = 3 };
enum { ORC_KIND_ASC = 0, ORC_KIND_DESC = 1, ORC_KIND_EXT = 2 };
enum { ORC_OK = 0, ORC_EINVAL = -1, ORC_ECAP = -2, ORC_ENOMEM = -3, ORC_EINTERNAL = -4 };

typedef struct {
  uint64_t i, j, k;   /* merge [i,j) with [j,k), 0-based half-open (P:410 footnote) */
  uint32_t power;     /* power of the boundary j */
  uint32_t pad;
} orc_merge_t;

typedef struct {
  uint64_t n, runs, merges, merge_cost_M;   /* M: P:416-419 */
  uint64_t minrun;
  uint64_t comp_runs, comp_merge;           /* comparisons: run formation / merge phase (C16) */
  uint64_t moves_runs;                      /* run formation: reversal + insertion sort assignments */
  uint64_t moves_merge_out;                 /* element writes of merge outputs (== M, C14) */
  uint64_t moves_staging;                   /* A: left-run copies; B: extraction pushes;
                                               C: copies of pushed buffers into stackBuf */
  uint64_t moves_copy;                      /* B: final Copy (evictions + page copies) */
  uint64_t max_stack;                       /* max stack height */
  uint64_t reversed_elems, extended_runs;
  uint64_t page_elems;                      /* B: page size P (elements) */
  uint64_t peak_extra_pages;                /* B: pages allocated beyond the input's */
  uint64_t peak_extra_elems;                /* A: max buffer length; B: peak_extra_pages*P */
  uint64_t peak_meta_words;                 /* B: page-list + free-list entries (peak) */
  uint64_t evictions;                       /* B: pages evicted by Copy */
} orc_stats_t;

uint32_t orc_minrun(uint64_t n);
uint32_t orc_power(uint64_t n, uint64_t i, uint64_t j, uint64_t k);
uint32_t orc_power_brute(uint64_t n, uint64_t i, uint64_t j, uint64_t k);
uint64_t orc_page_size(uint64_t n, uint32_t T);
int orc_less(int key_type, uint64_t a, uint64_t b);

/* Sort keys[0,n) (and vals, if non-NULL) in place with Powersort (variant A
 * or B), writing the plan: run_start[runs], run_kind[runs] (cap_runs entries
 * available), merges[runs-1] in Alg. 1 execution order. minrun_override=0
 * means the paper's rule. */
int orc_sort(int key_type, void* keys, uint32_t* vals, uint64_t n, int variant,
             uint32_t minrun_override, uint64_t* run_start, uint8_t* run_kind,
             uint64_t cap_runs, orc_merge_t* merges, orc_stats_t* st);

/* Test hook (variant B only): page-size word count T used for P (reading R9)
 * instead of the element's own (0 = the element's); lets the page flow of the
 * paper's wider types (ptr T = 2, blob30 T = 30) be measured on the
 * same key array.  Process-global, not thread safe. */
void orc_set_vm_words(uint32_t T);

/* Plan only: ExtractRun boundaries + Power + Alg. 1 without moving data. */
int orc_plan(int key_type, const void* keys, uint64_t n, uint32_t minrun_override,
             uint64_t* run_start, uint8_t* run_kind, uint64_t cap_runs,
             orc_merge_t* merges, orc_stats_t* st);

/* Alg. 1's policy alone over given run starts (for run-set examples). */
int orc_policy(uint64_t n, const uint64_t* run_start, uint64_t r, orc_merge_t* merges,
               uint64_t* max_stack);

#ifdef __cplusplus
}
#endif
#endif
