/*
 * vmps_oracle.c -- plain, slow, single-threaded CPU oracle of Powersort
 * (arXiv 2605.27147).  TEST INFRASTRUCTURE ONLY (see vmps_oracle.h).
 *
 * What it computes, in the paper's order and notation:
 *   - minrun: Timsort's rule, P:756 ("start from l = n, then repeatedly set
 *     l = ceil(l/2) until l < 64").
 *   - ExtractRun (P:756 insertion sort; descending runs per
 *     BASELINE.json north_star, reading R3): a run starting at s is
 *     strictly descending if a[s+1] < a[s] (then it extends while strictly
 *     descending and is reversed), otherwise it is the maximal non-decreasing
 *     prefix; a run shorter than minrun is extended to min(n, s+minrun) by a
 *     straight stable insertion sort.
 *   - Power: least p with an integer c such that
 *     (i+j)/2n < c*2^-p <= (j+k)/2n.  orc_power_brute is that definition
 *     literally; orc_power is the exact 64-bit fixed-point form.
 *   - Alg. 1 Abstract Powersort, with the final loop read as
 *     pop-and-merge (reading R2).
 *   - Variant A "standard copy-merge" (Fig. 1): copy the LEFT run to
 *     a buffer, merge left-to-right back into the input, ties to the left
 *     (Alg. 2 StandardMerge).  No tail skip (reading R8).
 *   - Variant C "Pingpong" (Sec. 3): buffers on the
 *     stack live in stackBuf[i,j) (n extra elements), curr / next / work in
 *     input[i,j); a pushed buffer is copied into stackBuf (line 10 of Alg. 1);
 *     MergeBuffers merges stackBuf[i,j) with input[j,k) left to right into
 *     input[i,k); at the last pop of a line-7 loop it instead merges right to
 *     left into stackBuf[i,k), taking the right run's element on
 *     ties (it must land later; SPEC's backward tie rule, reading R16), so
 *     the push that follows copies nothing.  The final unwind (lines 12-13)
 *     always merges into input, so Copy does nothing.  C0 is the same
 *     without the last-pop merge.
 *   - Variant B "Virtual-Memory" (Sec. 4): pages of P elements
 *     (rounding per reading R9), free list, page
 *     lists as arrays (App. A), PushBack/PopFront,
 *     NewBuffer segmentation with a never-freed partial last page
 *     (P:574-576), page-by-page merging with PageMerge (Alg. 2, P:652-666,
 *     P:641-647), Copy with eviction using an inverse page map
 *     instead of the quadratic scan (footnote P:588).
 *
 * The f32 order (reading R5): -0.0 precedes +0.0, every NaN is greater than
 * every non-NaN and all NaNs compare equal.  Written out with <math.h>
 * predicates, not with the bit trick the CUDA path uses.
 */
#include "vmps_oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* element type and order                                                    */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t key; /* u32 / f32 bits in the low 32 bits */
  uint32_t val;
} item;

static int f32_less(uint32_t abits, uint32_t bbits) {
  float a, b;
  memcpy(&a, &abits, 4);
  memcpy(&b, &bbits, 4);
  if (isnan(a)) return 0;  /* NaN is never less than anything (NaNs last, equal) */
  if (isnan(b)) return 1;  /* every non-NaN precedes NaN */
  if (a < b) return 1;
  if (a > b) return 0;
  return signbit(a) && !signbit(b); /* -0.0 precedes +0.0 */
}

int orc_less(int key_type, uint64_t a, uint64_t b) {
  if (key_type == ORC_F32) return f32_less((uint32_t)a, (uint32_t)b);
  return a < b; /* unsigned integer order (reading R6) */
}

typedef struct ctx {
  int key_type;
  uint64_t n;
  uint64_t minrun;
  item* a;               /* the input array, as items (NULL in the plan-only pass) */
  const void* raw;       /* plan-only pass: the caller's keys, read in place */
  uint64_t* counter;     /* comparison counter currently charged */
  orc_stats_t* st;
  /* plan output */
  uint64_t* run_start;
  uint8_t* run_kind;
  uint64_t cap_runs;
  orc_merge_t* merges;
  int err;
  /* variant A */
  item* abuf;
  /* variant B */
  struct vm* vm;
  /* variant C */
  item* stack_buf;
  int last_pop_opt;  /* C: 1, C0: 0 */
  int last_pop;      /* set by powersort(): this merge is the last pop before a push */
} ctx;

static int less(ctx* c, const item* x, const item* y) {
  (*c->counter)++;
  return orc_less(c->key_type, x->key, y->key);
}

/* key of input position i for run detection (items, or raw keys when dry) */
static uint64_t key_at(const ctx* c, uint64_t i) {
  if (c->a) return c->a[i].key;
  if (c->key_type == ORC_U64) return ((const uint64_t*)c->raw)[i];
  return ((const uint32_t*)c->raw)[i];
}

/* "a[x] < a[y]" on the unmodified input, counted */
static int less_at(ctx* c, uint64_t x, uint64_t y) {
  (*c->counter)++;
  return orc_less(c->key_type, key_at(c, x), key_at(c, y));
}

/* ------------------------------------------------------------------------ */
/* minrun and Power                                     */
/* ------------------------------------------------------------------------ */
uint32_t orc_minrun(uint64_t n) {
  uint64_t l = n;
  while (l >= 64) l = (l + 1) / 2; /* l <- ceil(l/2) until l < 64 */
  return (uint32_t)l;
}

/* Literal definition: smallest p >= 1 such that there is an integer c with
 * (i+j)/(2n) < c * 2^-p <= (j+k)/(2n).  Multiply through by 2n*2^p:
 * (i+j)*2^p < c*2n <= (j+k)*2^p.  Brute force over c; for tests (small n). */
uint32_t orc_power_brute(uint64_t n, uint64_t i, uint64_t j, uint64_t k) {
  for (uint32_t p = 1; p < 62; ++p) {
    uint64_t two_p = 1ull << p;
    for (uint64_t cc = 0; cc <= two_p; ++cc) {
      unsigned __int128 lhs = (unsigned __int128)(i + j) * two_p;
      unsigned __int128 mid = (unsigned __int128)cc * (2 * n);
      unsigned __int128 rhs = (unsigned __int128)(j + k) * two_p;
      if (lhs < mid && mid <= rhs) return p;
    }
  }
  return 0;
}

/* Exact fixed point: with a=(i+j)/2n and b=(j+k)/2n in [0,1), an integer c
 * with a < c 2^-p <= b exists iff floor(a 2^p) != floor(b 2^p), i.e. iff the
 * binary expansions of a and b differ within their first p bits.  So p is
 * one plus the number of common leading bits of floor(a 2^64) and
 * floor(b 2^64) (they differ since b - a >= 1/n > 2^-64).  (F2 in SURVEY.) */
uint32_t orc_power(uint64_t n, uint64_t i, uint64_t j, uint64_t k) {
  uint64_t A = (uint64_t)((((unsigned __int128)(i + j)) << 63) / n);
  uint64_t B = (uint64_t)((((unsigned __int128)(j + k)) << 63) / n);
  return 1u + (uint32_t)__builtin_clzll(A ^ B);
}

/* Page size ("P ~ sqrt(n / (T lg n))", power of 2): largest power
 * of two <= sqrt(n/(T log2 n)), clamped to [16, n] (reading R9). */
uint64_t orc_page_size(uint64_t n, uint32_t T) {
  if (n < 2) return 16;
  double x = sqrt((double)n / ((double)T * log2((double)n)));
  uint64_t P = 1;
  while ((double)(P * 2) <= x) P *= 2;
  if (P < 16) P = 16;
  if (P > n) P = n;
  return P;
}

/* ------------------------------------------------------------------------ */
/* Run formation shared by both variants (ExtractRun, P:399 / P:756)       */
/* ------------------------------------------------------------------------ */
/* Natural run scan on the unmodified input a[s..n): returns its end e and
 * whether it is strictly descending.  Reads only positions >= s, which no
 * earlier run has touched (Alg. 1 consumes work left to right). */
static uint64_t natural_run(ctx* c, uint64_t s, int* desc) {
  uint64_t n = c->n, e;
  if (s + 1 < n && less_at(c, s + 1, s)) {
    e = s + 2;
    while (e < n && less_at(c, e, e - 1)) e++;
    *desc = 1;
  } else {
    e = s + 1;
    while (e < n && !less_at(c, e, e - 1)) e++;
    *desc = 0;
  }
  return e;
}

/* Random access into a run being formed (array for A, page list for B). */
typedef struct {
  item* (*at)(void* self, uint64_t x);
  void* self;
} accessor;

static void reverse_run(ctx* c, accessor* r, uint64_t len) {
  for (uint64_t x = 0, y = len - 1; x < y; ++x, --y) {
    item t = *r->at(r->self, x);
    *r->at(r->self, x) = *r->at(r->self, y);
    *r->at(r->self, y) = t;
    c->st->moves_runs += 3;
  }
  c->st->reversed_elems += len;
}

/* Straight insertion sort of positions [sorted_len, len) into the sorted
 * prefix [0, sorted_len); stable (shift only while strictly less). */
static void insertion_extend(ctx* c, accessor* r, uint64_t sorted_len, uint64_t len) {
  for (uint64_t x = sorted_len; x < len; ++x) {
    item t = *r->at(r->self, x);
    c->st->moves_runs++;
    uint64_t y = x;
    while (y > 0 && less(c, &t, r->at(r->self, y - 1))) {
      *r->at(r->self, y) = *r->at(r->self, y - 1);
      c->st->moves_runs++;
      y--;
    }
    *r->at(r->self, y) = t;
    c->st->moves_runs++;
  }
}

/* Record a run in the plan. */
static void emit_run(ctx* c, uint64_t s, uint8_t kind) {
  uint64_t r = c->st->runs++;
  if (r < c->cap_runs) {
    c->run_start[r] = s;
    c->run_kind[r] = kind;
  } else {
    c->err = ORC_ECAP;
  }
}

/* The run [s, e) with its kind, per ExtractRun: returns e. */
static uint64_t run_bounds(ctx* c, uint64_t s, int* desc, uint64_t* nat_end, uint8_t* kind) {
  uint64_t e = natural_run(c, s, desc);
  *nat_end = e;
  *kind = *desc ? ORC_KIND_DESC : ORC_KIND_ASC;
  if (e - s < c->minrun) {
    uint64_t e2 = s + c->minrun < c->n ? s + c->minrun : c->n;
    *kind |= ORC_KIND_EXT;
    c->st->extended_runs++;
    e = e2;
  }
  return e;
}

/* ------------------------------------------------------------------------ */
/* Buffers and the strategy interface                           */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t lo, hi; /* subsegment of the original index space */
  int h;           /* strategy handle (B: page-list slot) */
} buf;

typedef struct strategy {
  void (*new_buffer)(ctx*);
  buf (*extract_run)(ctx*, uint64_t s);
  buf (*merge_buffers)(ctx*, buf x, buf y);
  void (*copy)(ctx*, buf curr);
  void (*push)(ctx*, buf* b); /* optional: the buffer moves onto the stack (C) */
} strategy;

static void record_merge(ctx* c, buf x, buf y, uint32_t p) {
  uint64_t m = c->st->merges++;
  c->merges[m].i = x.lo;
  c->merges[m].j = x.hi;
  c->merges[m].k = y.hi;
  c->merges[m].power = p;
  c->merges[m].pad = 0;
  c->st->merge_cost_M += y.hi - x.lo; /* merge cost: sum of input lengths */
}

/* Alg. 1, Abstract Powersort. */
static void powersort(ctx* c, strategy* S) {
  uint64_t n = c->n;
  buf stk[72];
  uint32_t pw[72];
  int top = 0;
  S->new_buffer(c);                         /* line 1 */
  buf curr = S->extract_run(c, 0);          /* line 3 */
  while (curr.hi < n && !c->err) {          /* line 4: work not empty */
    buf next = S->extract_run(c, curr.hi);  /* line 5 */
    uint32_t p = orc_power(n, curr.lo, curr.hi, next.hi); /* line 6 */
    while (top > 0 && pw[top - 1] >= p) {   /* line 7 */
      record_merge(c, stk[top - 1], curr, pw[top - 1]);
      c->last_pop = !(top > 1 && pw[top - 2] >= p); /* the loop ends after this pop */
      curr = S->merge_buffers(c, stk[top - 1], curr); /* line 8 */
      top--;                                /* line 9 */
    }
    c->last_pop = 0;
    if (top >= 71) { c->err = ORC_EINTERNAL; return; }
    if (S->push) S->push(c, &curr);
    stk[top] = curr;                        /* line 10 */
    pw[top] = p;
    top++;
    if ((uint64_t)top > c->st->max_stack) c->st->max_stack = (uint64_t)top;
    curr = next;                            /* line 11 */
  }
  while (top > 0 && !c->err) {              /* lines 12-13, with Pop (R2) */
    record_merge(c, stk[top - 1], curr, pw[top - 1]);
    curr = S->merge_buffers(c, stk[top - 1], curr);
    top--;
  }
  if (!c->err) S->copy(c, curr);            /* line 14 */
}

/* ------------------------------------------------------------------------ */
/* Variant A: standard copy-merge (Fig. 1)                                  */
/* ------------------------------------------------------------------------ */
static item* arr_at(void* self, uint64_t x) { return (item*)self + x; }

static void a_new_buffer(ctx* c) { (void)c; } /* buffers are subsegments of input */

static buf a_extract_run(ctx* c, uint64_t s) {
  int desc;
  uint64_t nat;
  uint8_t kind;
  uint64_t e = run_bounds(c, s, &desc, &nat, &kind);
  accessor r = {arr_at, c->a + s};
  if (desc) reverse_run(c, &r, nat - s);
  if (e > nat) insertion_extend(c, &r, nat - s, e - s);
  emit_run(c, s, kind);
  buf b = {s, e, 0};
  return b;
}

static buf a_merge(ctx* c, buf x, buf y) {
  uint64_t nl = x.hi - x.lo;
  item* a = c->a;
  /* (1) copy the left run to the buffer */
  for (uint64_t t = 0; t < nl; ++t) c->abuf[t] = a[x.lo + t];
  c->st->moves_staging += nl;
  if (nl > c->st->peak_extra_elems) c->st->peak_extra_elems = nl;
  /* (2) merge buffer and a[j,k) into a[i,k), left to right, ties to the left */
  uint64_t xa = 0, xb = y.lo, o = x.lo;
  c->counter = &c->st->comp_merge;
  while (xa < nl && xb < y.hi) {
    if (!less(c, &a[xb], &c->abuf[xa])) a[o++] = c->abuf[xa++]; /* buf[xa] <= b[xb] */
    else a[o++] = a[xb++];
  }
  while (xa < nl) a[o++] = c->abuf[xa++];
  while (xb < y.hi) { a[o] = a[xb]; o++; xb++; } /* no tail skip: written once */
  c->st->moves_merge_out += y.hi - x.lo;
  c->counter = &c->st->comp_runs;
  buf r = {x.lo, y.hi, 0};
  return r;
}

static void a_copy(ctx* c, buf curr) { (void)c; (void)curr; } /* already in input */

/* ------------------------------------------------------------------------ */
/* Variant C: Pingpong (Sec. 3)                                  */
/* buf.h: 0 = the buffer lives in input[lo,hi), 1 = in stackBuf[lo,hi)      */
/* ------------------------------------------------------------------------ */
static buf c_extract_run(ctx* c, uint64_t s) {
  buf b = a_extract_run(c, s); /* ExtractRun: the run stays in input */
  b.h = 0;
  return b;
}

/* Pushing a buffer that lives in input copies it to stackBuf. */
static void c_push(ctx* c, buf* b) {
  if (b->h == 1) return; /* produced by a last-pop merge: already in stackBuf */
  for (uint64_t t = b->lo; t < b->hi; ++t) c->stack_buf[t] = c->a[t];
  c->st->moves_staging += b->hi - b->lo;
  b->h = 1;
}

static buf c_merge(ctx* c, buf x, buf y) {
  item* sb = c->stack_buf;
  item* a = c->a;
  if (x.h != 1 || y.h != 0) { c->err = ORC_EINTERNAL; return x; }
  c->counter = &c->st->comp_merge;
  buf r = {x.lo, y.hi, 0};
  if (c->last_pop_opt && c->last_pop) {
    /* last pop: merge right to left into stackBuf[i,k); from the
     * back, a tie outputs the right run's element first (it lands later) */
    uint64_t xa = x.hi, xb = y.hi, o = y.hi; /* one past the next element */
    while (xa > x.lo && xb > y.lo) {
      if (less(c, &a[xb - 1], &sb[xa - 1])) sb[--o] = sb[--xa]; /* b < a: a is larger */
      else sb[--o] = a[--xb];                                  /* a <= b: b goes last */
    }
    while (xb > y.lo) { --o; sb[o] = a[--xb]; }
    while (xa > x.lo) { --o; sb[o] = sb[--xa]; } /* written once (no tail skip, R8) */
    r.h = 1;
  } else {
    /* merge stackBuf[i,j) and input[j,k) left to right into input[i,k) */
    uint64_t xa = x.lo, xb = y.lo, o = x.lo;
    while (xa < x.hi && xb < y.hi) {
      if (!less(c, &a[xb], &sb[xa])) a[o++] = sb[xa++]; /* a <= b: ties to the left */
      else a[o++] = a[xb++];
    }
    while (xa < x.hi) a[o++] = sb[xa++];
    while (xb < y.hi) { a[o] = a[xb]; o++; xb++; }
  }
  c->st->moves_merge_out += y.hi - x.lo;
  c->counter = &c->st->comp_runs;
  return r;
}

static void c_copy(ctx* c, buf curr) {
  if (curr.h != 0) c->err = ORC_EINTERNAL; /* the final unwind merges into input */
}

/* ------------------------------------------------------------------------ */
/* Variant B: Virtual-Memory pages (Sec. 4)                                 */
/* ------------------------------------------------------------------------ */
typedef struct {
  uint64_t* pg;   /* page-id list (App. A: arrays, not linked lists) */
  uint64_t h0;    /* index of the first live entry of pg */
  uint64_t np, cap;
  uint64_t front; /* offset consumed in the first page */
  uint64_t len;   /* logical length */
  int used;
} pbuf;

typedef struct vm {
  uint64_t P;
  uint64_t n_in_pages; /* ceil(n/P) input pages, ids 0.. */
  uint64_t n_full_in;  /* floor(n/P) */
  item** mem;          /* page id -> storage */
  uint64_t n_pages, cap_pages;
  uint64_t* free_list;
  uint64_t n_free, cap_free;
  pbuf* bufs;
  int nbufs, capbufs;
  int work;
  uint64_t meta_now;
} vm;

static void vm_meta(ctx* c, int64_t d) {
  c->vm->meta_now += d;
  if (c->vm->meta_now > c->st->peak_meta_words) c->st->peak_meta_words = c->vm->meta_now;
}

/* Get a page: from the free list if possible, else a fresh page. */
static uint64_t vm_get_page(ctx* c) {
  vm* v = c->vm;
  if (v->n_free > 0) {
    vm_meta(c, -1);
    return v->free_list[--v->n_free];
  }
  if (v->n_pages == v->cap_pages) {
    v->cap_pages *= 2;
    v->mem = (item**)realloc(v->mem, v->cap_pages * sizeof(item*));
  }
  uint64_t id = v->n_pages++;
  v->mem[id] = (item*)malloc(v->P * sizeof(item));
  if (!v->mem[id]) c->err = ORC_ENOMEM;
  c->st->peak_extra_pages = v->n_pages - v->n_in_pages;
  return id;
}

/* Release a page to the free list; the partial last input page is never
 * declared free (P:574-576 footnote). */
static void vm_release(ctx* c, uint64_t id) {
  vm* v = c->vm;
  if (id == v->n_full_in && v->n_full_in < v->n_in_pages) return;
  if (v->n_free == v->cap_free) {
    v->cap_free = v->cap_free ? 2 * v->cap_free : 64;
    v->free_list = (uint64_t*)realloc(v->free_list, v->cap_free * sizeof(uint64_t));
  }
  v->free_list[v->n_free++] = id;
  vm_meta(c, +1);
}

static int vm_new_pbuf(ctx* c) {
  vm* v = c->vm;
  for (int h = 0; h < v->nbufs; ++h)
    if (!v->bufs[h].used) {
      memset(&v->bufs[h], 0, sizeof(pbuf));
      v->bufs[h].used = 1;
      return h;
    }
  if (v->nbufs == v->capbufs) {
    v->capbufs *= 2;
    v->bufs = (pbuf*)realloc(v->bufs, v->capbufs * sizeof(pbuf));
  }
  memset(&v->bufs[v->nbufs], 0, sizeof(pbuf));
  v->bufs[v->nbufs].used = 1;
  return v->nbufs++;
}

static void vm_free_pbuf(ctx* c, int h) {
  pbuf* b = &c->vm->bufs[h];
  vm_meta(c, -(int64_t)(b->np - b->h0));
  free(b->pg);
  b->pg = NULL;
  b->np = b->cap = b->h0 = 0;
  b->used = 0;
}

static void pbuf_append_page(ctx* c, pbuf* b, uint64_t id) {
  if (b->np == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 8;
    b->pg = (uint64_t*)realloc(b->pg, b->cap * sizeof(uint64_t));
  }
  b->pg[b->np++] = id;
  vm_meta(c, +1);
}

/* Pop the first page (after it was fully consumed) and release it. */
static void pbuf_drop_first_page(ctx* c, pbuf* b) {
  vm_release(c, b->pg[b->h0]);
  b->h0++;
  vm_meta(c, -1);
  b->front = 0;
}

static item* pbuf_at(ctx* c, pbuf* b, uint64_t x) {
  uint64_t q = b->front + x;
  return c->vm->mem[b->pg[b->h0 + q / c->vm->P]] + q % c->vm->P;
}

/* PushBack: insert into the last page, taking a new page when full. */
static void pbuf_push_back(ctx* c, int h, const item* it) {
  pbuf* b = &c->vm->bufs[h];
  uint64_t q = b->front + b->len;
  if (q == (b->np - b->h0) * c->vm->P) {
    uint64_t id = vm_get_page(c);
    b = &c->vm->bufs[h];
    pbuf_append_page(c, b, id);
  }
  c->vm->mem[b->pg[b->h0 + q / c->vm->P]][q % c->vm->P] = *it;
  b->len++;
}

/* PopFront: an emptied page goes to the free list. */
static item pbuf_pop_front(ctx* c, int h) {
  pbuf* b = &c->vm->bufs[h];
  item it = c->vm->mem[b->pg[b->h0]][b->front];
  b->front++;
  b->len--;
  if (b->front == c->vm->P || b->len == 0) pbuf_drop_first_page(c, b);
  return it;
}

typedef struct {
  ctx* c;
  int h;
} pacc;
static item* pacc_at(void* self, uint64_t x) {
  pacc* p = (pacc*)self;
  return pbuf_at(p->c, &p->c->vm->bufs[p->h], x);
}

/* NewBuffer: segment the input into pages. */
static void b_new_buffer(ctx* c) {
  vm* v = c->vm;
  int h = vm_new_pbuf(c);
  v->work = h;
  for (uint64_t q = 0; q < v->n_in_pages; ++q) pbuf_append_page(c, &v->bufs[h], q);
  v->bufs[h].front = 0;
  v->bufs[h].len = c->n;
}

/* ExtractRun: pop the run from work, push into fresh pages. */
static buf b_extract_run(ctx* c, uint64_t s) {
  int desc;
  uint64_t nat;
  uint8_t kind;
  /* work's remaining elements still sit at their original positions (input
   * pages are only reused after being fully popped), so scan a[] directly */
  uint64_t e = run_bounds(c, s, &desc, &nat, &kind);
  int h = vm_new_pbuf(c);
  for (uint64_t t = s; t < e; ++t) {
    item it = pbuf_pop_front(c, c->vm->work);
    pbuf_push_back(c, h, &it);
    c->st->moves_staging++;
  }
  pacc pa = {c, h};
  accessor r = {pacc_at, &pa};
  if (desc) reverse_run(c, &r, nat - s);
  if (e > nat) insertion_extend(c, &r, nat - s, e - s);
  emit_run(c, s, kind);
  buf b = {s, e, h};
  return b;
}

/* MergeBuffers page by page with PageMerge (Alg. 2). */
static buf b_merge(ctx* c, buf x, buf y) {
  vm* v = c->vm;
  uint64_t P = v->P;
  int hz = vm_new_pbuf(c);
  c->counter = &c->st->comp_merge;
  for (;;) {
    pbuf* X = &v->bufs[x.h];
    pbuf* Y = &v->bufs[y.h];
    if (X->len == 0 || Y->len == 0) break;
    pbuf* Z = &v->bufs[hz];
    if ((Z->front + Z->len) == (Z->np - Z->h0) * P) { /* output page full: take a page */
      uint64_t id = vm_get_page(c);
      X = &v->bufs[x.h];
      Y = &v->bufs[y.h];
      Z = &v->bufs[hz];
      pbuf_append_page(c, Z, id);
    }
    item* pa = v->mem[X->pg[X->h0]];
    item* pb = v->mem[Y->pg[Y->h0]];
    uint64_t qz = Z->front + Z->len;
    item* pr = v->mem[Z->pg[Z->h0 + qz / P]];
    uint64_t xa = X->front, ya = X->front + X->len < P ? X->front + X->len : P;
    uint64_t xb = Y->front, yb = Y->front + Y->len < P ? Y->front + Y->len : P;
    uint64_t xr = qz % P, yr = P;
    uint64_t xr0 = xr, xa0 = xa, xb0 = xb;
    /* PageMerge: while x_a < y_a and x_b < y_b and x_r < y_r */
    while (xa < ya && xb < yb && xr < yr) {
      if (!less(c, &pb[xb], &pa[xa])) pr[xr] = pa[xa++]; /* a[x_a] <= b[x_b] */
      else pr[xr] = pb[xb++];
      xr++;
    }
    c->st->moves_merge_out += xr - xr0;
    Z->len += xr - xr0;
    X->front = xa;
    X->len -= xa - xa0;
    Y->front = xb;
    Y->len -= xb - xb0;
    if (X->front == P || X->len == 0) pbuf_drop_first_page(c, X);
    if (Y->front == P || Y->len == 0) pbuf_drop_first_page(c, Y);
  }
  /* the rest of the non-empty input, element by element (reading R8) */
  int hr = v->bufs[x.h].len ? x.h : y.h;
  while (v->bufs[hr].len) {
    item it = pbuf_pop_front(c, hr);
    pbuf_push_back(c, hz, &it);
    c->st->moves_merge_out++;
  }
  c->counter = &c->st->comp_runs;
  vm_free_pbuf(c, x.h);
  vm_free_pbuf(c, y.h);
  buf r = {x.lo, y.hi, hz};
  return r;
}

/* Copy: place curr's pages into input page order, evicting a page
 * still referenced later; collision lookup via an inverse map (R10). */
static void b_copy(ctx* c, buf curr) {
  vm* v = c->vm;
  uint64_t P = v->P, n = c->n;
  pbuf* B = &v->bufs[curr.h];
  if (B->front != 0 || B->len != n || B->h0 != 0) { c->err = ORC_EINTERNAL; return; }
  int64_t* owner = (int64_t*)malloc((v->n_pages + 8) * sizeof(int64_t));
  uint64_t cap_owner = v->n_pages + 8;
  for (uint64_t id = 0; id < cap_owner; ++id) owner[id] = -1;
  for (uint64_t q = 0; q < B->np; ++q) owner[B->pg[q]] = (int64_t)q;
  for (uint64_t q = 0; q < B->np; ++q) {
    B = &v->bufs[curr.h];
    uint64_t src = B->pg[q];
    uint64_t cnt = (q + 1) * P <= n ? P : n - q * P;
    if (src == q) continue; /* already in place */
    if (owner[q] >= 0) {   /* input page q still holds a later logical page: evict */
      uint64_t q2 = (uint64_t)owner[q];
      uint64_t cnt2 = (q2 + 1) * P <= n ? P : n - q2 * P;
      uint64_t e = vm_get_page(c); /* "a new page": free list first */
      B = &v->bufs[curr.h];
      if (e >= cap_owner) {
        owner = (int64_t*)realloc(owner, (e + 8) * sizeof(int64_t));
        for (uint64_t id = cap_owner; id < e + 8; ++id) owner[id] = -1;
        cap_owner = e + 8;
      }
      memcpy(v->mem[e], v->mem[q], cnt2 * sizeof(item));
      c->st->moves_copy += cnt2;
      c->st->evictions++;
      B->pg[q2] = e;
      owner[e] = (int64_t)q2;
      owner[q] = -1;
      src = B->pg[q];
    }
    memcpy(v->mem[q], v->mem[src], cnt * sizeof(item));
    c->st->moves_copy += cnt;
    owner[src] = -1;
    vm_release(c, src);
    B->pg[q] = q;
    owner[q] = (int64_t)q;
  }
  free(owner);
}

/* ------------------------------------------------------------------------ */
/* Dry strategy for orc_plan: ExtractRun boundaries + policy, no data moves */
/* ------------------------------------------------------------------------ */
static void d_new_buffer(ctx* c) { (void)c; }
static buf d_extract_run(ctx* c, uint64_t s) {
  int desc;
  uint64_t nat;
  uint8_t kind;
  uint64_t e = run_bounds(c, s, &desc, &nat, &kind);
  emit_run(c, s, kind);
  buf b = {s, e, 0};
  return b;
}
static buf d_merge(ctx* c, buf x, buf y) {
  (void)c;
  buf r = {x.lo, y.hi, 0};
  return r;
}
static void d_copy(ctx* c, buf curr) { (void)c; (void)curr; }

static uint32_t g_vm_words = 0;
void orc_set_vm_words(uint32_t T) { g_vm_words = T; }

/* ------------------------------------------------------------------------ */
/* entry points                                                             */
/* ------------------------------------------------------------------------ */
static int run_common(int key_type, void* keys, uint32_t* vals, uint64_t n, int variant,
                      uint32_t minrun_override, uint64_t* run_start, uint8_t* run_kind,
                      uint64_t cap_runs, orc_merge_t* merges, orc_stats_t* st, int dry) {
  if (!st) return ORC_EINVAL;
  memset(st, 0, sizeof(*st));
  if (key_type < ORC_U32 || key_type > ORC_F32) return ORC_EINVAL;
  if (n > 0 && !keys) return ORC_EINVAL;
  st->n = n;
  if (n == 0) return ORC_OK;
  ctx c;
  memset(&c, 0, sizeof(c));
  c.key_type = key_type;
  c.n = n;
  c.minrun = minrun_override ? minrun_override : orc_minrun(n);
  st->minrun = c.minrun;
  c.st = st;
  c.counter = &st->comp_runs;
  c.run_start = run_start;
  c.run_kind = run_kind;
  c.cap_runs = cap_runs;
  c.merges = merges;
  c.raw = keys;
  if (!dry) {
    c.a = (item*)malloc(n * sizeof(item));
    if (!c.a) return ORC_ENOMEM;
    for (uint64_t t = 0; t < n; ++t) {
      c.a[t].key = key_type == ORC_U64 ? ((const uint64_t*)keys)[t] : ((const uint32_t*)keys)[t];
      c.a[t].val = vals ? vals[t] : (uint32_t)t;
    }
  }
  strategy S;
  S.push = NULL;
  if (dry) {
    S.new_buffer = d_new_buffer; S.extract_run = d_extract_run;
    S.merge_buffers = d_merge; S.copy = d_copy;
  } else if (variant == ORC_VARIANT_COPYMERGE) {
    S.new_buffer = a_new_buffer; S.extract_run = a_extract_run;
    S.merge_buffers = a_merge; S.copy = a_copy;
    c.abuf = (item*)malloc(n * sizeof(item));
    if (!c.abuf) { free(c.a); return ORC_ENOMEM; }
  } else if (variant == ORC_VARIANT_PINGPONG || variant == ORC_VARIANT_PINGPONG_PLAIN) {
    S.new_buffer = a_new_buffer; S.extract_run = c_extract_run;
    S.merge_buffers = c_merge; S.copy = c_copy; S.push = c_push;
    c.stack_buf = (item*)malloc(n * sizeof(item)); /* stackBuf: n elements */
    if (!c.stack_buf) { free(c.a); return ORC_ENOMEM; }
    c.last_pop_opt = variant == ORC_VARIANT_PINGPONG;
    st->peak_extra_elems = n;
  } else if (variant == ORC_VARIANT_VM) {
    S.new_buffer = b_new_buffer; S.extract_run = b_extract_run;
    S.merge_buffers = b_merge; S.copy = b_copy;
    uint32_t T = (key_type == ORC_U64 ? 2u : 1u) + (vals ? 1u : 0u); /* words (R9) */
    if (g_vm_words) T = g_vm_words;
    vm* v = (vm*)calloc(1, sizeof(vm));
    v->P = orc_page_size(n, T);
    v->n_full_in = n / v->P;
    v->n_in_pages = (n + v->P - 1) / v->P;
    v->cap_pages = v->n_in_pages + 64;
    v->mem = (item**)malloc(v->cap_pages * sizeof(item*));
    for (uint64_t q = 0; q < v->n_in_pages; ++q) v->mem[q] = c.a + q * v->P;
    v->n_pages = v->n_in_pages;
    v->capbufs = 128;
    v->bufs = (pbuf*)calloc(v->capbufs, sizeof(pbuf));
    c.vm = v;
    st->page_elems = v->P;
  } else {
    free(c.a);
    return ORC_EINVAL;
  }
  /* the merge array must hold runs-1 records; the caller sizes it with cap_runs */
  if (n == 1) {
    emit_run(&c, 0, ORC_KIND_ASC); /* step 1: runs = [0], no merges */
  } else {
    powersort(&c, &S);
  }
  int err = c.err;
  if (!err && !dry) {
    for (uint64_t t = 0; t < n; ++t) {
      if (key_type == ORC_U64) ((uint64_t*)keys)[t] = c.a[t].key;
      else ((uint32_t*)keys)[t] = (uint32_t)c.a[t].key;
      if (vals) vals[t] = c.a[t].val;
    }
  }
  if (c.vm) {
    vm* v = c.vm;
    st->peak_extra_elems = st->peak_extra_pages * v->P;
    for (uint64_t id = v->n_in_pages; id < v->n_pages; ++id) free(v->mem[id]);
    for (int h = 0; h < v->nbufs; ++h) free(v->bufs[h].pg);
    free(v->bufs);
    free(v->mem);
    free(v->free_list);
    free(v);
  }
  free(c.abuf);
  free(c.stack_buf);
  free(c.a);
  return err;
}

int orc_sort(int key_type, void* keys, uint32_t* vals, uint64_t n, int variant,
             uint32_t minrun_override, uint64_t* run_start, uint8_t* run_kind,
             uint64_t cap_runs, orc_merge_t* merges, orc_stats_t* st) {
  return run_common(key_type, keys, vals, n, variant, minrun_override, run_start, run_kind,
                    cap_runs, merges, st, 0);
}

int orc_plan(int key_type, const void* keys, uint64_t n, uint32_t minrun_override,
             uint64_t* run_start, uint8_t* run_kind, uint64_t cap_runs, orc_merge_t* merges,
             orc_stats_t* st) {
  return run_common(key_type, (void*)keys, NULL, n, 0, minrun_override, run_start, run_kind,
                    cap_runs, merges, st, 1);
}

/* Alg. 1's policy alone over given run starts: the merge plan of
 * runs [run_start[t], run_start[t+1]) (run_start[r] = n implied). */
int orc_policy(uint64_t n, const uint64_t* run_start, uint64_t r, orc_merge_t* merges,
               uint64_t* max_stack) {
  if (r == 0 || run_start[0] != 0) return ORC_EINVAL;
  for (uint64_t t = 1; t < r; ++t)
    if (run_start[t] <= run_start[t - 1] || run_start[t] >= n) return ORC_EINVAL;
  uint64_t lo[72], hi[72];
  uint32_t pw[72];
  int top = 0;
  uint64_t m = 0, ms = 0;
  uint64_t clo = 0, chi = r > 1 ? run_start[1] : n;
  for (uint64_t t = 1; t < r; ++t) {
    uint64_t nhi = t + 1 < r ? run_start[t + 1] : n;
    uint32_t p = orc_power(n, clo, chi, nhi);
    while (top > 0 && pw[top - 1] >= p) {
      merges[m].i = lo[top - 1]; merges[m].j = hi[top - 1]; merges[m].k = chi;
      merges[m].power = pw[top - 1]; merges[m].pad = 0; m++;
      clo = lo[top - 1];
      top--;
    }
    if (top >= 71) return ORC_EINTERNAL;
    lo[top] = clo; hi[top] = chi; pw[top] = p; top++;
    if ((uint64_t)top > ms) ms = (uint64_t)top;
    clo = chi; chi = nhi;
  }
  while (top > 0) {
    merges[m].i = lo[top - 1]; merges[m].j = hi[top - 1]; merges[m].k = chi;
    merges[m].power = pw[top - 1]; merges[m].pad = 0; m++;
    clo = lo[top - 1];
    top--;
  }
  if (max_stack) *max_stack = ms;
  return ORC_OK;
}
