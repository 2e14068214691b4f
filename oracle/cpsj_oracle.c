/*
 * cpsj_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference CPSJoin self-join path
 * (simjoin, /root/reference/pkg/src/simjoin) used as the CHECKER for the
 * B200 kernels.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library; the product
 * package never links or calls it.
 *
 * Every function cites the reference lines it restates.  Abbreviations:
 *   hsh = pkg/src/simjoin/hashing.py, emb = embed.py, cps = cpsjoin.py.
 *
 * Parity pin: oracle/gen_golden.py runs the reference itself on seeded
 * inputs and writes tests/golden/ (npz files); tests/test_oracle_golden.py checks
 * this file against those vectors bit for bit.
 *
 * Floating point: compiled with -ffp-contract=off so every double
 * expression rounds exactly like numpy's element-wise float64 ops.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

/* Minimal dynamic parallel-for over [0, n) on pthreads (chunked work
 * stealing through one atomic counter). */
typedef void (*body_fn)(void *arg, int64_t lo, int64_t hi, int tid);
typedef struct { body_fn fn; void *arg; int64_t n, chunk; int64_t next; int tid; } PF;
typedef struct { PF *pf; int tid; } PFT;

static void *pf_worker(void *p) {
    PFT *t = p;
    PF *pf = t->pf;
    for (;;) {
        int64_t lo = __atomic_fetch_add(&pf->next, pf->chunk, __ATOMIC_RELAXED);
        if (lo >= pf->n) break;
        int64_t hi = lo + pf->chunk < pf->n ? lo + pf->chunk : pf->n;
        pf->fn(pf->arg, lo, hi, t->tid);
    }
    return NULL;
}

static int resolve_threads(int nthreads) {
    if (nthreads > 0) return nthreads;
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int)c : 1;
}

static void parallel_for(int64_t n, int64_t chunk, int nthreads, body_fn fn, void *arg) {
    PF pf = {fn, arg, n, chunk > 0 ? chunk : 1, 0, 0};
    int nt = resolve_threads(nthreads);
    if (nt <= 1 || n <= pf.chunk) { if (n > 0) fn(arg, 0, n, 0); return; }
    pthread_t *th = malloc(nt * sizeof(pthread_t));
    PFT *ts = malloc(nt * sizeof(PFT));
    for (int i = 0; i < nt; i++) { ts[i].pf = &pf; ts[i].tid = i; }
    for (int i = 1; i < nt; i++) pthread_create(&th[i], NULL, pf_worker, &ts[i]);
    pf_worker(&ts[0]);
    for (int i = 1; i < nt; i++) pthread_join(th[i], NULL);
    free(th); free(ts);
}

#define GAMMA 0x9E3779B97F4A7C15ULL
#define M1 0xBF58476D1CE4E5B9ULL
#define M2 0x94D049BB133111EBULL

/* SplitMix64 finaliser: hsh:49-56 */
uint64_t orc_mix64(uint64_t z) {
    z += GAMMA;
    z = (z ^ (z >> 30)) * M1;
    z = (z ^ (z >> 27)) * M2;
    return z ^ (z >> 31);
}

/* k-th word of a node's counter stream: hsh:59-63 */
static inline uint64_t stream_word(uint64_t seed, uint64_t k) {
    return orc_mix64(seed ^ orc_mix64(k));
}

/* uniform in [0,1] from a stream word: hsh:66-68 (u64 -> f64 rounds to
 * nearest, then an exact scaling by 2^-64) */
static inline double stream_uniform(uint64_t seed, uint64_t k) {
    return (double)stream_word(seed, k) * 0x1p-64;
}

void orc_word_stream(uint64_t seed, int64_t n, uint64_t offset, uint64_t *out) {
    for (int64_t i = 0; i < n; i++) out[i] = stream_word(seed, offset + (uint64_t)i);
}

/* tabulation hash of one 32-bit key with a (4,256) u64 table: hsh:86-92 */
static inline uint64_t tab_hash(const uint64_t *tab, uint32_t key) {
    return tab[key & 0xFF] ^ tab[256 + ((key >> 8) & 0xFF)] ^
           tab[512 + ((key >> 16) & 0xFF)] ^ tab[768 + (key >> 24)];
}

/* MinHash of one set: argmin of the 64-bit hash, ties to the smaller token
 * (hsh:117-126; vector form hsh:129-146). */
static inline uint32_t set_minhash(const uint64_t *tab, const uint32_t *tok, int64_t len) {
    uint64_t best = tab_hash(tab, tok[0]);
    uint32_t arg = tok[0];
    for (int64_t i = 1; i < len; i++) {
        uint64_t g = tab_hash(tab, tok[i]);
        if (g < best || (g == best && tok[i] < arg)) { best = g; arg = tok[i]; }
    }
    return arg;
}

/* values[r, f] = h_f(x_r): emb:117-128.  tables is (F,4,256) u64. */
typedef struct {
    const uint32_t *tok; const int64_t *off; const uint64_t *tables; const uint64_t *bit_tables;
    int32_t F; uint32_t *values; uint64_t *sketch;
} MHArgs;

static void minhash_body(void *p, int64_t lo, int64_t hi, int tid) {
    MHArgs *a = p;
    (void)tid;
    for (int64_t r = lo; r < hi; r++) {
        const uint32_t *x = a->tok + a->off[r];
        int64_t len = a->off[r + 1] - a->off[r];
        for (int32_t f = 0; f < a->F; f++)
            a->values[r * a->F + f] = len > 0 ? set_minhash(a->tables + (int64_t)f * 1024, x, len) : 0u;
    }
}

void orc_minhash(const uint32_t *tok, const int64_t *off, int64_t n,
                 const uint64_t *tables, int32_t F, uint32_t *out, int nthreads) {
    MHArgs a = {tok, off, tables, NULL, F, out, NULL};
    parallel_for(n, 64, nthreads, minhash_body, &a);
}

/* 1-bit minwise sketch, bit i = low bit of bit-hash_i(minhash_i):
 * hsh:197-211 (scalar form hsh:187-194). */
static void sketch_body(void *p, int64_t lo, int64_t hi, int tid) {
    MHArgs *a = p;
    (void)tid;
    int32_t ell = a->F / 64, bits = a->F;
    for (int64_t r = lo; r < hi; r++) {
        const uint32_t *x = a->tok + a->off[r];
        int64_t len = a->off[r + 1] - a->off[r];
        const uint64_t *mh_tables = a->tables, *bit_tables = a->bit_tables;
        uint64_t *w = a->sketch + r * ell;
        for (int32_t k = 0; k < ell; k++) w[k] = 0;
        if (len == 0) continue;
        for (int32_t i = 0; i < bits; i++) {
            uint32_t h = set_minhash(mh_tables + (int64_t)i * 1024, x, len);
            uint64_t b = tab_hash(bit_tables + (int64_t)i * 1024, h) & 1ULL;
            w[i >> 6] |= b << (i & 63);
        }
    }
}

void orc_sketch(const uint32_t *tok, const int64_t *off, int64_t n,
                const uint64_t *mh_tables, const uint64_t *bit_tables, int32_t ell,
                uint64_t *out, int nthreads) {
    MHArgs a = {tok, off, mh_tables, bit_tables, 64 * ell, NULL, out};
    parallel_for(n, 64, nthreads, sketch_body, &a);
}

/* ------------------------------------------------------------------ */
/* join                                                                 */
/* ------------------------------------------------------------------ */

typedef struct {
    const uint32_t *tok;
    const int64_t *off;
    const int64_t *sizes;   /* emb.sizes: used by the size filter and union */
    int64_t n;
    const uint32_t *values; /* (n, t) */
    int32_t t;
    const uint64_t *sketch; /* (n, ell) */
    int32_t ell;
    double lam, eps;
    int32_t limit, kstar, depth_cap;
    int use_ct;             /* CPSJoinParams.use_count_table */
} Ctx;

typedef struct {
    int64_t *a, *b;
    double *sim;
    int64_t len, cap;
    int64_t pre, cand, res;
    int64_t max_depth, peak;
    int64_t *cap_events;   /* survivor counts of depth-capped nodes */
    int64_t n_cap_events, cap_events_cap;
    int error;             /* 1 = node-sketch pick index out of range */
} Acc;

static void acc_push(Acc *acc, int64_t a, int64_t b, double s) {
    if (acc->len == acc->cap) {
        acc->cap = acc->cap ? acc->cap * 2 : 1024;
        acc->a = realloc(acc->a, acc->cap * sizeof(int64_t));
        acc->b = realloc(acc->b, acc->cap * sizeof(int64_t));
        acc->sim = realloc(acc->sim, acc->cap * sizeof(double));
    }
    acc->a[acc->len] = a; acc->b[acc->len] = b; acc->sim[acc->len] = s;
    acc->len++;
}

static inline int sketch_dist(const Ctx *c, int64_t x, int64_t y) {
    const uint64_t *sx = c->sketch + x * c->ell, *sy = c->sketch + y * c->ell;
    int d = 0;
    for (int k = 0; k < c->ell; k++) d += __builtin_popcountll(sx[k] ^ sy[k]);
    return d;
}

/* size filter: cps:129-137 (self-join: no side mask) */
static inline int size_ok(const Ctx *c, int64_t x, int64_t y) {
    int64_t sa = c->sizes[x], sb = c->sizes[y];
    int64_t mn = sa < sb ? sa : sb, mx = sa < sb ? sb : sa;
    return (double)mn >= c->lam * (double)mx - 1e-9;
}

/* exact verification of one candidate: cps:114-127 (the sparse row product
 * there counts common column indices; here a merge of sorted rows) */
static void verify(const Ctx *c, Acc *acc, int64_t x, int64_t y) {
    acc->cand++;
    const uint32_t *p = c->tok + c->off[x], *pe = c->tok + c->off[x + 1];
    const uint32_t *q = c->tok + c->off[y], *qe = c->tok + c->off[y + 1];
    int64_t inter = 0;
    while (p < pe && q < qe) {
        if (*p == *q) { inter++; p++; q++; }
        else if (*p < *q) p++;
        else q++;
    }
    int64_t uni = c->sizes[x] + c->sizes[y] - inter;
    double sim = (double)inter / (double)uni;
    if (sim >= c->lam) { acc->res++; acc_push(acc, x, y, sim); }
}

/* all pairs i<j of a node in member order: cps:139-157 */
static void brute_force_pairs(const Ctx *c, Acc *acc, const int64_t *mem, int64_t m) {
    if (m < 2) return;
    acc->pre += m * (m - 1) / 2;
    int accept = 64 * c->ell - c->kstar;  /* matches >= k*  <=>  dist <= mbits - k* */
    for (int64_t i = 0; i < m; i++)
        for (int64_t j = i + 1; j < m; j++)
            if (sketch_dist(c, mem[i], mem[j]) <= accept && size_ok(c, mem[i], mem[j]))
                verify(c, acc, mem[i], mem[j]);
}

/* one member against a member list without itself: cps:159-171 */
static void brute_force_point(const Ctx *c, Acc *acc, int64_t x, const int64_t *mem,
                              const uint8_t *alive, int64_t m) {
    int accept = 64 * c->ell - c->kstar;
    int64_t others = 0;
    for (int64_t j = 0; j < m; j++) if (alive[j] && mem[j] != x) others++;
    if (others == 0) return;
    acc->pre += others;
    for (int64_t j = 0; j < m; j++) {
        if (!alive[j] || mem[j] == x) continue;
        if (sketch_dist(c, x, mem[j]) <= accept && size_ok(c, x, mem[j]))
            verify(c, acc, x, mem[j]);
    }
}

static int cmp_u32_first(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : (x > y);
}

/* pre-split pruning, returns survivors in member order: cps:248-275,
 * node sketch cps:182-198, estimates cps:201-206 */
static int64_t brute_force_step(const Ctx *c, Acc *acc, const int64_t *mem, int64_t m,
                                uint64_t seed, int64_t *surv) {
    if (m <= c->limit) { brute_force_pairs(c, acc, mem, m); return 0; }
    double thr = (1.0 - c->eps) * c->lam;
    uint8_t *flag = malloc(m);
    int64_t nflag = 0;
    if (c->use_ct) {
        /* exact embedded average similarity: cps:209-219.  count[dense id]
         * over the node, summed over each member's t tokens, minus t;
         * dense ids are equal exactly when (position, value) are */
        int64_t *sum = calloc(m, sizeof(int64_t));
        typedef struct { uint32_t v; int64_t k; } VK;
        VK *tmp = malloc(m * sizeof(VK));
        for (int32_t i = 0; i < c->t; i++) {
            for (int64_t k = 0; k < m; k++) { tmp[k].v = c->values[mem[k] * c->t + i]; tmp[k].k = k; }
            qsort(tmp, m, sizeof(VK), cmp_u32_first);
            int64_t g = 0;
            while (g < m) {
                int64_t e = g + 1;
                while (e < m && tmp[e].v == tmp[g].v) e++;
                for (int64_t q = g; q < e; q++) sum[tmp[q].k] += e - g;
                g = e;
            }
        }
        for (int64_t k = 0; k < m; k++) {
            double est = (double)(sum[k] - c->t) / (double)((int64_t)c->t * (m - 1));
            flag[k] = est > thr;
            nflag += flag[k];
        }
        free(tmp);
        free(sum);
    } else {
        int32_t mbits = 64 * c->ell;
        uint64_t nsk[64];
        memset(nsk, 0, sizeof(nsk));
        for (int32_t i = 0; i < mbits; i++) {
            double u = stream_uniform(seed, (uint64_t)c->t + (uint64_t)i);
            int64_t idx = (int64_t)(u * (double)m);
            if (idx >= m) { acc->error = 1; idx = m - 1; }
            uint64_t w = c->sketch[mem[idx] * c->ell + (i >> 6)];
            nsk[i >> 6] |= ((w >> (i & 63)) & 1ULL) << (i & 63);
        }
        for (int64_t k = 0; k < m; k++) {
            const uint64_t *s = c->sketch + mem[k] * c->ell;
            int64_t dist = 0;
            for (int w = 0; w < c->ell; w++) dist += __builtin_popcountll(s[w] ^ nsk[w]);
            double est = 2.0 * (double)(mbits - dist) / (double)mbits - 1.0;
            flag[k] = est > thr;
            nflag += flag[k];
        }
    }
    if (nflag) {
        uint8_t *alive = malloc(m);
        memset(alive, 1, m);
        for (int64_t k = 0; k < m; k++) {
            if (!flag[k]) continue;
            brute_force_point(c, acc, mem[k], mem, alive, m);
            alive[k] = 0;
        }
        free(alive);
    }
    int64_t ns = 0;
    for (int64_t k = 0; k < m; k++) if (!flag[k]) surv[ns++] = mem[k];
    free(flag);
    return ns;
}

typedef struct { int64_t *mem; int64_t m; int64_t depth; uint64_t seed; int64_t S; } Node;
typedef struct { Node *v; int64_t len, cap; } NodeVec;
static void nv_push(NodeVec *q, Node nd) {
    if (q->len == q->cap) { q->cap = q->cap ? 2 * q->cap : 64; q->v = realloc(q->v, q->cap * sizeof(Node)); }
    q->v[q->len++] = nd;
}

typedef struct { uint32_t v; int64_t idx; } VI;
static int cmp_vi(const void *a, const void *b) {
    const VI *x = a, *y = b;
    if (x->v != y->v) return x->v < y->v ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx);  /* stable */
}

typedef struct { int64_t *surv; VI *buf; int32_t *sel; } Scratch;

/* one node of _run_tree (cps:288-305): max_depth at pop, BruteForce step,
 * depth cap, then split_buckets (cps:222-245) appending the children to
 * `out` in the reference's order (position asc, value asc, groups >= 2)
 * with seeds mix64(seed ^ mix64(t + 64 ell + k)) (cps:301).  Frees nd.mem.
 * Returns the number of children appended. */
static int64_t process_node(const Ctx *c, Acc *acc, Node nd, Scratch *w, NodeVec *out) {
    if (nd.depth > acc->max_depth) acc->max_depth = nd.depth;
    int64_t ns = brute_force_step(c, acc, nd.mem, nd.m, nd.seed, w->surv);
    free(nd.mem);
    if (ns < 2) return 0;
    if (nd.depth >= c->depth_cap) {
        if (acc->n_cap_events == acc->cap_events_cap) {
            acc->cap_events_cap = acc->cap_events_cap ? 2 * acc->cap_events_cap : 16;
            acc->cap_events = realloc(acc->cap_events, acc->cap_events_cap * sizeof(int64_t));
        }
        acc->cap_events[acc->n_cap_events++] = ns;
        return 0;
    }
    double p_sel = 1.0 / (c->lam * (double)c->t);
    uint64_t child_off = (uint64_t)c->t + 64ULL * (uint64_t)c->ell;
    int32_t nsel = 0;
    for (int32_t i = 0; i < c->t; i++)
        if (stream_uniform(nd.seed, (uint64_t)i) < p_sel) w->sel[nsel++] = i;
    int64_t nchild = 0;
    for (int32_t s = 0; s < nsel; s++) {
        for (int64_t k = 0; k < ns; k++) {
            w->buf[k].v = c->values[w->surv[k] * c->t + w->sel[s]];
            w->buf[k].idx = k;
        }
        qsort(w->buf, ns, sizeof(VI), cmp_vi);
        int64_t g = 0;
        while (g < ns) {
            int64_t e = g + 1;
            while (e < ns && w->buf[e].v == w->buf[g].v) e++;
            if (e - g >= 2) {
                int64_t *cm = malloc((e - g) * sizeof(int64_t));
                for (int64_t k = g; k < e; k++) cm[k - g] = w->surv[w->buf[k].idx];
                nv_push(out, (Node){cm, e - g, nd.depth + 1, stream_word(nd.seed, child_off + (uint64_t)nchild), 0});
                nchild++;
            }
            g = e;
        }
    }
    return nchild;
}

static Scratch scratch_new(const Ctx *c) {
    Scratch w = {malloc((c->n ? c->n : 1) * sizeof(int64_t)), malloc((c->n ? c->n : 1) * sizeof(VI)),
                 malloc(c->t * sizeof(int32_t))};
    return w;
}
static void scratch_free(Scratch *w) { free(w->surv); free(w->buf); free(w->sel); }

/* depth-first run of the subtree below node `nd` (cps:278-305).  `base` is
 * the total size of the nodes below nd on the reference's stack when nd is
 * popped, so the stack totals (peak_live_members, cps:292-304) are the
 * reference's own. */
static void run_subtree(const Ctx *c, Acc *acc, Node nd, int64_t base, Scratch *w) {
    NodeVec stack = {0, 0, 0};
    nv_push(&stack, nd);
    int64_t stack_total = base + nd.m;
    if (stack_total > acc->peak) acc->peak = stack_total;
    while (stack.len) {
        Node top = stack.v[--stack.len];
        stack_total -= top.m;
        int64_t before = stack.len;
        int64_t nchild = process_node(c, acc, top, w, &stack);
        for (int64_t k = before; k < stack.len; k++) stack_total += stack.v[k].m;
        if (nchild && stack_total > acc->peak) acc->peak = stack_total;
    }
    free(stack.v);
}

/* one tree, depth first: cps:278-305 */
static void run_tree(const Ctx *c, Acc *acc, uint64_t tree_seed) {
    int64_t n = c->n;
    int64_t *root = malloc(n * sizeof(int64_t));
    for (int64_t i = 0; i < n; i++) root[i] = i;
    Scratch w = scratch_new(c);
    run_subtree(c, acc, (Node){root, n, 0, tree_seed, 0}, 0, &w);
    scratch_free(&w);
}

typedef struct { const Ctx *c; Acc *accs; const uint64_t *seeds; } TreeArgs;
static void tree_body(void *p, int64_t lo, int64_t hi, int tid) {
    TreeArgs *a = p;
    (void)tid;
    for (int64_t r = lo; r < hi; r++) run_tree(a->c, &a->accs[r], a->seeds[r]);
}

static int cmp_key(const void *a, const void *b) {
    uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
    return x < y ? -1 : (x > y);
}

typedef struct { uint64_t key; double sim; } KS;
static int cmp_ks(const void *a, const void *b) { return cmp_key(a, b); }

/* cpsjoin_self: cps:331-351, dedup cps:308-319.  Repetitions run on
 * separate threads; their accumulators merge by sum/max and the pair union
 * is sorted, so the output is independent of the thread count.
 * Returns 0, or 1 when a node-sketch pick fell out of range (the
 * reference raises IndexError there, cps:193). */
int orc_self_join_ct(const uint32_t *tok, const int64_t *off, const int64_t *sizes, int64_t n,
                     const uint32_t *values, int32_t t, const uint64_t *sketch, int32_t ell,
                     double lam, double eps, int32_t limit, int32_t kstar, int32_t depth_cap,
                     const uint64_t *rep_seeds, int32_t reps, int nthreads,
                     uint64_t **out_keys, double **out_sims, int64_t *out_n,
                     int64_t *counters /* pre, cand, res, max_depth, peak */,
                     int64_t **cap_events, int64_t *n_cap_events, int use_count_table);

int orc_self_join(const uint32_t *tok, const int64_t *off, const int64_t *sizes, int64_t n,
                  const uint32_t *values, int32_t t, const uint64_t *sketch, int32_t ell,
                  double lam, double eps, int32_t limit, int32_t kstar, int32_t depth_cap,
                  const uint64_t *rep_seeds, int32_t reps, int nthreads,
                  uint64_t **out_keys, double **out_sims, int64_t *out_n,
                  int64_t *counters, int64_t **cap_events, int64_t *n_cap_events) {
    return orc_self_join_ct(tok, off, sizes, n, values, t, sketch, ell, lam, eps, limit, kstar, depth_cap,
                            rep_seeds, reps, nthreads, out_keys, out_sims, out_n, counters, cap_events,
                            n_cap_events, 0);
}

/* merge per-repetition (or per-thread) accumulators: counters by sum/max,
 * the pair union sorted by key and deduplicated (cps:308-319).  An
 * accumulator with counted == 0 contributes its pairs, max_depth and peak
 * but not pre/cand/res or depth-cap events (the frontier mode's part above
 * the cut on ranks != 0). */
static int merge_accs(Acc *accs, const int *counted, int64_t nacc, uint64_t **out_keys, double **out_sims,
                      int64_t *out_n, int64_t *counters, int64_t **cap_events, int64_t *n_cap_events) {
    int64_t total = 0, nev = 0;
    for (int64_t r = 0; r < nacc; r++) {
        total += accs[r].len;
        if (!counted || counted[r]) nev += accs[r].n_cap_events;
    }
    KS *ks = malloc((total ? total : 1) * sizeof(KS));
    int64_t *ev = malloc((nev ? nev : 1) * sizeof(int64_t));
    int64_t k = 0, e = 0;
    int err = 0;
    memset(counters, 0, 5 * sizeof(int64_t));
    for (int64_t r = 0; r < nacc; r++) {
        Acc *a = &accs[r];
        for (int64_t i = 0; i < a->len; i++) {
            uint64_t lo = (uint64_t)(a->a[i] < a->b[i] ? a->a[i] : a->b[i]);
            uint64_t hi = (uint64_t)(a->a[i] < a->b[i] ? a->b[i] : a->a[i]);
            ks[k].key = (lo << 32) | hi;
            ks[k].sim = a->sim[i];
            k++;
        }
        if (!counted || counted[r]) {
            for (int64_t i = 0; i < a->n_cap_events; i++) ev[e++] = a->cap_events[i];
            counters[0] += a->pre; counters[1] += a->cand; counters[2] += a->res;
        }
        if (a->max_depth > counters[3]) counters[3] = a->max_depth;
        if (a->peak > counters[4]) counters[4] = a->peak;
        err |= a->error;
        free(a->a); free(a->b); free(a->sim); free(a->cap_events);
    }
    qsort(ks, total, sizeof(KS), cmp_ks);
    int64_t u = 0;
    for (int64_t i = 0; i < total; i++)
        if (u == 0 || ks[u - 1].key != ks[i].key) ks[u++] = ks[i];
    uint64_t *keys = malloc((u ? u : 1) * sizeof(uint64_t));
    double *sims = malloc((u ? u : 1) * sizeof(double));
    for (int64_t i = 0; i < u; i++) { keys[i] = ks[i].key; sims[i] = ks[i].sim; }
    free(ks);
    *out_keys = keys; *out_sims = sims; *out_n = u;
    *cap_events = ev; *n_cap_events = nev;
    return err;
}

int orc_self_join_ct(const uint32_t *tok, const int64_t *off, const int64_t *sizes, int64_t n,
                     const uint32_t *values, int32_t t, const uint64_t *sketch, int32_t ell,
                     double lam, double eps, int32_t limit, int32_t kstar, int32_t depth_cap,
                     const uint64_t *rep_seeds, int32_t reps, int nthreads,
                     uint64_t **out_keys, double **out_sims, int64_t *out_n,
                     int64_t *counters /* pre, cand, res, max_depth, peak */,
                     int64_t **cap_events, int64_t *n_cap_events, int use_count_table) {
    Ctx c = {tok, off, sizes, n, values, t, sketch, ell, lam, eps, limit, kstar, depth_cap, use_count_table};
    Acc *accs = calloc(reps > 0 ? reps : 1, sizeof(Acc));
    if (n >= 2) {
        TreeArgs ta = {&c, accs, rep_seeds};
        parallel_for(reps, 1, nthreads, tree_body, &ta);
    }
    int err = merge_accs(accs, NULL, reps, out_keys, out_sims, out_n, counters, cap_events, n_cap_events);
    free(accs);
    return err;
}

/* Frontier sharding (the B200 library's cpsj_plan.frontier_*; SURVEY 8(e);
 * not a reference feature -- its contract is that the union over ranks is
 * cpsjoin_self, cps:331-351).  Every rank expands all repetition trees
 * breadth-first down to depth `fdepth` (level order: repetitions in order,
 * children in parent order, each parent's children in the reference's
 * order), then keeps its share of that level -- node i belongs to rank
 * floor(ranks (2 C_i + c_i) / (2 C_N)), c = m + m (m - 1) / 64 for a leaf
 * (m <= limit), m * bit_length(m) otherwise, C_i the cost of nodes before i
 * -- and runs the kept subtrees depth first with their reference stack
 * base S (S(child_j) = S(parent) + sizes of children before j).  Rank 0
 * reports the counters and pairs of the part above the cut; every rank
 * reports the pairs and counters of its kept subtrees, the cut depth as
 * reached, and the stack peak of what it expanded. */
typedef struct { const Ctx *c; Acc *accs; Node *nodes; const int64_t *kept; Scratch *w; } KeptArgs;
static void kept_body(void *p, int64_t lo, int64_t hi, int tid) {
    KeptArgs *a = p;
    for (int64_t i = lo; i < hi; i++) {
        Node nd = a->nodes[a->kept[i]];
        run_subtree(a->c, &a->accs[tid], nd, nd.S, &a->w[tid]);
    }
}

static int64_t frontier_cost(int64_t m, int32_t limit) {
    if (m <= limit) return m + m * (m - 1) / 64;
    int64_t b = 0;
    while ((m >> b) != 0) ++b;
    return m * b;
}

int orc_self_join_frontier(const uint32_t *tok, const int64_t *off, const int64_t *sizes, int64_t n,
                           const uint32_t *values, int32_t t, const uint64_t *sketch, int32_t ell,
                           double lam, double eps, int32_t limit, int32_t kstar, int32_t depth_cap,
                           const uint64_t *rep_seeds, int32_t reps, int nthreads,
                           int32_t rank, int32_t ranks, int32_t fdepth,
                           uint64_t **out_keys, double **out_sims, int64_t *out_n,
                           int64_t *counters, int64_t **cap_events, int64_t *n_cap_events) {
    Ctx c = {tok, off, sizes, n, values, t, sketch, ell, lam, eps, limit, kstar, depth_cap, 0};
    int nt = resolve_threads(nthreads);
    Acc *accs = calloc(nt + 1, sizeof(Acc));   /* [0] = above the cut, [1 + tid] = kept subtrees */
    int *counted = calloc(nt + 1, sizeof(int));
    counted[0] = rank == 0;
    for (int i = 1; i <= nt; i++) counted[i] = 1;
    if (n >= 2 && reps > 0) {
        Acc *top = &accs[0];
        top->peak = n;
        Scratch w = scratch_new(&c);
        NodeVec level = {0, 0, 0};
        for (int32_t r = 0; r < reps; r++) {
            int64_t *root = malloc(n * sizeof(int64_t));
            for (int64_t i = 0; i < n; i++) root[i] = i;
            nv_push(&level, (Node){root, n, 0, rep_seeds[r], 0});
        }
        for (int32_t d = 0; d < fdepth && level.len; d++) {
            NodeVec next = {0, 0, 0};
            for (int64_t i = 0; i < level.len; i++) {
                Node nd = level.v[i];
                int64_t before = next.len;
                int64_t nchild = process_node(&c, top, nd, &w, &next);
                int64_t S = nd.S;
                for (int64_t k = before; k < next.len; k++) { next.v[k].S = S; S += next.v[k].m; }
                if (nchild && S > top->peak) top->peak = S;
            }
            free(level.v);
            level = next;
        }
        scratch_free(&w);
        if (level.len) {
            if (fdepth > top->max_depth) top->max_depth = fdepth;
            int64_t total = 0;
            for (int64_t i = 0; i < level.len; i++) total += frontier_cost(level.v[i].m, limit);
            int64_t *kept = malloc(level.len * sizeof(int64_t));
            int64_t nk = 0, before = 0;
            for (int64_t i = 0; i < level.len; i++) {
                int64_t cst = frontier_cost(level.v[i].m, limit);
                __int128 num = (__int128)ranks * (__int128)(2 * before + cst);
                int64_t owner = (int64_t)(num / (__int128)(2 * total));
                if (owner == rank) kept[nk++] = i;
                else free(level.v[i].mem);
                before += cst;
            }
            Scratch *ws = malloc(nt * sizeof(Scratch));
            for (int i = 0; i < nt; i++) ws[i] = scratch_new(&c);
            KeptArgs ka = {&c, accs + 1, level.v, kept, ws};
            parallel_for(nk, 1, nt, kept_body, &ka);
            for (int i = 0; i < nt; i++) scratch_free(&ws[i]);
            free(ws);
            free(kept);
        }
        if (rank != 0) top->len = 0;  /* pairs above the cut: rank 0 reports them */
        free(level.v);
    }
    int err = merge_accs(accs, counted, nt + 1, out_keys, out_sims, out_n, counters, cap_events, n_cap_events);
    free(accs);
    free(counted);
    return err;
}

void orc_free(void *p) { free(p); }

/* Exact all-pairs join (recall ground truth, not part of the reference:
 * SPEC.md:440-509 specifies AllPairs but it is not shipped).  Every pair with
 * |x n y| / |x u y| >= lam by prefix filtering: order tokens by ascending
 * frequency; a pair with J >= lam overlaps in >= ceil(lam*|x|) tokens, so
 * it shares a token inside both prefixes of length |x| - ceil(lam*|x|) + 1.
 * The prefix is taken one token longer than necessary at exact integer
 * boundaries, which only adds candidates.  Candidates are verified by
 * merge intersection on the original rows and sim = inter / union. */
typedef struct { uint32_t r; uint32_t tok; } RT;
static int cmp_rt(const void *a, const void *b) {
    const RT *x = a, *y = b;
    return x->r < y->r ? -1 : (x->r > y->r);
}

typedef struct {
    const uint32_t *tok; const int64_t *off; const uint32_t *pre; const int64_t *poff;
    const int64_t *ioff; const int64_t *rows; double lam; Acc *accs; int64_t **marks;
} ExArgs;

static void exact_body(void *p, int64_t lo, int64_t hi, int tid) {
    ExArgs *a = p;
    Acc *acc = &a->accs[tid];
    int64_t *mark = a->marks[tid];
    const uint32_t *tok = a->tok;
    const int64_t *off = a->off;
    double lam = a->lam;
    for (int64_t x = lo; x < hi; x++) {
        int64_t sx = off[x + 1] - off[x];
        for (int64_t i = a->poff[x]; i < a->poff[x + 1]; i++) {
            uint32_t v = a->pre[i];
            for (int64_t k = a->ioff[v]; k < a->ioff[v + 1]; k++) {
                int64_t y = a->rows[k];
                if (y >= x) break;
                if (mark[y] == x) continue;
                mark[y] = x;
                int64_t sy = off[y + 1] - off[y];
                int64_t mn = sx < sy ? sx : sy, mx = sx < sy ? sy : sx;
                if ((double)mn < lam * (double)mx - 1e-9) continue;
                const uint32_t *p1 = tok + off[y], *pe = tok + off[y + 1];
                const uint32_t *q = tok + off[x], *qe = tok + off[x + 1];
                int64_t inter = 0;
                while (p1 < pe && q < qe) {
                    if (*p1 == *q) { inter++; p1++; q++; }
                    else if (*p1 < *q) p1++;
                    else q++;
                }
                double sim = (double)inter / (double)(sx + sy - inter);
                if (sim >= lam) acc_push(acc, y, x, sim);
            }
        }
    }
}

int orc_exact_join(const uint32_t *tok, const int64_t *off, int64_t n, uint32_t d, double lam,
                   int nthreads, uint64_t **out_keys, double **out_sims, int64_t *out_n) {
    int64_t nnz = off[n];
    int64_t *cnt = calloc((size_t)d + 1, sizeof(int64_t));
    for (int64_t i = 0; i < nnz; i++) cnt[tok[i]]++;
    uint64_t *order = malloc(((size_t)d ? d : 1) * sizeof(uint64_t));
    for (uint32_t v = 0; v < d; v++) order[v] = ((uint64_t)cnt[v] << 32) | v;
    qsort(order, d, sizeof(uint64_t), cmp_key);
    uint32_t *rank = malloc(((size_t)d ? d : 1) * sizeof(uint32_t));
    for (uint32_t i = 0; i < d; i++) rank[(uint32_t)(order[i] & 0xFFFFFFFFu)] = i;
    free(order);
    /* prefix (by rank) of every set */
    int64_t *plen = malloc((n ? n : 1) * sizeof(int64_t));
    int64_t *poff = malloc((n + 1) * sizeof(int64_t));
    poff[0] = 0;
    for (int64_t r = 0; r < n; r++) {
        int64_t len = off[r + 1] - off[r];
        int64_t omin = (int64_t)__builtin_ceil(lam * (double)len - 1e-9);
        int64_t p = len - omin + 1;
        if (p > len) p = len;
        if (p < 1) p = len > 0 ? 1 : 0;
        plen[r] = p;
        poff[r + 1] = poff[r] + p;
    }
    uint32_t *pre = malloc((poff[n] ? poff[n] : 1) * sizeof(uint32_t));
    {
        RT *tmp = malloc(64 * sizeof(RT));
        int64_t tcap = 64;
        for (int64_t r = 0; r < n; r++) {
            int64_t len = off[r + 1] - off[r];
            if (len > tcap) { tcap = len; tmp = realloc(tmp, tcap * sizeof(RT)); }
            for (int64_t i = 0; i < len; i++) { tmp[i].tok = tok[off[r] + i]; tmp[i].r = rank[tok[off[r] + i]]; }
            qsort(tmp, len, sizeof(RT), cmp_rt);
            for (int64_t i = 0; i < plen[r]; i++) pre[poff[r] + i] = tmp[i].tok;
        }
        free(tmp);
    }
    free(rank);
    /* inverted index over prefixes: token -> rows (ascending) */
    int64_t *ioff = calloc((size_t)d + 1, sizeof(int64_t));
    for (int64_t i = 0; i < poff[n]; i++) ioff[pre[i] + 1]++;
    for (uint32_t v = 0; v < d; v++) ioff[v + 1] += ioff[v];
    int64_t *fill = malloc(((size_t)d ? d : 1) * sizeof(int64_t));
    memcpy(fill, ioff, (size_t)d * sizeof(int64_t));
    int64_t *rows = malloc((poff[n] ? poff[n] : 1) * sizeof(int64_t));
    for (int64_t r = 0; r < n; r++)
        for (int64_t i = poff[r]; i < poff[r + 1]; i++) rows[fill[pre[i]]++] = r;
    free(fill); free(cnt);
    int nt = resolve_threads(nthreads);
    Acc *accs = calloc(nt, sizeof(Acc));
    int64_t **marks = calloc(nt, sizeof(int64_t *));
    for (int i = 0; i < nt; i++) {
        marks[i] = malloc((n ? n : 1) * sizeof(int64_t));
        for (int64_t j = 0; j < n; j++) marks[i][j] = -1;
    }
    ExArgs ea = {tok, off, pre, poff, ioff, rows, lam, accs, marks};
    parallel_for(n, 256, nt, exact_body, &ea);
    for (int i = 0; i < nt; i++) free(marks[i]);
    free(marks);
    int64_t total = 0;
    for (int i = 0; i < nt; i++) total += accs[i].len;
    KS *ks = malloc((total ? total : 1) * sizeof(KS));
    int64_t k = 0;
    for (int i = 0; i < nt; i++) {
        for (int64_t j = 0; j < accs[i].len; j++) {
            ks[k].key = ((uint64_t)accs[i].a[j] << 32) | (uint64_t)accs[i].b[j];
            ks[k].sim = accs[i].sim[j];
            k++;
        }
        free(accs[i].a); free(accs[i].b); free(accs[i].sim);
    }
    free(accs);
    qsort(ks, total, sizeof(KS), cmp_ks);
    uint64_t *keys = malloc((total ? total : 1) * sizeof(uint64_t));
    double *sims = malloc((total ? total : 1) * sizeof(double));
    for (int64_t i = 0; i < total; i++) { keys[i] = ks[i].key; sims[i] = ks[i].sim; }
    free(ks); free(pre); free(poff); free(plen); free(ioff); free(rows);
    *out_keys = keys; *out_sims = sims; *out_n = total;
    return 0;
}
