/*
 * oracle/gbs_oracle.c -- CPU ORACLE for GPU Bucket Sort
 *                        (Dehne & Zaboli, "Deterministic Sample Sort For GPUs",
 *                         arXiv 1002.4464; Algorithm 1).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / `--impl reference` leg may load this library.  The product path
 * (paper_1002_4464_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or constant generator with it.
 *
 * Plain, slow, single-threaded C.  Every function follows one step of Algorithm 1
 * in the paper's order and notation; library primitives used as steps: qsort
 * (a sort) and a binary search over a strictly increasing array (a count).
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n.
 * Readings "Rk" of places where the paper is silent/ambiguous are listed in
 * DESIGN.md section 3 (R1 item width, R2 equidistant index, R3 duplicate keys via
 * implicit tags, R4 bucket boundary rule, R5 scan order, R8 tail padding, ...).
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute force against a naive sort on
 * every input of length <= 8 over {0,1,2,0xFFFFFFFF}; the tight bucket-size
 * bound (attained, never exceeded); the closed form |B_j| = n/s for all-equal and
 * sorted inputs; conservation of counts; the paper's worked parameters
 * (P:249-259, 269-274, 318-319); SPEC per-operation examples (S:105, S:132,
 * S:141); stability with 90% duplicates; PSRS output vs a naive sort.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define O_SENTINEL_KEY 0xFFFFFFFFu

/* An item of a problem: key, optional value, and its position in the problem's
 * input order.  (key, pos) is a strict total order (R3). */
typedef struct {
    uint32_t key;
    uint32_t val;
    uint64_t pos;
} oitem_t;

/* Level-1 intermediates, for stage parity (all optional; NULL = not recorded). */
typedef struct {
    uint32_t *sorted_keys;    /* n:      A after Step 2 (sorted sublists, in place)     */
    uint64_t *samples;        /* m*s:    Step 3 local samples, (key<<32)|tag            */
    uint64_t *sorted_samples; /* m*s:    Step 4                                          */
    uint64_t *splitters;      /* s:      Step 5 global samples g_0..g_{s-1}              */
    uint32_t *a;              /* m*s:    Step 6 bucket sizes a_ij (real items), [i*s+j] */
    uint32_t *l;              /* m*s:    Step 7 offsets l_ij, [i*s+j]                     */
    uint32_t *relocated;      /* n:      Step 8 array R = B_1 ... B_s                    */
    uint64_t *bucket_total;   /* s:      |B_j| counting the virtual sentinels (R8)       */
} oracle_trace_t;

/* ---------------------------------------------------------------- helpers */

static int cmp_key_pos(const void *x, const void *y)
{
    const oitem_t *a = (const oitem_t *)x, *b = (const oitem_t *)y;
    if (a->key != b->key) return a->key < b->key ? -1 : 1;
    if (a->pos != b->pos) return a->pos < b->pos ? -1 : 1;
    return 0;
}

static int cmp_u64(const void *x, const void *y)
{
    uint64_t a = *(const uint64_t *)x, b = *(const uint64_t *)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* Composite (key, tag) as one unsigned 64-bit number: lexicographic order on
 * (key, tag) equals numeric order because tag < 2^32 (R3, R12). */
static uint64_t composite(uint32_t key, uint64_t tag) { return ((uint64_t)key << 32) | tag; }

/* Stable sort by key: sort by (key, pos) with pos = current index.  The order is
 * total, so the result is unique and equals std::stable_sort (R7). */
static void stable_sort_by_key(oitem_t *x, uint64_t len)
{
    for (uint64_t q = 0; q < len; ++q) x[q].pos = q;
    if (len > 1) qsort(x, (size_t)len, sizeof(oitem_t), cmp_key_pos);
}

/* ------------------------------------------------------- bound arithmetic */

/* Tight bucket-size bound of one level (implies P:318-319's
 * |B_j| <= 2n/s).  n' = m*L items (real + virtual sentinels), d = L/s:
 *   j <  s-1 :  n'/s - (m-1)(d-1) <= |B_j| <= n'/s + (m-1)(d-1)
 *   j == s-1 :  |B_{s-1}| <= n'/s
 * Derivation: let c_i = #samples of A_i that are <= g_j; sum_i c_i = (j+1)m and
 * #items of A_i <= g_j lies in [c_i d, c_i d + d - 1], with exactly c_i d for the
 * sublist that owns g_j. */
void oracle_bucket_bound(uint64_t cap, uint32_t L, uint32_t s,
                         uint64_t *m_out, uint64_t *np_out,
                         uint64_t *hi_out, uint64_t *lo_out, uint64_t *last_out)
{
    uint64_t m = (cap + L - 1) / L, np = m * L, d = L / s;
    uint64_t slack = (m - 1) * (d - 1);
    if (m_out) *m_out = m;
    if (np_out) *np_out = np;
    if (hi_out) *hi_out = np / s + slack;
    if (lo_out) *lo_out = (np / s > slack) ? np / s - slack : 0;
    if (last_out) *last_out = np / s;
}

/* ------------------------------------------------------------ the steps */

/* Step 1 + Step 2: split the problem of capacity `cap`
 * into m = ceil(cap/L) sublists of L items; positions len..mL-1 are virtual
 * sentinels with key 0xFFFFFFFF and pos = position (R8), so they follow
 * every real item in (key, pos) order.  Each sublist is sorted locally; after the
 * sort, tag(i, r) = iL + r (R3). */
static void step1_2_split_local_sort(oitem_t *A, const oitem_t *X, uint64_t len,
                                     uint64_t m, uint32_t L)
{
    uint64_t np = m * L;
    for (uint64_t p = 0; p < np; ++p) {
        if (p < len) { A[p] = X[p]; A[p].pos = p; }
        else { A[p].key = O_SENTINEL_KEY; A[p].val = 0; A[p].pos = p; }
    }
    for (uint64_t i = 0; i < m; ++i)
        qsort(A + i * L, L, sizeof(oitem_t), cmp_key_pos);
}

/* Step 3: s equidistant samples of each sorted sublist:
 * the last element of each of s segments of d = L/s items, i.e. sorted positions
 * (k+1)d - 1 (R2), kept as composites (key, tag = iL + (k+1)d - 1). */
void oracle_local_samples(const uint32_t *sorted_keys, uint64_t tag0, uint32_t L,
                          uint32_t s, uint64_t *out)
{
    uint32_t d = L / s;
    for (uint32_t k = 0; k < s; ++k) {
        uint32_t r = (k + 1) * d - 1;
        out[k] = composite(sorted_keys[r], tag0 + r);
    }
}

/* Step 4: sort all s*m samples (composites are distinct). */
static void step4_sort_samples(uint64_t *S, uint64_t count)
{
    qsort(S, (size_t)count, sizeof(uint64_t), cmp_u64);
}

/* Step 5: s equidistant global samples g_k = sorted[(k+1)m - 1]
 * (same segment-end convention as Step 3, R2).  g_{s-1} is the maximum of
 * all samples, hence of all items: exactly s buckets exist. */
void oracle_global_samples(const uint64_t *sorted, uint64_t m, uint32_t s, uint64_t *g)
{
    for (uint32_t k = 0; k < s; ++k) g[k] = sorted[(uint64_t)(k + 1) * m - 1];
}

/* Number of r in [0, L) with composite(keys[r], tag0 + r) <= g.  In a sorted
 * sublist that composite is strictly increasing in r, so the count is the
 * partition point (found by bisection; tests pin it with a linear count). */
static uint64_t count_le(const uint32_t *keys, uint64_t tag0, uint64_t L, uint64_t g)
{
    uint64_t lo = 0, hi = L;
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (composite(keys[mid], tag0 + mid) <= g) lo = mid + 1; else hi = mid;
    }
    return lo;
}

/* Step 6: locate every global sample in sorted sublist
 * A_i.  Bucket j of A_i holds the items x with g_{j-1} < x <= g_j in (key, tag)
 * order (R4).  P_ij = #{r : (A_i[r], iL+r) <= g_j}; since the sentinels
 * are the largest items of A_i, the real items of bucket j are the first
 * v_i = #real items of A_i: Q_ij = min(P_ij, v_i) and a_ij = Q_ij - Q_i,j-1. */
void oracle_sample_index(const uint32_t *sorted_keys, uint64_t tag0, uint32_t L,
                         uint32_t valid, const uint64_t *g, uint32_t s,
                         uint32_t *a_row, uint64_t *total_row /* nullable */)
{
    uint64_t prevQ = 0, prevP = 0;
    for (uint32_t j = 0; j < s; ++j) {
        uint64_t P = count_le(sorted_keys, tag0, L, g[j]);
        uint64_t Q = P < valid ? P : valid;
        a_row[j] = (uint32_t)(Q - prevQ);
        if (total_row) total_row[j] = P - prevP;
        prevQ = Q; prevP = P;
    }
}

/* Step 7: l_ij = starting location of bucket A_ij in the
 * final sequence = exclusive prefix sum of a in the order a_11..a_m1, a_12, ...
 * (column-major, R5).  Matrices are stored row-major [i*s + j]. */
void oracle_offsets(const uint32_t *a, uint64_t m, uint32_t s, uint32_t *l)
{
    uint64_t run = 0;
    for (uint32_t j = 0; j < s; ++j)
        for (uint64_t i = 0; i < m; ++i) {
            l[i * s + j] = (uint32_t)run;
            run += a[i * s + j];
        }
}

/* ------------------------------------------------------ one GBS problem */

/* Algorithm 1 on one problem X[0..len) with static capacity cap >= len,
 * plan levels (Ls[0], ss[0]), (Ls[1], ss[1]), ...; nlev == 0 means a single
 * local sort.  Returns 0, or -1 (allocation), -3 (bound violated). */
static int gbs_problem(oitem_t *X, uint64_t len, uint64_t cap, const uint32_t *Ls,
                       const uint32_t *ss, int nlev, oracle_trace_t *tr)
{
    if (len <= 1) return 0;
    if (nlev == 0) { stable_sort_by_key(X, len); return 0; }

    const uint32_t L = Ls[0], s = ss[0];
    uint64_t m, np, hi;
    oracle_bucket_bound(cap, L, s, &m, &np, &hi, NULL, NULL);
    const uint64_t ms = m * s;

    int rc = -1;
    oitem_t *A = malloc(np * sizeof(oitem_t));
    uint32_t *Akeys = malloc(np * sizeof(uint32_t));
    uint64_t *S = malloc(ms * sizeof(uint64_t));
    uint64_t *g = malloc((size_t)s * sizeof(uint64_t));
    uint32_t *a = malloc(ms * sizeof(uint32_t));
    uint32_t *l = malloc(ms * sizeof(uint32_t));
    uint64_t *tot = calloc(s, sizeof(uint64_t));
    uint64_t *row_tot = malloc((size_t)s * sizeof(uint64_t));
    oitem_t *R = malloc((len ? len : 1) * sizeof(oitem_t));
    if (!A || !Akeys || !S || !g || !a || !l || !tot || !row_tot || !R) goto out;

    /* Steps 1-2 */
    step1_2_split_local_sort(A, X, len, m, L);
    for (uint64_t p = 0; p < np; ++p) Akeys[p] = A[p].key;
    if (tr && tr->sorted_keys) for (uint64_t p = 0; p < len; ++p) tr->sorted_keys[p] = Akeys[p];

    /* Step 3 */
    for (uint64_t i = 0; i < m; ++i) oracle_local_samples(Akeys + i * L, i * L, L, s, S + i * s);
    if (tr && tr->samples) memcpy(tr->samples, S, ms * sizeof(uint64_t));

    /* Step 4 */
    step4_sort_samples(S, ms);
    if (tr && tr->sorted_samples) memcpy(tr->sorted_samples, S, ms * sizeof(uint64_t));

    /* Step 5 */
    oracle_global_samples(S, m, s, g);
    if (tr && tr->splitters) memcpy(tr->splitters, g, (size_t)s * sizeof(uint64_t));

    /* Step 6 */
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t v = len > i * L ? len - i * L : 0;
        if (v > L) v = L;
        oracle_sample_index(Akeys + i * L, i * L, L, (uint32_t)v, g, s, a + i * s, row_tot);
        for (uint32_t j = 0; j < s; ++j) tot[j] += row_tot[j];
    }
    if (tr && tr->a) memcpy(tr->a, a, ms * sizeof(uint32_t));
    if (tr && tr->bucket_total) memcpy(tr->bucket_total, tot, (size_t)s * sizeof(uint64_t));

    /* Step 7 */
    oracle_offsets(a, m, s, l);
    if (tr && tr->l) memcpy(tr->l, l, ms * sizeof(uint32_t));

    /* Step 8: move bucket A_ij to l_ij; R = B_1 ... B_s. */
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t start = 0;
        for (uint32_t j = 0; j < s; ++j) {
            uint32_t cnt = a[i * s + j];
            for (uint32_t q = 0; q < cnt; ++q) R[l[i * s + j] + q] = A[i * L + start + q];
            start += cnt;
        }
    }
    if (tr && tr->relocated) for (uint64_t p = 0; p < len; ++p) tr->relocated[p] = R[p].key;

    /* Step 9: sort every B_j.  The ties inside B_j are in
     * tag order already, so a stable sort by key gives the global (key, tag)
     * order.  With a nested level, B_j is a problem of capacity hi (R9). */
    for (uint32_t j = 0; j < s; ++j) {
        uint64_t b0 = l[j];                       /* l_0j: row 0, column j */
        uint64_t b1 = (j + 1 < s) ? l[j + 1] : len;
        if (tot[j] > hi) { rc = -3; goto out; }
        rc = gbs_problem(R + b0, b1 - b0, hi, Ls + 1, ss + 1, nlev - 1, NULL);
        if (rc) goto out;
    }
    /* Output (Alg. 1: "Array A sorted", in place). */
    for (uint64_t p = 0; p < len; ++p) X[p] = R[p];
    rc = 0;
out:
    free(A); free(Akeys); free(S); free(g); free(a); free(l); free(tot); free(row_tot); free(R);
    return rc;
}

static int plan_ok(const uint32_t *Ls, const uint32_t *ss, int nlev)
{
    for (int k = 0; k < nlev; ++k) {
        uint32_t L = Ls[k], s = ss[k];
        if (L < 1 || s < 1 || s > L || (L & (L - 1)) || (s & (s - 1))) return 0;
    }
    return nlev >= 0 && nlev <= 4;
}

/* ------------------------------------------------------------ entry points */

/* Sort keys (and, if vals != NULL, their values, stable by key) in place with the
 * given plan.  n <= 2^31 (tags are 32-bit, R10).  Returns 0 / -1 / -2 / -3. */
int oracle_gbs_sort(uint32_t *keys, uint32_t *vals, uint64_t n, const uint32_t *Ls,
                    const uint32_t *ss, int nlev, oracle_trace_t *tr)
{
    if (!plan_ok(Ls, ss, nlev)) return -2;
    if (n > (1ull << 31)) return -2;
    if (n == 0) return 0;
    oitem_t *X = malloc(n * sizeof(oitem_t));
    if (!X) return -1;
    for (uint64_t p = 0; p < n; ++p) { X[p].key = keys[p]; X[p].val = vals ? vals[p] : 0; X[p].pos = p; }
    int rc = gbs_problem(X, n, n, Ls, ss, nlev, tr);
    if (rc == 0)
        for (uint64_t p = 0; p < n; ++p) { keys[p] = X[p].key; if (vals) vals[p] = X[p].val; }
    free(X);
    return rc;
}

/* Brute-force helper: `rows` independent problems of n keys each (row-major). */
int oracle_gbs_sort_batch(uint32_t *keys, uint64_t rows, uint64_t n, const uint32_t *Ls,
                          const uint32_t *ss, int nlev)
{
    for (uint64_t r = 0; r < rows; ++r) {
        int rc = oracle_gbs_sort(keys + r * n, NULL, n, Ls, ss, nlev, NULL);
        if (rc) return rc;
    }
    return 0;
}

/* Multi-GPU outer level (not in the paper, R15): Alg. 1 with
 * one sublist per rank.  E1 sort each shard; E2 s_r regular samples per rank at
 * positions (k+1) n_l / s_r - 1 tagged with the global position r n_l + pos;
 * E4 sort all p s_r samples; E5 splitters G_k = sorted[(k+1) s_r - 1];
 * E6 cut_{r,k} = #{pos : (S_r[pos], r n_l + pos) <= G_k}; E8 rank k receives
 * S_r[cut_{r,k-1}, cut_{r,k}) from every r in rank order; E9 rank k sorts what it
 * received (stable).  out = concatenation of the rank outputs in rank order;
 * counts[k] = |out_k|; cuts[r*p + k] = cut_{r,k}. */
int oracle_psrs(const uint32_t *keys, uint64_t n_local, int p, uint32_t s_r,
                uint32_t *out, uint64_t *counts, uint64_t *cuts)
{
    if (p < 1 || s_r < 1 || s_r > n_local || n_local >= (1ull << 32) ||
        (uint64_t)p * n_local > (1ull << 32)) return -2;
    const uint64_t N = (uint64_t)p * n_local;
    int rc = -1;
    oitem_t *sh = malloc(N * sizeof(oitem_t));
    uint32_t *shk = malloc(N * sizeof(uint32_t));
    uint64_t *S = malloc((uint64_t)p * s_r * sizeof(uint64_t));
    uint64_t *G = malloc((uint64_t)p * sizeof(uint64_t));
    oitem_t *recv = malloc(N * sizeof(oitem_t));
    if (!sh || !shk || !S || !G || !recv) goto out;

    for (int r = 0; r < p; ++r) {                                   /* E1 */
        oitem_t *x = sh + (uint64_t)r * n_local;
        for (uint64_t q = 0; q < n_local; ++q) x[q].key = keys[(uint64_t)r * n_local + q];
        stable_sort_by_key(x, n_local);
        for (uint64_t q = 0; q < n_local; ++q) shk[(uint64_t)r * n_local + q] = x[q].key;
        for (uint32_t k = 0; k < s_r; ++k) {                        /* E2 */
            uint64_t pos = (uint64_t)(k + 1) * n_local / s_r - 1;
            S[(uint64_t)r * s_r + k] = composite(x[pos].key, (uint64_t)r * n_local + pos);
        }
    }
    qsort(S, (size_t)p * s_r, sizeof(uint64_t), cmp_u64);         /* E4 */
    for (int k = 0; k < p; ++k) G[k] = S[(uint64_t)(k + 1) * s_r - 1]; /* E5 */
    for (int r = 0; r < p; ++r)                                     /* E6 */
        for (int k = 0; k < p; ++k)
            cuts[r * p + k] = count_le(shk + (uint64_t)r * n_local, (uint64_t)r * n_local,
                                       n_local, G[k]);
    uint64_t o = 0;
    for (int k = 0; k < p; ++k) {                                   /* E8 + E9 */
        uint64_t c = 0;
        for (int r = 0; r < p; ++r) {
            uint64_t lo = k ? cuts[r * p + k - 1] : 0, hi = cuts[r * p + k];
            for (uint64_t q = lo; q < hi; ++q) recv[c++] = sh[(uint64_t)r * n_local + q];
        }
        stable_sort_by_key(recv, c);
        for (uint64_t q = 0; q < c; ++q) out[o + q] = recv[q].key;
        counts[k] = c;
        o += c;
    }
    rc = (o == N) ? 0 : -3;
out:
    free(sh); free(shk); free(S); free(G); free(recv);
    return rc;
}
