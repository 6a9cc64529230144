/*
 * ORACLE -- test infrastructure only.  Not part of the product path.
 *
 * A plain-C, float64 restatement of the reference's two-stage MP-WSD hot path
 * (/root/reference/pkg/src/feclab/decoders.py), used as the checker by tests/,
 * by __graft_entry__.smoke() and as bench.py's CPU baseline.  Nothing in
 * paper_2602_08501_b200/ links or calls this file.
 *
 * Each function cites the reference lines it restates.  Parity pins: the
 * golden vectors in tests/golden/ were produced by the reference itself
 * (tests/golden/make_golden.py); tests/test_oracle_golden.py checks this
 * restatement against them.
 *
 * Bit layout: bit j of a vector is bit (j % 64) of uint64 word j / 64
 * (binlin.py:1-8).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int n, k, kp, w64;
    const int32_t *info_set;   /* kp, ascending */
    const uint64_t *gen;       /* k x w64: effective generator */
    int is_ca;                 /* 1: CRC-concatenated polar (gate + projection) */
    int crc_deg;
    uint32_t crc_poly;         /* bit i = coefficient of x^i */
} orc_code_t;

typedef struct {
    int size;                  /* members including the zero codeword */
    const uint64_t *members;   /* size x w64, zero first */
    int filter_m;              /* resolved filter size m (decoders.py:88-96) */
} orc_sphere_t;

typedef struct {
    int list_size;             /* L */
    int num_paths;             /* A */
    int max_iter;              /* T */
    int gated;                 /* activation_mode == crc_gated */
    int osd_order;             /* >= 0: OsdStage(order, cap) instead of SclStage(L) */
    int osd_cap;               /* list_cap, <= 0: None */
} orc_params_t;

static inline int getbit(const uint64_t *w, int j) { return (int)((w[j >> 6] >> (j & 63)) & 1u); }
static inline void setbit(uint64_t *w, int j, int b) {
    if (b) w[j >> 6] |= (1ull << (j & 63)); else w[j >> 6] &= ~(1ull << (j & 63));
}

/* polar_transform_bits (codebook.py:166-178): first half ^= second half at every scale */
static void polar_transform_u8(uint8_t *b, int n) {
    for (int h = 1; h < n; h *= 2)
        for (int blk = 0; blk < n; blk += 2 * h)
            for (int i = 0; i < h; i++) b[blk + i] ^= b[blk + h + i];
}

/* crc_check (codebook.py:154-163): v read MSB-first divisible by g(x) */
static int crc_ok(const uint8_t *v, int len, int deg, uint32_t poly) {
    uint8_t buf[1024];
    memcpy(buf, v, (size_t)len);
    for (int i = 0; i < len - deg; i++)
        if (buf[i])
            for (int j = 0; j <= deg; j++) buf[i + j] ^= (uint8_t)((poly >> (deg - j)) & 1u);
    for (int i = len - deg; i < len; i++) if (buf[i]) return 0;
    return 1;
}

/* encode = mat_vec_mul (binlin.py:185-196; codebook.py:282-284) */
static void encode_msg(const orc_code_t *c, const uint8_t *msg, uint64_t *out) {
    memset(out, 0, sizeof(uint64_t) * (size_t)c->w64);
    for (int i = 0; i < c->k; i++)
        if (msg[i])
            for (int w = 0; w < c->w64; w++) out[w] ^= c->gen[(size_t)i * c->w64 + w];
}

static double sqdist(const double *y, const uint64_t *cw, int n) {   /* channel.py:90-93 */
    double s = 0.0;
    for (int i = 0; i < n; i++) { double d = y[i] - (getbit(cw, i) ? -1.0 : 1.0); s += d * d; }
    return s;
}

/* ------------------------------------------------------------------------ */
/* SCL: scl_decode (decoders.py:181-268) with _scl_f/_scl_g (:173-178).      */

static inline double sgn(double a) { return (double)((a > 0.0) - (a < 0.0)); }

typedef struct {
    int n, stages, L;
    double *llr, *llr_tmp;     /* L x (stages+1) x n */
    uint8_t *bit, *bit_tmp;    /* L x (stages+1) x n */
    double *pm, *pm2, *pm_tmp;
    int *order, *src;
    uint8_t *natural, *flipped, *frozen;
    int8_t *node_state;
} scl_ws_t;

static void scl_ws_init(scl_ws_t *ws, int n, int L) {
    int st = 0; while ((1 << st) < n) st++;
    ws->n = n; ws->stages = st; ws->L = L;
    size_t cells = (size_t)L * (st + 1) * n;
    ws->llr = malloc(cells * sizeof(double)); ws->llr_tmp = malloc(cells * sizeof(double));
    ws->bit = malloc(cells); ws->bit_tmp = malloc(cells);
    ws->pm = malloc(sizeof(double) * L); ws->pm2 = malloc(sizeof(double) * 2 * L);
    ws->pm_tmp = malloc(sizeof(double) * L);
    ws->order = malloc(sizeof(int) * 2 * L); ws->src = malloc(sizeof(int) * L);
    ws->natural = malloc((size_t)L); ws->flipped = malloc((size_t)L);
    ws->frozen = malloc((size_t)n); ws->node_state = malloc((size_t)(2 * n));
}

static void scl_ws_free(scl_ws_t *ws) {
    free(ws->llr); free(ws->llr_tmp); free(ws->bit); free(ws->bit_tmp);
    free(ws->pm); free(ws->pm2); free(ws->pm_tmp); free(ws->order); free(ws->src);
    free(ws->natural); free(ws->flipped); free(ws->frozen); free(ws->node_state);
}

/* stable argsort of v[0..cnt) (decoders.py:222, kind="stable") */
static void stable_order(const double *v, int cnt, int *order) {
    for (int i = 0; i < cnt; i++) order[i] = i;
    for (int i = 1; i < cnt; i++) {           /* insertion sort is stable */
        int x = order[i]; int j = i - 1;
        while (j >= 0 && v[order[j]] > v[x]) { order[j + 1] = order[j]; j--; }
        order[j + 1] = x;
    }
}

/* Returns the number of finite paths; writes u rows, codewords and metrics in
 * ascending-PM order (ties by slot index, decoders.py:261-268). */
static int scl_one(scl_ws_t *ws, const double *llrs, const int32_t *info, int kp,
                   uint8_t *u_out /* L x n */, uint64_t *cw_out /* L x w64 */,
                   double *pm_out, int w64) {
    const int n = ws->n, st = ws->stages, L = ws->L;
    const size_t lvl = (size_t)n, path = (size_t)(st + 1) * n;
    memset(ws->frozen, 1, (size_t)n);
    for (int i = 0; i < kp; i++) ws->frozen[info[i]] = 0;
    memset(ws->llr, 0, sizeof(double) * L * path);
    memset(ws->bit, 0, (size_t)L * path);
    for (int l = 0; l < L; l++) memcpy(ws->llr + l * path, llrs, sizeof(double) * n);
    for (int l = 0; l < L; l++) ws->pm[l] = INFINITY;
    ws->pm[0] = 0.0;
    memset(ws->node_state, 0, (size_t)(2 * n));

    int depth = 0, node = 0;
    for (;;) {
        if (depth == st) {
            if (ws->frozen[node]) {                                   /* :216-218 */
                for (int l = 0; l < L; l++) {
                    double dm = ws->llr[l * path + st * lvl + node];
                    ws->bit[l * path + st * lvl + node] = 0;
                    ws->pm[l] = ws->pm[l] + fabs(dm) * (double)(dm < 0.0);
                }
            } else {                                                   /* :219-228 */
                for (int l = 0; l < L; l++) {
                    double dm = ws->llr[l * path + st * lvl + node];
                    ws->natural[l] = (uint8_t)(dm < 0.0);
                    ws->pm2[l] = ws->pm[l];
                    ws->pm2[L + l] = ws->pm[l] + fabs(dm);
                }
                stable_order(ws->pm2, 2 * L, ws->order);
                for (int j = 0; j < L; j++) {
                    int o = ws->order[j];
                    ws->src[j] = o % L;
                    ws->flipped[j] = (uint8_t)(o >= L);
                    ws->pm_tmp[j] = ws->pm2[o];
                }
                for (int j = 0; j < L; j++) {
                    memcpy(ws->llr_tmp + j * path, ws->llr + ws->src[j] * path, sizeof(double) * path);
                    memcpy(ws->bit_tmp + j * path, ws->bit + ws->src[j] * path, path);
                }
                double *td = ws->llr; ws->llr = ws->llr_tmp; ws->llr_tmp = td;
                uint8_t *tb = ws->bit; ws->bit = ws->bit_tmp; ws->bit_tmp = tb;
                for (int j = 0; j < L; j++) {
                    ws->pm[j] = ws->pm_tmp[j];
                    ws->bit[j * path + st * lvl + node] =
                        (uint8_t)(ws->natural[ws->src[j]] ^ ws->flipped[j]);
                }
            }
            if (node == n - 1) break;
            node /= 2; depth -= 1;
        } else {
            int seg = n >> depth, half = seg / 2;
            int sidx = (1 << depth) - 1 + node;
            int lo = node * seg;
            if (ws->node_state[sidx] == 0) {                           /* f, :239-244 */
                for (int l = 0; l < L; l++) {
                    const double *b = ws->llr + l * path + depth * lvl + lo;
                    double *o = ws->llr + l * path + (depth + 1) * lvl + lo;
                    for (int i = 0; i < half; i++) {
                        double a = b[i], c = b[half + i];
                        o[i] = sgn(a) * sgn(c) * fmin(fabs(a), fabs(c));
                    }
                }
                ws->node_state[sidx] = 1; node = 2 * node; depth += 1;
            } else if (ws->node_state[sidx] == 1) {                    /* g, :245-252 */
                for (int l = 0; l < L; l++) {
                    const double *b = ws->llr + l * path + depth * lvl + lo;
                    const uint8_t *ub = ws->bit + l * path + (depth + 1) * lvl + lo;
                    double *o = ws->llr + l * path + (depth + 1) * lvl + lo + half;
                    for (int i = 0; i < half; i++)
                        o[i] = b[half + i] + (1.0 - 2.0 * (double)ub[i]) * b[i];
                }
                ws->node_state[sidx] = 2; node = 2 * node + 1; depth += 1;
            } else {                                                   /* combine, :253-259 */
                for (int l = 0; l < L; l++) {
                    uint8_t *up = ws->bit + l * path + depth * lvl + lo;
                    const uint8_t *ch = ws->bit + l * path + (depth + 1) * lvl + lo;
                    for (int i = 0; i < half; i++) { up[i] = ch[i] ^ ch[half + i]; up[half + i] = ch[half + i]; }
                }
                node /= 2; depth -= 1;
            }
        }
    }
    /* finite paths, stable sort by pm (:261-268) */
    int cnt = 0;
    int idx[1024];
    double val[1024];
    for (int l = 0; l < L; l++) if (isfinite(ws->pm[l])) { idx[cnt] = l; val[cnt] = ws->pm[l]; cnt++; }
    int ord[1024];
    stable_order(val, cnt, ord);
    uint8_t row[1024];
    for (int r = 0; r < cnt; r++) {
        int l = idx[ord[r]];
        memcpy(row, ws->bit + l * path + st * lvl, (size_t)n);
        if (u_out) memcpy(u_out + (size_t)r * n, row, (size_t)n);
        polar_transform_u8(row, n);
        uint64_t *cw = cw_out + (size_t)r * w64;
        memset(cw, 0, sizeof(uint64_t) * w64);
        for (int i = 0; i < n; i++) if (row[i]) cw[i >> 6] |= 1ull << (i & 63);
        pm_out[r] = val[ord[r]];
    }
    return cnt;
}

/* ------------------------------------------------------------------------ */
/* Sphere search: _wsd_step_core (decoders.py:360-398), wsd_trajectory        */
/* (:420-452) and mp_wsd (:455-514).                                          */

typedef struct {
    int n, w64, size, nz, m;
    const uint64_t *members;
    int32_t *supp_off, *supp_cat;   /* supports of nonzero members (wsphere.py:211-228) */
    double *t, *gains, *xb;
    int *heap;                      /* top-m selection */
    int *picks;
} hop_ws_t;

static void hop_ws_init(hop_ws_t *h, const orc_sphere_t *s, int n, int w64) {
    h->n = n; h->w64 = w64; h->size = s->size; h->nz = s->size - 1; h->m = s->filter_m;
    h->members = s->members;
    h->supp_off = malloc(sizeof(int32_t) * (size_t)(h->nz + 1));
    int total = 0;
    for (int p = 1; p < s->size; p++)
        for (int w = 0; w < w64; w++) total += __builtin_popcountll(s->members[(size_t)p * w64 + w]);
    h->supp_cat = malloc(sizeof(int32_t) * (size_t)(total + 1));
    int pos = 0;
    for (int p = 1; p < s->size; p++) {
        h->supp_off[p - 1] = pos;
        for (int i = 0; i < n; i++) if (getbit(s->members + (size_t)p * w64, i)) h->supp_cat[pos++] = i;
    }
    h->supp_off[h->nz] = pos;
    h->t = malloc(sizeof(double) * n); h->xb = malloc(sizeof(double) * n);
    h->gains = malloc(sizeof(double) * (size_t)(h->nz + 1));
    h->heap = malloc(sizeof(int) * (size_t)(h->nz + 1));
    h->picks = malloc(sizeof(int) * (size_t)(h->nz + 1));
}

static void hop_ws_free(hop_ws_t *h) {
    free(h->supp_off); free(h->supp_cat); free(h->t); free(h->xb);
    free(h->gains); free(h->heap); free(h->picks);
}

/* "a before b" in the stable descending-gain order of argsort(-gains) */
static inline int gain_before(const double *g, int a, int b) {
    return g[a] > g[b] || (g[a] == g[b] && a < b);
}

static void heap_sift_down(int *hp, int cnt, int i, const double *g) {
    /* heap root = the element that comes LAST in gain order (worst of the kept) */
    for (;;) {
        int l = 2 * i + 1, r = l + 1, w = i;
        if (l < cnt && gain_before(g, hp[w], hp[l])) w = l;
        if (r < cnt && gain_before(g, hp[w], hp[r])) w = r;
        if (w == i) return;
        int t = hp[i]; hp[i] = hp[w]; hp[w] = t; i = w;
    }
}

/* One step.  Returns accepted member index (>=1) or 0.  Updates words/ed. */
static int wsd_step(hop_ws_t *h, const double *y, double yy, uint64_t *words, double *ed) {
    const int n = h->n, nz = h->nz;
    if (nz == 0) return 0;
    for (int i = 0; i < n; i++) h->t[i] = y[i] * (getbit(words, i) ? -1.0 : 1.0);   /* :374 */
    int m_eff = h->m < nz ? h->m : nz;
    int cnt;
    if (m_eff < nz) {
        for (int p = 0; p < nz; p++) {                                 /* _scan_gains :353-357 */
            double s = 0.0;
            for (int q = h->supp_off[p]; q < h->supp_off[p + 1]; q++) s += h->t[h->supp_cat[q]];
            h->gains[p] = -2.0 * s;
        }
        /* picks = argsort(-gains, stable)[:m_eff]  (:379) via a bounded heap */
        int hc = 0;
        for (int p = 0; p < nz; p++) {
            if (hc < m_eff) {
                int i = hc++; h->heap[i] = p;
                while (i > 0) { int par = (i - 1) / 2;
                    if (gain_before(h->gains, h->heap[par], h->heap[i])) {
                        int t = h->heap[i]; h->heap[i] = h->heap[par]; h->heap[par] = t; i = par;
                    } else break; }
            } else if (gain_before(h->gains, p, h->heap[0])) {
                h->heap[0] = p; heap_sift_down(h->heap, hc, 0, h->gains);
            }
        }
        cnt = hc;
        for (int j = cnt - 1; j >= 0; j--) {                           /* pop worst-first */
            h->picks[j] = h->heap[0];
            h->heap[0] = h->heap[j];
            heap_sift_down(h->heap, j, 0, h->gains);
        }
    } else {
        cnt = nz;
        for (int p = 0; p < nz; p++) h->picks[p] = p;
    }
    /* corr = signs[picks] @ t ; eds = (y.y + N) - 2 corr ; best = argmin (:385-391) */
    int best = 0; double best_val = INFINITY;
    for (int j = 0; j < cnt; j++) {
        const uint64_t *pw = h->members + (size_t)(h->picks[j] + 1) * h->w64;
        double corr = 0.0;
        for (int i = 0; i < n; i++) corr += (getbit(pw, i) ? -1.0 : 1.0) * h->t[i];
        double e = (yy + (double)n) - 2.0 * corr;
        if (e < best_val) { best_val = e; best = j; }
    }
    int member = h->picks[best] + 1;                                     /* :392 */
    const uint64_t *pw = h->members + (size_t)member * h->w64;
    uint64_t nw[16];
    for (int w = 0; w < h->w64; w++) nw[w] = words[w] ^ pw[w];
    double best_ed = sqdist(y, nw, n);                                   /* :393-394 */
    if (best_ed < *ed) {                                                 /* :395-397 */
        memcpy(words, nw, sizeof(uint64_t) * h->w64);
        *ed = best_ed;
        return member;
    }
    return 0;
}

/* mp_wsd over A anchors; independent per-anchor loops (SURVEY App. A rule 11) */
static void mp_wsd_one(hop_ws_t *h, const double *y, const uint64_t *anchors, int A, int T,
                       uint64_t *best_out, double *best_ed_out, int32_t *iters_out,
                       int32_t *hops_out /* A x T or NULL */, double *traj_ed_out /* A or NULL */) {
    const int n = h->n, w64 = h->w64;
    double yy = 0.0;
    for (int i = 0; i < n; i++) yy += y[i] * y[i];
    uint64_t cur[16];
    double best_ed = INFINITY; int best_k = 0;
    uint64_t bestw[16];
    for (int a = 0; a < A; a++) {
        memcpy(cur, anchors + (size_t)a * w64, sizeof(uint64_t) * w64);
        double ed = sqdist(y, cur, n);                                 /* :473-478 */
        int used = 0;
        for (int it = 0; it < T; it++) {                               /* :442-451 */
            int mem = wsd_step(h, y, yy, cur, &ed);
            used++;
            if (hops_out) hops_out[(size_t)a * T + it] = mem ? mem : -1;
            if (!mem) break;
        }
        if (hops_out) for (int it = used; it < T; it++) hops_out[(size_t)a * T + it] = -1;
        iters_out[a] = used;
        if (traj_ed_out) traj_ed_out[a] = ed;
        if (ed < best_ed) { best_ed = ed; best_k = a; memcpy(bestw, cur, sizeof(uint64_t) * w64); }  /* :505 */
    }
    (void)best_k;
    memcpy(best_out, bestw, sizeof(uint64_t) * w64);
    *best_ed_out = best_ed;
}

/* ------------------------------------------------------------------------ */
/* osd_decode (decoders.py:274-317).                                         */

typedef struct { double key; int idx; } osd_ent_t;

static int osd_ent_cmp(const void *a, const void *b) {
    const osd_ent_t *x = (const osd_ent_t *)a, *y = (const osd_ent_t *)b;
    if (x->key < y->key) return -1;
    if (x->key > y->key) return 1;
    return (x->idx > y->idx) - (x->idx < y->idx);     /* stable: ties by position */
}

static long long osd_count(int k, int order) {
    long long c = 0, b = 1;
    for (int w = 0; w <= order && w <= k; w++) { c += b; b = b * (k - w) / (w + 1); }
    return c;
}

/* Sorted candidate list: words (C x w64) and squared EDs in ascending order.
 * Returns C, or -1 if the generator is rank deficient (:289-290). */
static long long osd_one(const orc_code_t *c, const double *y, int order, uint64_t **words_out,
                         double **ed_out) {
    const int n = c->n, k = c->k, w64 = c->w64;
    /* column_order = argsort(-|y|, stable) (:287) */
    osd_ent_t *col = malloc(sizeof(osd_ent_t) * (size_t)n);
    for (int i = 0; i < n; i++) { col[i].key = -fabs(y[i]); col[i].idx = i; }
    qsort(col, (size_t)n, sizeof(osd_ent_t), osd_ent_cmp);
    /* row_reduce in that column order (binlin.py:209-247) */
    uint64_t *work = malloc(sizeof(uint64_t) * (size_t)k * w64), *tmp = malloc(sizeof(uint64_t) * w64);
    memcpy(work, c->gen, sizeof(uint64_t) * (size_t)k * w64);
    int *piv = malloc(sizeof(int) * (size_t)k);
    int rank = 0;
    for (int t = 0; t < n && rank < k; t++) {
        const int cc = col[t].idx;
        int p = -1;
        for (int r = rank; r < k; r++) if (getbit(work + (size_t)r * w64, cc)) { p = r; break; }
        if (p < 0) continue;
        if (p != rank) {
            memcpy(tmp, work + (size_t)rank * w64, sizeof(uint64_t) * w64);
            memcpy(work + (size_t)rank * w64, work + (size_t)p * w64, sizeof(uint64_t) * w64);
            memcpy(work + (size_t)p * w64, tmp, sizeof(uint64_t) * w64);
        }
        for (int r = 0; r < k; r++)
            if (r != rank && getbit(work + (size_t)r * w64, cc))
                for (int w = 0; w < w64; w++) work[(size_t)r * w64 + w] ^= work[(size_t)rank * w64 + w];
        piv[rank++] = cc;
    }
    free(col);
    if (rank != k) { free(work); free(tmp); free(piv); return -1; }
    /* base = XOR of basis rows with y[pivot] < 0 (:294-299) */
    uint64_t *base = calloc((size_t)w64, sizeof(uint64_t));
    for (int r = 0; r < k; r++)
        if (y[piv[r]] < 0)
            for (int w = 0; w < w64; w++) base[w] ^= work[(size_t)r * w64 + w];
    /* candidates in itertools.combinations order, weight 0..order (:301-306, :320-323) */
    const long long C = osd_count(k, order);
    uint64_t *words = malloc(sizeof(uint64_t) * (size_t)C * w64);
    long long q = 0;
    int comb[64];
    for (int w = 0; w <= order && w <= k; w++) {
        for (int i = 0; i < w; i++) comb[i] = i;
        for (;;) {
            uint64_t *o = words + (size_t)q * w64;
            memcpy(o, base, sizeof(uint64_t) * w64);
            for (int i = 0; i < w; i++)
                for (int x = 0; x < w64; x++) o[x] ^= work[(size_t)comb[i] * w64 + x];
            q++;
            int i = w - 1;
            while (i >= 0 && comb[i] == k - w + i) i--;
            if (i < 0) break;
            comb[i]++;
            for (int j = i + 1; j < w; j++) comb[j] = comb[j - 1] + 1;
        }
    }
    /* squared EDs and stable argsort (:310-313) */
    osd_ent_t *ent = malloc(sizeof(osd_ent_t) * (size_t)C);
    for (long long i = 0; i < C; i++) { ent[i].key = sqdist(y, words + (size_t)i * w64, n); ent[i].idx = (int)i; }
    qsort(ent, (size_t)C, sizeof(osd_ent_t), osd_ent_cmp);
    uint64_t *sw = malloc(sizeof(uint64_t) * (size_t)C * w64);
    double *se = malloc(sizeof(double) * (size_t)C);
    for (long long i = 0; i < C; i++) {
        memcpy(sw + (size_t)i * w64, words + (size_t)ent[i].idx * w64, sizeof(uint64_t) * w64);
        se[i] = ent[i].key;
    }
    free(ent); free(words); free(base); free(work); free(tmp); free(piv);
    *words_out = sw; *ed_out = se;
    return C;
}

typedef struct {
    const orc_code_t *code; const float *y32; int order, cap, f0, f1;
    int32_t *list_n; uint64_t *list_cw; double *list_ed;
} osd_job_t;

static void *osd_worker(void *arg) {
    osd_job_t *jb = (osd_job_t *)arg;
    const int n = jb->code->n, w64 = jb->code->w64;
    double *y = malloc(sizeof(double) * n);
    for (int f = jb->f0; f < jb->f1; f++) {
        for (int i = 0; i < n; i++) y[i] = (double)jb->y32[(size_t)f * n + i];
        uint64_t *cw; double *ed;
        long long C = osd_one(jb->code, y, jb->order, &cw, &ed);
        long long m = C < jb->cap ? C : jb->cap;
        jb->list_n[f] = (int32_t)m;
        memcpy(jb->list_cw + (size_t)f * jb->cap * w64, cw, sizeof(uint64_t) * (size_t)m * w64);
        memcpy(jb->list_ed + (size_t)f * jb->cap, ed, sizeof(double) * (size_t)m);
        free(cw); free(ed);
    }
    free(y);
    return NULL;
}

/* ------------------------------------------------------------------------ */
/* two_stage_decode (decoders.py:520-583) over a batch, threaded by frame.   */

typedef struct {
    const orc_code_t *code; const orc_sphere_t *sph; const orc_params_t *prm;
    const float *y32; double sigma; int f0, f1;
    uint8_t *stage; uint64_t *best; double *best_ed; int32_t *n_anchor; int32_t *iters;
    int32_t *hops; uint64_t *anchors_out;
    int32_t *list_n; uint64_t *list_cw; double *list_pm;
} ts_job_t;

static void *two_stage_worker(void *arg) {
    ts_job_t *jb = (ts_job_t *)arg;
    const orc_code_t *c = jb->code; const orc_params_t *p = jb->prm;
    const int n = c->n, w64 = c->w64, L = p->list_size, A = p->num_paths, T = p->max_iter;
    scl_ws_t ws; scl_ws_init(&ws, n, L);
    hop_ws_t hw; hop_ws_init(&hw, jb->sph, n, w64);
    double *y = malloc(sizeof(double) * n), *llr = malloc(sizeof(double) * n);
    uint8_t *u = malloc((size_t)L * n);
    uint64_t *cw = malloc(sizeof(uint64_t) * (size_t)L * w64);
    double *pm = malloc(sizeof(double) * L);
    uint64_t *anc = malloc(sizeof(uint64_t) * (size_t)A * w64);
    uint8_t v[1024], msg[1024];
    for (int f = jb->f0; f < jb->f1; f++) {
        for (int i = 0; i < n; i++) {
            y[i] = (double)jb->y32[(size_t)f * n + i];
            llr[i] = 2.0 * y[i] / (jb->sigma * jb->sigma);             /* :550 */
        }
        if (p->osd_order >= 0) {                                        /* :555-556 */
            uint64_t *ow; double *oe;
            long long C = osd_one(c, y, p->osd_order, &ow, &oe);
            long long m = (p->osd_cap > 0 && p->osd_cap < C) ? p->osd_cap : C;
            int done1 = 0;
            if (p->gated) {                                             /* :559-570 */
                uint8_t bits[1024];
                for (long long r = 0; r < m && !done1; r++) {
                    for (int i = 0; i < n; i++) bits[i] = (uint8_t)getbit(ow + (size_t)r * w64, i);
                    polar_transform_u8(bits, n);                       /* precoded_of_codeword */
                    for (int j = 0; j < c->kp; j++) v[j] = bits[c->info_set[j]];
                    if (crc_ok(v, c->kp, c->crc_deg, c->crc_poly)) {
                        memcpy(jb->best + (size_t)f * w64, ow + (size_t)r * w64, sizeof(uint64_t) * w64);
                        jb->best_ed[f] = sqdist(y, ow + (size_t)r * w64, n);
                        jb->stage[f] = 0; jb->n_anchor[f] = 0;
                        done1 = 1;
                    }
                }
            }
            if (!done1) {
                int na = m < A ? (int)m : A;                             /* :572-576, in subcode */
                memcpy(anc, ow, sizeof(uint64_t) * (size_t)na * w64);
                if (jb->anchors_out)
                    memcpy(jb->anchors_out + (size_t)f * A * w64, anc, sizeof(uint64_t) * (size_t)na * w64);
                mp_wsd_one(&hw, y, anc, na, T, jb->best + (size_t)f * w64, &jb->best_ed[f],
                           jb->iters + (size_t)f * A, jb->hops ? jb->hops + (size_t)f * A * T : NULL, NULL);
                jb->stage[f] = 1; jb->n_anchor[f] = na;
            }
            free(ow); free(oe);
            continue;
        }
        int cnt = scl_one(&ws, llr, c->info_set, c->kp, u, cw, pm, w64);
        if (jb->list_n) {
            jb->list_n[f] = cnt;
            memcpy(jb->list_cw + (size_t)f * L * w64, cw, sizeof(uint64_t) * (size_t)cnt * w64);
            memcpy(jb->list_pm + (size_t)f * L, pm, sizeof(double) * (size_t)cnt);
        }
        int done = 0;
        if (p->gated) {                                                 /* :559-570 */
            for (int r = 0; r < cnt && !done; r++) {
                for (int j = 0; j < c->kp; j++) v[j] = u[(size_t)r * n + c->info_set[j]];
                if (crc_ok(v, c->kp, c->crc_deg, c->crc_poly)) {
                    encode_msg(c, v, jb->best + (size_t)f * w64);
                    jb->best_ed[f] = sqdist(y, cw + (size_t)r * w64, n);
                    jb->stage[f] = 0; jb->n_anchor[f] = 0;
                    done = 1;
                }
            }
        }
        if (done) continue;
        int na = cnt < A ? cnt : A;                                     /* :572-579, :468 */
        for (int r = 0; r < na; r++) {
            if (c->is_ca) {
                for (int j = 0; j < c->k; j++) msg[j] = u[(size_t)r * n + c->info_set[j]];
                encode_msg(c, msg, anc + (size_t)r * w64);
            } else {
                memcpy(anc + (size_t)r * w64, cw + (size_t)r * w64, sizeof(uint64_t) * w64);
            }
        }
        if (jb->anchors_out)
            memcpy(jb->anchors_out + (size_t)f * A * w64, anc, sizeof(uint64_t) * (size_t)na * w64);
        mp_wsd_one(&hw, y, anc, na, T, jb->best + (size_t)f * w64, &jb->best_ed[f],
                   jb->iters + (size_t)f * A, jb->hops ? jb->hops + (size_t)f * A * T : NULL, NULL);
        jb->stage[f] = 1; jb->n_anchor[f] = na;
    }
    free(y); free(llr); free(u); free(cw); free(pm); free(anc);
    scl_ws_free(&ws); hop_ws_free(&hw);
    return NULL;
}

static void run_threads(void *(*fn)(void *), void *jobs, size_t job_size, int nthreads) {
    pthread_t th[256];
    if (nthreads <= 1) { fn(jobs); return; }
    for (int t = 0; t < nthreads; t++) pthread_create(&th[t], NULL, fn, (char *)jobs + t * job_size);
    for (int t = 0; t < nthreads; t++) pthread_join(th[t], NULL);
}

int orc_two_stage_batch(const orc_code_t *code, const orc_sphere_t *sph, const orc_params_t *prm,
                        const float *y32, int F, double sigma, int nthreads,
                        uint8_t *stage, uint64_t *best, double *best_ed, int32_t *n_anchor,
                        int32_t *iters, int32_t *hops, uint64_t *anchors_out,
                        int32_t *list_n, uint64_t *list_cw, double *list_pm) {
    if (code->n > 1024 || code->w64 > 16 || prm->list_size > 512) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > F) nthreads = F > 0 ? F : 1;
    ts_job_t jobs[256];
    for (int t = 0; t < nthreads; t++) {
        ts_job_t *j = &jobs[t];
        j->code = code; j->sph = sph; j->prm = prm; j->y32 = y32; j->sigma = sigma;
        j->f0 = (int)((long long)F * t / nthreads); j->f1 = (int)((long long)F * (t + 1) / nthreads);
        j->stage = stage; j->best = best; j->best_ed = best_ed; j->n_anchor = n_anchor;
        j->iters = iters; j->hops = hops; j->anchors_out = anchors_out;
        j->list_n = list_n; j->list_cw = list_cw; j->list_pm = list_pm;
    }
    run_threads(two_stage_worker, jobs, sizeof(ts_job_t), nthreads);
    return 0;
}

/* mp_wsd only, anchors given (decoders.py:455-514); used to test the hop alone. */
typedef struct {
    const orc_sphere_t *sph; int n, w64, A, T; const float *y32; const uint64_t *anchors;
    int f0, f1; uint64_t *best; double *best_ed; int32_t *iters; int32_t *hops; double *traj_ed;
} mp_job_t;

static void *mp_worker(void *arg) {
    mp_job_t *jb = (mp_job_t *)arg;
    hop_ws_t hw; hop_ws_init(&hw, jb->sph, jb->n, jb->w64);
    double *y = malloc(sizeof(double) * jb->n);
    for (int f = jb->f0; f < jb->f1; f++) {
        for (int i = 0; i < jb->n; i++) y[i] = (double)jb->y32[(size_t)f * jb->n + i];
        mp_wsd_one(&hw, y, jb->anchors + (size_t)f * jb->A * jb->w64, jb->A, jb->T,
                   jb->best + (size_t)f * jb->w64, &jb->best_ed[f], jb->iters + (size_t)f * jb->A,
                   jb->hops ? jb->hops + (size_t)f * jb->A * jb->T : NULL,
                   jb->traj_ed ? jb->traj_ed + (size_t)f * jb->A : NULL);
    }
    free(y); hop_ws_free(&hw);
    return NULL;
}

int orc_mpwsd_batch(const orc_sphere_t *sph, int n, int w64, const float *y32,
                    const uint64_t *anchors, int F, int A, int T, int nthreads,
                    uint64_t *best, double *best_ed, int32_t *iters, int32_t *hops, double *traj_ed) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > F) nthreads = F > 0 ? F : 1;
    mp_job_t jobs[256];
    for (int t = 0; t < nthreads; t++) {
        mp_job_t *j = &jobs[t];
        j->sph = sph; j->n = n; j->w64 = w64; j->A = A; j->T = T; j->y32 = y32; j->anchors = anchors;
        j->f0 = (int)((long long)F * t / nthreads); j->f1 = (int)((long long)F * (t + 1) / nthreads);
        j->best = best; j->best_ed = best_ed; j->iters = iters; j->hops = hops; j->traj_ed = traj_ed;
    }
    run_threads(mp_worker, jobs, sizeof(mp_job_t), nthreads);
    return 0;
}

/* scl_decode on float64 LLRs (decoders.py:181-268), one frame */
int orc_scl(const double *llrs, int n, const int32_t *info_set, int kp, int L,
            uint8_t *u_out, uint64_t *cw_out, double *pm_out) {
    int w64 = (n + 63) / 64;
    if (n > 1024 || L > 512) return -1;
    scl_ws_t ws; scl_ws_init(&ws, n, L);
    int cnt = scl_one(&ws, llrs, info_set, kp, u_out, cw_out, pm_out, w64);
    scl_ws_free(&ws);
    return cnt;
}

int orc_crc_ok(const uint8_t *v, int len, int deg, uint32_t poly) { return crc_ok(v, len, deg, poly); }

/* osd_decode over a batch: list_cw F x cap x w64, list_ed F x cap (cap >= 1). */
int orc_osd_batch(const orc_code_t *code, const float *y32, int F, int order, int cap, int nthreads,
                  int32_t *list_n, uint64_t *list_cw, double *list_ed) {
    if (order < 0 || cap < 1 || code->k > 64) return -1;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    if (nthreads > F) nthreads = F > 0 ? F : 1;
    osd_job_t jobs[256];
    for (int t = 0; t < nthreads; t++) {
        osd_job_t *j = &jobs[t];
        j->code = code; j->y32 = y32; j->order = order; j->cap = cap;
        j->f0 = (int)((long long)F * t / nthreads); j->f1 = (int)((long long)F * (t + 1) / nthreads);
        j->list_n = list_n; j->list_cw = list_cw; j->list_ed = list_ed;
    }
    run_threads(osd_worker, jobs, sizeof(osd_job_t), nthreads);
    return 0;
}
