/*
 * dt_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the minimpi derived-datatype engine
 * (/root/reference/pkg/src/minimpi/datatype.py) in plain C.  It exists so the
 * CUDA product (paper_2402_12274_b200/, libmpx.so) can be checked byte for
 * byte against the reference algorithm on the GPU box, where the Python
 * reference is not available.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline -- never as the product.
 *
 * Pinned against golden vectors produced by the real reference
 * (tests/golden/make_golden.py, fixtures tests/golden/NAME.json.gz); see
 * tests/test_oracle_golden.py.
 *
 * Layout tree (datatype.py:45-215): EMPTY / RUN(off,len) / REP(count,stride,
 * body,base) / SEQ(children with run/byte prefix arrays).  Each node caches
 * runs, nbytes, node_count, first_start, last_end, min_off, max_end.
 * Builders keep the invariant "traversal-adjacent runs are never
 * byte-adjacent" (datatype.py:38-41) so node.runs is the maximal-run count.
 *
 * Memory: every node lives in one bump arena; orc_reset() drops everything.
 * Nodes are immutable and shared between trees, exactly like the Python
 * objects.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { K_EMPTY = 0, K_RUN = 1, K_REP = 2, K_SEQ = 3 };

typedef struct ONode ONode;
struct ONode {
    int kind;
    int64_t off, len;                   /* RUN */
    int64_t count, stride, base;        /* REP */
    const ONode *body;                  /* REP */
    const ONode **kids;                 /* SEQ */
    int64_t nkids;
    int64_t *rp, *bp;                   /* SEQ run_prefix / byte_prefix, nkids+1 */
    int64_t runs, nbytes, node_count;
    int64_t first_start, last_end, min_off, max_end;
};

typedef struct {
    const ONode *layout;
    int64_t size, lb, ub;
    int live;
} OType;

/* ------------------------------------------------------------------ arena */

typedef struct Blk { struct Blk *next; size_t used, cap; char mem[]; } Blk;
static Blk *g_arena = NULL;

static void *amalloc(size_t n) {
    n = (n + 15) & ~(size_t)15;
    if (!g_arena || g_arena->used + n > g_arena->cap) {
        size_t cap = n > (1u << 22) ? n : (1u << 22);
        Blk *b = (Blk *)malloc(sizeof(Blk) + cap);
        if (!b) abort();
        b->next = g_arena; b->used = 0; b->cap = cap;
        g_arena = b;
    }
    void *p = g_arena->mem + g_arena->used;
    g_arena->used += n;
    return p;
}

static OType *g_types = NULL;
static int64_t g_ntypes = 0, g_captypes = 0;

void orc_reset(void) {
    while (g_arena) { Blk *n = g_arena->next; free(g_arena); g_arena = n; }
    free(g_types); g_types = NULL; g_ntypes = g_captypes = 0;
}

/* ------------------------------------------------------------ node makers */

static const ONode EMPTY_NODE = { K_EMPTY, 0, 0, 0, 0, 0, NULL, NULL, 0, NULL,
                                  NULL, 0, 0, 1, 0, 0, 0, 0 };
#define EMPTY (&EMPTY_NODE)

static int64_t mn(int64_t a, int64_t b) { return a < b ? a : b; }
static int64_t mx(int64_t a, int64_t b) { return a > b ? a : b; }

/* datatype.py:68-108 */
static const ONode *mk_run(int64_t off, int64_t len) {
    ONode *n = (ONode *)amalloc(sizeof(ONode));
    memset(n, 0, sizeof *n);
    n->kind = K_RUN; n->off = off; n->len = len;
    n->runs = 1; n->nbytes = len; n->node_count = 1;
    n->first_start = off; n->last_end = off + len;
    n->min_off = off; n->max_end = off + len;
    return n;
}

/* datatype.py:124-137 */
static const ONode *mk_rep(int64_t count, int64_t stride, const ONode *body,
                           int64_t base) {
    ONode *n = (ONode *)amalloc(sizeof(ONode));
    memset(n, 0, sizeof *n);
    n->kind = K_REP; n->count = count; n->stride = stride; n->body = body;
    n->base = base;
    n->runs = count * body->runs;
    n->nbytes = count * body->nbytes;
    n->node_count = 1 + body->node_count;
    int64_t span = (count - 1) * stride;
    n->first_start = base + body->first_start;
    n->last_end = base + span + body->last_end;
    n->min_off = base + mn(0, span) + body->min_off;
    n->max_end = base + mx(0, span) + body->max_end;
    return n;
}

/* datatype.py:175-196 */
static const ONode *mk_seq(const ONode **kids, int64_t nk) {
    ONode *n = (ONode *)amalloc(sizeof(ONode));
    memset(n, 0, sizeof *n);
    n->kind = K_SEQ; n->nkids = nk;
    n->kids = (const ONode **)amalloc(sizeof(ONode *) * (size_t)nk);
    memcpy(n->kids, kids, sizeof(ONode *) * (size_t)nk);
    n->rp = (int64_t *)amalloc(sizeof(int64_t) * (size_t)(nk + 1));
    n->bp = (int64_t *)amalloc(sizeof(int64_t) * (size_t)(nk + 1));
    n->rp[0] = n->bp[0] = 0;
    int64_t nc = 1, lo = kids[0]->min_off, hi = kids[0]->max_end;
    for (int64_t i = 0; i < nk; i++) {
        n->rp[i + 1] = n->rp[i] + kids[i]->runs;
        n->bp[i + 1] = n->bp[i] + kids[i]->nbytes;
        nc += kids[i]->node_count;
        lo = mn(lo, kids[i]->min_off);
        hi = mx(hi, kids[i]->max_end);
    }
    n->runs = n->rp[nk]; n->nbytes = n->bp[nk]; n->node_count = nc;
    n->first_start = kids[0]->first_start;
    n->last_end = kids[nk - 1]->last_end;
    n->min_off = lo; n->max_end = hi;
    return n;
}

/* datatype.py:218-225 */
static const ONode *shift(const ONode *n, int64_t d) {
    if (d == 0 || n->runs == 0) return n;
    if (n->kind == K_RUN) return mk_run(n->off + d, n->len);
    if (n->kind == K_REP) return mk_rep(n->count, n->stride, n->body, n->base + d);
    const ONode **k = (const ONode **)malloc(sizeof(ONode *) * (size_t)n->nkids);
    for (int64_t i = 0; i < n->nkids; i++) k[i] = shift(n->kids[i], d);
    const ONode *r = mk_seq(k, n->nkids);
    free(k);
    return r;
}

/* datatype.py:228-243 */
static void first_run(const ONode *n, int64_t *off, int64_t *len) {
    int64_t acc = 0;
    for (;;) {
        if (n->kind == K_RUN) { *off = acc + n->off; *len = n->len; return; }
        if (n->kind == K_REP) { acc += n->base; n = n->body; continue; }
        n = n->kids[0];
    }
}
static void last_run(const ONode *n, int64_t *off, int64_t *len) {
    int64_t acc = 0;
    for (;;) {
        if (n->kind == K_RUN) { *off = acc + n->off; *len = n->len; return; }
        if (n->kind == K_REP) {
            acc += n->base + (n->count - 1) * n->stride; n = n->body; continue;
        }
        n = n->kids[n->nkids - 1];
    }
}

/* datatype.py:246-259: drop empties, unwrap singletons, flatten nested SEQs */
static const ONode *seq_raw(const ONode **parts, int64_t np) {
    int64_t kept = 0, flat = 0;
    const ONode *only = NULL;
    for (int64_t i = 0; i < np; i++) {
        if (parts[i]->runs == 0) continue;
        kept++; only = parts[i];
        flat += parts[i]->kind == K_SEQ ? parts[i]->nkids : 1;
    }
    if (kept == 0) return EMPTY;
    if (kept == 1) return only;
    const ONode **f = (const ONode **)malloc(sizeof(ONode *) * (size_t)flat);
    int64_t j = 0;
    for (int64_t i = 0; i < np; i++) {
        const ONode *p = parts[i];
        if (p->runs == 0) continue;
        if (p->kind == K_SEQ)
            for (int64_t c = 0; c < p->nkids; c++) f[j++] = p->kids[c];
        else
            f[j++] = p;
    }
    const ONode *r = mk_seq(f, flat);
    free(f);
    return r;
}

/* datatype.py:262-267 */
static const ONode *make_rep(int64_t count, int64_t stride, const ONode *body,
                             int64_t base) {
    if (count <= 0 || body->runs == 0) return EMPTY;
    if (count == 1) return shift(body, base);
    return mk_rep(count, stride, body, base);
}

/* datatype.py:270-280 */
static const ONode *drop_first(const ONode *n) {
    if (n->kind == K_RUN) return EMPTY;
    if (n->kind == K_REP) {
        const ONode *rest = make_rep(n->count - 1, n->stride, n->body,
                                     n->base + n->stride);
        if (n->body->runs == 1) return rest;
        const ONode *p[2] = { shift(drop_first(n->body), n->base), rest };
        return seq_raw(p, 2);
    }
    const ONode **p = (const ONode **)malloc(sizeof(ONode *) * (size_t)n->nkids);
    p[0] = drop_first(n->kids[0]);
    for (int64_t i = 1; i < n->nkids; i++) p[i] = n->kids[i];
    const ONode *r = seq_raw(p, n->nkids);
    free(p);
    return r;
}

/* datatype.py:283-293 */
static const ONode *drop_last(const ONode *n) {
    if (n->kind == K_RUN) return EMPTY;
    if (n->kind == K_REP) {
        const ONode *head = make_rep(n->count - 1, n->stride, n->body, n->base);
        if (n->body->runs == 1) return head;
        int64_t last_base = n->base + (n->count - 1) * n->stride;
        const ONode *p[2] = { head, shift(drop_last(n->body), last_base) };
        return seq_raw(p, 2);
    }
    const ONode **p = (const ONode **)malloc(sizeof(ONode *) * (size_t)n->nkids);
    for (int64_t i = 0; i + 1 < n->nkids; i++) p[i] = n->kids[i];
    p[n->nkids - 1] = drop_last(n->kids[n->nkids - 1]);
    const ONode *r = seq_raw(p, n->nkids);
    free(p);
    return r;
}

/* datatype.py:296-315 */
static const ONode *replicate(const ONode *body, int64_t count, int64_t stride) {
    if (body->runs == 0 || count == 0) return EMPTY;
    if (count == 1) return body;
    if (body->last_end != stride + body->first_start)
        return mk_rep(count, stride, body, 0);
    if (body->runs == 1)
        return mk_run(body->first_start, (count - 1) * stride + body->nbytes);
    int64_t h_off, h_len, t_off, t_len;
    first_run(body, &h_off, &h_len);
    last_run(body, &t_off, &t_len);
    const ONode *mid = drop_last(drop_first(body));
    const ONode *ip[2] = { mid, mk_run(t_off, t_len + h_len) };
    const ONode *inner = seq_raw(ip, 2);
    const ONode *tail = shift(drop_first(body), (count - 1) * stride);
    const ONode *op[3] = { mk_run(h_off, h_len),
                           make_rep(count - 1, stride, inner, 0), tail };
    return seq_raw(op, 3);
}

/* datatype.py:318-337 */
static const ONode *concat(const ONode **parts, int64_t np) {
    const ONode **acc = (const ONode **)malloc(sizeof(ONode *) * (size_t)(3 * np + 1));
    int64_t na = 0;
    for (int64_t i = 0; i < np; i++) {
        const ONode *p = parts[i];
        if (p->runs == 0) continue;
        if (na && acc[na - 1]->last_end == p->first_start) {
            const ONode *prev = acc[--na];
            int64_t t_off, t_len, h_off, h_len;
            last_run(prev, &t_off, &t_len);
            first_run(p, &h_off, &h_len);
            const ONode *rem = drop_last(prev);
            if (rem->runs) acc[na++] = rem;
            acc[na++] = mk_run(t_off, t_len + h_len);
            const ONode *rest = drop_first(p);
            if (rest->runs) acc[na++] = rest;
        } else {
            acc[na++] = p;
        }
    }
    const ONode *r = seq_raw(acc, na);
    free(acc);
    return r;
}

/* ------------------------------------------------------------ type table */

static int64_t new_type(const ONode *lay, int64_t size, int64_t lb, int64_t ub) {
    if (g_ntypes == g_captypes) {
        g_captypes = g_captypes ? 2 * g_captypes : 64;
        g_types = (OType *)realloc(g_types, sizeof(OType) * (size_t)g_captypes);
    }
    g_types[g_ntypes].layout = lay;
    g_types[g_ntypes].size = size;
    g_types[g_ntypes].lb = lb;
    g_types[g_ntypes].ub = ub;
    g_types[g_ntypes].live = 1;
    return g_ntypes++;
}

/*
 * Spec program (prefix encoding of the flatten_oracle tuple forms,
 * tests/flatten_oracle.py:8-16, plus "indexed"):
 *   0 BASIC   size
 *   1 CONTIG  count child
 *   2 VECTOR  count bl stride_elems child
 *   3 HVECTOR count bl stride_bytes child
 *   4 IDXBLK  bl n d[n] child
 *   5 STRUCT  n bl[n] d[n] child[n]
 *   6 SUBARR  nd full[nd] sub[nd] off[nd] child
 *   7 RESIZED lb extent child
 *   8 INDEXED n bl[n] d[n] child          (MPI_Type_indexed, displs in extents)
 * Returns the type handle, or -1 on a malformed program.
 */
static int64_t build(const int64_t *s, int64_t n, int64_t *pos);

static int64_t build_child(const int64_t *s, int64_t n, int64_t *pos) {
    return build(s, n, pos);
}

#define NEED(k) do { if (*pos + (k) > n) return -1; } while (0)

static int64_t build(const int64_t *s, int64_t n, int64_t *pos) {
    NEED(1);
    int64_t kind = s[(*pos)++];
    switch (kind) {
    case 0: { /* datatype.py:410-412 */
        NEED(1);
        int64_t sz = s[(*pos)++];
        return new_type(sz > 0 ? mk_run(0, sz) : EMPTY, sz, 0, sz);
    }
    case 1: { /* type_contiguous, datatype.py:444-455 */
        NEED(1);
        int64_t count = s[(*pos)++];
        int64_t c = build_child(s, n, pos); if (c < 0) return -1;
        OType ch = g_types[c];
        int64_t ext = ch.ub - ch.lb;
        const ONode *lay = replicate(ch.layout, count, ext);
        int64_t lb = 0, ub = 0;
        if (count) { lb = ch.lb; ub = (count - 1) * ext + ch.ub; }
        return new_type(lay, count * ch.size, lb, ub);
    }
    case 2: case 3: { /* type_vector / type_hvector, datatype.py:458-495 */
        NEED(3);
        int64_t count = s[(*pos)++], bl = s[(*pos)++], stride = s[(*pos)++];
        int64_t c = build_child(s, n, pos); if (c < 0) return -1;
        OType ch = g_types[c];
        int64_t ext = ch.ub - ch.lb;
        int64_t step = kind == 2 ? stride * ext : stride;
        const ONode *block = replicate(ch.layout, bl, ext);
        const ONode *lay = replicate(block, count, step);
        int64_t lb = 0, ub = 0;
        if (count && bl) {
            int64_t span = (count - 1) * step;
            lb = mn(0, span) + ch.lb;
            ub = mx(0, span) + (bl - 1) * ext + ch.ub;
        }
        return new_type(lay, count * bl * ch.size, lb, ub);
    }
    case 4: { /* type_indexed_block, datatype.py:498-516 */
        NEED(2);
        int64_t bl = s[(*pos)++], nd = s[(*pos)++];
        NEED(nd);
        const int64_t *d = s + *pos; *pos += nd;
        int64_t c = build_child(s, n, pos); if (c < 0) return -1;
        OType ch = g_types[c];
        int64_t ext = ch.ub - ch.lb;
        const ONode *block = replicate(ch.layout, bl, ext);
        const ONode **parts = (const ONode **)malloc(sizeof(ONode *) * (size_t)(nd + 1));
        int64_t dmin = 0, dmax = 0;
        for (int64_t i = 0; i < nd; i++) {
            parts[i] = shift(block, d[i] * ext);
            if (i == 0 || d[i] < dmin) dmin = d[i];
            if (i == 0 || d[i] > dmax) dmax = d[i];
        }
        const ONode *lay = concat(parts, nd);
        free(parts);
        int64_t lb = 0, ub = 0;
        if (nd && bl) { lb = dmin * ext + ch.lb; ub = (dmax + bl - 1) * ext + ch.ub; }
        return new_type(lay, nd * bl * ch.size, lb, ub);
    }
    case 5: case 8: { /* type_create_struct datatype.py:519-547; indexed = struct
                         with byte displacement d*extent and one shared child */
        NEED(1);
        int64_t nb = s[(*pos)++];
        NEED(2 * nb);
        const int64_t *bl = s + *pos; *pos += nb;
        const int64_t *d = s + *pos; *pos += nb;
        int64_t *kids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nb + 1));
        if (kind == 5) {
            for (int64_t i = 0; i < nb; i++) {
                kids[i] = build_child(s, n, pos);
                if (kids[i] < 0) { free(kids); return -1; }
            }
        } else {
            int64_t c = build_child(s, n, pos);
            if (c < 0) { free(kids); return -1; }
            for (int64_t i = 0; i < nb; i++) kids[i] = c;
        }
        const ONode **parts = (const ONode **)malloc(sizeof(ONode *) * (size_t)(nb + 1));
        int64_t size = 0, lb = 0, ub = 0;
        int have = 0;
        for (int64_t i = 0; i < nb; i++) {
            OType ch = g_types[kids[i]];
            int64_t ext = ch.ub - ch.lb;
            int64_t disp = kind == 5 ? d[i] : d[i] * ext;
            parts[i] = shift(replicate(ch.layout, bl[i], ext), disp);
            size += bl[i] * ch.size;
            if (bl[i] > 0) {
                int64_t b_lb = disp + ch.lb, b_ub = disp + (bl[i] - 1) * ext + ch.ub;
                lb = have ? mn(lb, b_lb) : b_lb;
                ub = have ? mx(ub, b_ub) : b_ub;
                have = 1;
            }
        }
        const ONode *lay = concat(parts, nb);
        free(parts); free(kids);
        return new_type(lay, size, lb, ub);
    }
    case 6: { /* type_create_subarray, C order, datatype.py:550-583 */
        NEED(1);
        int64_t nd = s[(*pos)++];
        NEED(3 * nd);
        const int64_t *full = s + *pos, *sub = s + *pos + nd, *offs = s + *pos + 2 * nd;
        *pos += 3 * nd;
        int64_t c = build_child(s, n, pos); if (c < 0 || nd < 1) return -1;
        OType ch = g_types[c];
        int64_t ext = ch.ub - ch.lb;
        int64_t *st = (int64_t *)malloc(sizeof(int64_t) * (size_t)nd);
        st[nd - 1] = ext;
        for (int64_t k = nd - 2; k >= 0; k--) st[k] = st[k + 1] * full[k + 1];
        const ONode *core = replicate(ch.layout, sub[nd - 1], ext);
        for (int64_t k = nd - 2; k >= 0; k--) core = replicate(core, sub[k], st[k]);
        int64_t base = 0, size = ch.size, vol = 1;
        for (int64_t k = 0; k < nd; k++) {
            base += offs[k] * st[k]; size *= sub[k]; vol *= full[k];
        }
        free(st);
        return new_type(shift(core, base), size, 0, vol * ext);
    }
    case 7: { /* type_create_resized, datatype.py:586-591 */
        NEED(2);
        int64_t lb = s[(*pos)++], extent = s[(*pos)++];
        int64_t c = build_child(s, n, pos); if (c < 0) return -1;
        OType ch = g_types[c];
        return new_type(ch.layout, ch.size, lb, lb + extent);
    }
    }
    return -1;
}

int64_t orc_build(const int64_t *spec, int64_t n) {
    int64_t pos = 0;
    int64_t h = build(spec, n, &pos);
    if (h >= 0 && pos != n) return -1;
    return h;
}

/* out: size, lb, ub, extent, runs(segment_count), node_count, min_off, max_end */
int orc_info(int64_t h, int64_t *out) {
    if (h < 0 || h >= g_ntypes) return -1;
    OType t = g_types[h];
    out[0] = t.size; out[1] = t.lb; out[2] = t.ub; out[3] = t.ub - t.lb;
    out[4] = t.layout->runs; out[5] = t.layout->node_count;
    out[6] = t.layout->min_off; out[7] = t.layout->max_end;
    return 0;
}

/* _layout_for, datatype.py:658-661 */
static const ONode *layout_for(int64_t h, int64_t count) {
    OType t = g_types[h];
    if (count == 1) return t.layout;
    return replicate(t.layout, count, t.ub - t.lb);
}

/* layout stats after count replication: runs, nbytes, min_off, max_end, node_count */
int orc_layout_info(int64_t h, int64_t count, int64_t *out) {
    if (h < 0 || h >= g_ntypes || count < 0) return -1;
    const ONode *l = layout_for(h, count);
    out[0] = l->runs; out[1] = l->nbytes; out[2] = l->min_off; out[3] = l->max_end;
    out[4] = l->node_count;
    return 0;
}

/* ------------------------------------------------------------ queries */

/* prefix_within, datatype.py:105-108 (RUN), 155-163 (REP), 208-215 (SEQ) */
static void prefix_within(const ONode *n, int64_t budget, int64_t *segs, int64_t *used) {
    *segs = 0; *used = 0;
    for (;;) {
        if (n->kind == K_EMPTY) return;
        if (n->kind == K_RUN) {
            if (n->len <= budget) { *segs += 1; *used += n->len; }
            return;
        }
        if (n->kind == K_REP) {
            int64_t per = n->body->nbytes;
            int64_t q = mn(budget / per, n->count);
            *segs += q * n->body->runs; *used += q * per;
            if (q >= n->count) return;
            budget -= q * per; n = n->body;
            continue;
        }
        /* bisect_right(byte_prefix, budget) - 1 */
        int64_t lo = 0, hi = n->nkids + 1;
        while (lo < hi) { int64_t m = (lo + hi) / 2; if (n->bp[m] <= budget) lo = m + 1; else hi = m; }
        int64_t i = lo - 1;
        *segs += n->rp[i]; *used += n->bp[i];
        if (i >= n->nkids) return;
        budget -= n->bp[i]; n = n->kids[i];
    }
}

/* type_iov_len, datatype.py:618-628 (no count argument in the reference) */
int orc_iov_len(int64_t h, int64_t max_bytes, int64_t *nseg, int64_t *nbytes) {
    if (h < 0 || h >= g_ntypes || max_bytes < -1) return -1;
    OType t = g_types[h];
    if (max_bytes == -1 || max_bytes >= t.size) {
        *nseg = t.layout->runs; *nbytes = t.size; return 0;
    }
    prefix_within(t.layout, max_bytes, nseg, nbytes);
    return 0;
}

/* Segment visitor: emit (datatype.py:98-99,139-143,198-200) and emit_from
 * (datatype.py:101-103,145-153,202-206).  The visitor returns nonzero to stop. */
typedef int (*visit_fn)(void *ctx, int64_t off, int64_t len);

static int emit(const ONode *n, int64_t shift_, visit_fn f, void *ctx) {
    switch (n->kind) {
    case K_EMPTY: return 0;
    case K_RUN: return f(ctx, shift_ + n->off, n->len);
    case K_REP: {
        int64_t start = shift_ + n->base;
        for (int64_t k = 0; k < n->count; k++)
            if (emit(n->body, start + k * n->stride, f, ctx)) return 1;
        return 0;
    }
    default:
        for (int64_t i = 0; i < n->nkids; i++)
            if (emit(n->kids[i], shift_, f, ctx)) return 1;
        return 0;
    }
}

static int emit_from(const ONode *n, int64_t k, int64_t shift_, visit_fn f, void *ctx) {
    switch (n->kind) {
    case K_EMPTY: return 0;
    case K_RUN: return k == 0 ? f(ctx, shift_ + n->off, n->len) : 0;
    case K_REP: {
        int64_t start = shift_ + n->base;
        int64_t q = k / n->body->runs, r = k % n->body->runs;
        if (r) {
            if (emit_from(n->body, r, start + q * n->stride, f, ctx)) return 1;
            q += 1;
        }
        for (int64_t j = q; j < n->count; j++)
            if (emit(n->body, start + j * n->stride, f, ctx)) return 1;
        return 0;
    }
    default: {
        int64_t lo = 0, hi = n->nkids + 1;   /* bisect_right(run_prefix, k) - 1 */
        while (lo < hi) { int64_t m = (lo + hi) / 2; if (n->rp[m] <= k) lo = m + 1; else hi = m; }
        int64_t i = lo - 1;
        if (emit_from(n->kids[i], k - n->rp[i], shift_, f, ctx)) return 1;
        for (int64_t c = i + 1; c < n->nkids; c++)
            if (emit(n->kids[c], shift_, f, ctx)) return 1;
        return 0;
    }
    }
}

typedef struct { int64_t *out; int64_t left, got; } IovCtx;
static int iov_visit(void *c, int64_t off, int64_t len) {
    IovCtx *x = (IovCtx *)c;
    if (x->left <= 0) return 1;
    x->out[2 * x->got] = off; x->out[2 * x->got + 1] = len;
    x->got++; x->left--;
    return x->left <= 0;
}

/* type_iov, datatype.py:631-650, generalised with count replication
 * (layout_for) so replicated layouts can be enumerated too.
 * Returns number of segments written into out_pairs (off,len interleaved),
 * -1 on a bad argument. */
int64_t orc_iov(int64_t h, int64_t count, int64_t iov_offset, int64_t max_iov_len,
                int64_t *out_pairs) {
    if (h < 0 || h >= g_ntypes || count < 0) return -1;
    const ONode *l = layout_for(h, count);
    int64_t total = l->runs;
    if (iov_offset < 0 || iov_offset > total || max_iov_len < -1) return -1;
    int64_t n = total - iov_offset;
    if (max_iov_len != -1 && max_iov_len < n) n = max_iov_len;
    if (n <= 0) return 0;
    IovCtx c = { out_pairs, n, 0 };
    emit_from(l, iov_offset, 0, iov_visit, &c);
    return c.got;
}

/* ------------------------------------------------------------ pack/unpack */

typedef struct { const uint8_t *src; uint8_t *dst; int64_t pos, n; } CopyCtx;

static int pack_visit(void *c, int64_t off, int64_t len) {
    CopyCtx *x = (CopyCtx *)c;
    memcpy(x->dst + x->pos, x->src + off, (size_t)len);
    x->pos += len;
    return 0;
}

/* pack, datatype.py:695-702 with _checked_view bounds (680-692).
 * Returns bytes written (= layout nbytes) or -1 (bad args / out of bounds). */
int64_t orc_pack(int64_t h, int64_t count, const uint8_t *src, int64_t src_len,
                 uint8_t *dst) {
    if (h < 0 || h >= g_ntypes || count < 0) return -1;
    const ONode *l = layout_for(h, count);
    if (l->runs) {
        if (l->min_off < 0 || l->max_end > src_len) return -1;
    }
    CopyCtx c = { src, dst, 0, 0 };
    emit(l, 0, pack_visit, &c);
    return c.pos;
}

static int unpack_visit(void *c, int64_t off, int64_t len) {
    CopyCtx *x = (CopyCtx *)c;
    if (x->pos >= x->n) return 1;
    int64_t take = len < x->n - x->pos ? len : x->n - x->pos;
    memcpy(x->dst + off, x->src + x->pos, (size_t)take);   /* last writer wins */
    x->pos += take;
    return 0;
}

/* unpack, datatype.py:705-728.  *truncated = 1 when data holds more bytes
 * than the layout (the reference raises TruncateError after the writes).
 * Returns bytes written or -1. */
int64_t orc_unpack(int64_t h, int64_t count, const uint8_t *data, int64_t n,
                   uint8_t *dst, int64_t dst_len, int *truncated) {
    if (h < 0 || h >= g_ntypes || count < 0) return -1;
    const ONode *l = layout_for(h, count);
    if (l->runs) {
        if (l->min_off < 0 || l->max_end > dst_len) return -1;
    }
    CopyCtx c = { data, dst, 0, n };
    emit(l, 0, unpack_visit, &c);
    *truncated = n > l->nbytes;
    return c.pos;
}

/* copy_between zipper, datatype.py:760-797 (dst_h < 0 means plain byte
 * region).  Returns bytes moved or -1.  Implemented over materialised iov
 * lists (test sizes only). */
int64_t orc_copy_between(int64_t sh, int64_t scount, const uint8_t *src, int64_t slen,
                         int64_t dh, int64_t dcount, uint8_t *dst, int64_t dlen) {
    if (sh < 0 || sh >= g_ntypes || scount < 0) return -1;
    const ONode *sl = layout_for(sh, scount);
    if (sl->runs && (sl->min_off < 0 || sl->max_end > slen)) return -1;
    const ONode *dl;
    if (dh < 0) dl = dlen ? mk_run(0, dlen) : EMPTY;
    else {
        if (dh >= g_ntypes || dcount < 0) return -1;
        dl = layout_for(dh, dcount);
        if (dl->runs && (dl->min_off < 0 || dl->max_end > dlen)) return -1;
    }
    int64_t ns = sl->runs, nd = dl->runs;
    int64_t *sv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * ns + 2));
    int64_t *dv = (int64_t *)malloc(sizeof(int64_t) * (size_t)(2 * nd + 2));
    IovCtx a = { sv, ns, 0 }, b = { dv, nd, 0 };
    if (ns) emit(sl, 0, iov_visit, &a);
    if (nd) emit(dl, 0, iov_visit, &b);
    int64_t i = 0, j = 0, so = 0, sn = 0, dof = 0, dn = 0, moved = 0;
    for (;;) {
        if (sn == 0) { if (i >= ns) break; so = sv[2 * i]; sn = sv[2 * i + 1]; i++; }
        if (dn == 0) { if (j >= nd) break; dof = dv[2 * j]; dn = dv[2 * j + 1]; j++; }
        int64_t k = sn < dn ? sn : dn;
        memmove(dst + dof, src + so, (size_t)k);
        so += k; sn -= k; dof += k; dn -= k; moved += k;
    }
    free(sv); free(dv);
    return moved;
}

/* Allreduce SUM oracle, comm.py:582-588: rank-ordered accumulation
 * acc = x0; acc += x1; ... in the element type (int64 wraps like C). */
void orc_allreduce_i64(const int64_t *const *bufs, int nranks, int64_t count, int64_t *out) {
    for (int64_t i = 0; i < count; i++) {
        uint64_t acc = (uint64_t)bufs[0][i];
        for (int r = 1; r < nranks; r++) acc += (uint64_t)bufs[r][i];
        out[i] = (int64_t)acc;
    }
}
void orc_allreduce_f64(const double *const *bufs, int nranks, int64_t count, double *out) {
    for (int64_t i = 0; i < count; i++) {
        double acc = bufs[0][i];
        for (int r = 1; r < nranks; r++) acc += bufs[r][i];
        out[i] = acc;
    }
}
