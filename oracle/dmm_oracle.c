/* dmm_oracle.c -- CPU restatement of the reference hot path. TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this
 * file (it is the checker, never the thing measured or shipped).  Every function
 * cites the reference file:line it restates; paths are relative to
 * /root/reference/proj/include/dmm/.
 *
 * Model: the reference Machine's cells (core.hpp:265-497) as a bank-major array with
 * capacity 4m+8 and the same region map (core.hpp:94-98), and MatrixView
 * (view.hpp:15-134) as (row list, column window, two scratch windows).  Row sorts
 * (radix or merge in the reference) are restated as plain sorts: both produce the
 * unique sorted order of the row, so the state after every step is identical.
 * Step metering, CAC auditing and tracing are not restated.
 */
#include "dmm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t word;
typedef uint32_t u32;
typedef uint64_t u64;

#define TRY(x)                  \
    do {                        \
        int _s = (x);           \
        if (_s != DMM_OK)       \
            return _s;          \
    } while (0)

/* ------------------------------------------------------------------------ */
/* L0 utilities  core.hpp:27-53                                               */
/* ------------------------------------------------------------------------ */
static u32 ilog2_ceil(u64 x) { /* core.hpp:27 */
    u32 k = 0;
    u64 p = 1;
    while (p < x) {
        p <<= 1;
        ++k;
    }
    return k;
}
static u64 next_pow2(u64 x) {                                        /* core.hpp:39 */
    u64 p = 1;
    while (p < x)
        p <<= 1;
    return p;
}
static u32 isqrt_floor(u32 x) { /* core.hpp:46 */
    u32 r = (u32)sqrt((double)x);
    while ((u64)r * r > x)
        --r;
    while ((u64)(r + 1) * (r + 1) <= x)
        ++r;
    return r;
}

/* ------------------------------------------------------------------------ */
/* RNG  rng.hpp:15-48 (std::mt19937_64, splitmix64, rejection rng_below)     */
/* ------------------------------------------------------------------------ */
void dmmo_rng_seed(dmmo_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (u64)i;
    r->mti = 312;
}

uint64_t dmmo_rng_next(dmmo_rng* r) {
    static const u64 UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, MA = 0xB5026F5AA96619E9ULL;
    if (r->mti >= 312) {
        int i;
        for (i = 0; i < 312 - 156; ++i) {
            u64 x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
        }
        for (; i < 311; ++i) {
            u64 x = (r->mt[i] & UM) | (r->mt[i + 1] & LM);
            r->mt[i] = r->mt[i + 156 - 312] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
        }
        u64 x = (r->mt[311] & UM) | (r->mt[0] & LM);
        r->mt[311] = r->mt[155] ^ (x >> 1) ^ ((x & 1) ? MA : 0);
        r->mti = 0;
    }
    u64 x = r->mt[r->mti++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

uint64_t dmmo_splitmix64(uint64_t x) { /* rng.hpp:17 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t dmmo_rng_below(dmmo_rng* r, uint64_t n) { /* rng.hpp:25 */
    const u64 limit = ~(u64)0 - (~(u64)0 % n + 1) % n;
    u64 x;
    do {
        x = dmmo_rng_next(r);
    } while (x > limit);
    return x % n;
}

static void fisher_yates(dmmo_rng* r, word* v, u64 n) { /* rng.hpp:34 */
    for (u64 i = n; i > 1; --i) {
        u64 j = dmmo_rng_below(r, i);
        word t = v[i - 1];
        v[i - 1] = v[j];
        v[j] = t;
    }
}

/* instance.hpp:48-76 */
void dmmo_gen_instance(int kind, uint32_t w, uint32_t m, uint64_t seed, uint64_t* grid) {
    dmmo_rng r;
    dmmo_rng_seed(&r, dmmo_splitmix64(seed ^ ((u64)w << 32) ^ m));
    const u64 n = (u64)w * m;
    if (kind == DMMO_KIND_SORT) {
        for (u64 i = 0; i < n; ++i)
            grid[i] = dmmo_rng_next(&r);
    } else if (kind == DMMO_KIND_PARTITION) {
        u64 k = 0;
        for (u32 label = 0; label < w; ++label)
            for (u32 c = 0; c < m; ++c)
                grid[k++] = label;
        fisher_yates(&r, grid, n);
    } else {
        for (u64 i = 0; i < n; ++i)
            grid[i] = i;
        fisher_yates(&r, grid, n); /* random_permutation rng.hpp:42 */
    }
}

void dmmo_gen_sort_u32(uint32_t w, uint32_t m, uint64_t seed, uint64_t* grid) {
    /* Builder-defined uint32 tile generator: the reference's sort
     * generator emits full 64-bit words; tile k uses Rng(splitmix64(seed))() >> 32. */
    dmmo_rng r;
    dmmo_rng_seed(&r, dmmo_splitmix64(seed));
    const u64 n = (u64)w * m;
    for (u64 i = 0; i < n; ++i)
        grid[i] = dmmo_rng_next(&r) >> 32;
}

/* ------------------------------------------------------------------------ */
/* L1 machine model  core.hpp:84-120, 265-497                               */
/* ------------------------------------------------------------------------ */
typedef struct {
    u32 w, m, cap;
    int strict;
    word* cells; /* bank-major: cells[bank*cap + off]  core.hpp:432 */
} machine_t;

static int machine_init(machine_t* mc, u32 w, u32 m, int strict) { /* MachineConfig::standard core.hpp:105 */
    if (w < 1 || m < 1)
        return DMM_SHAPE_VIOLATION;
    mc->w = w;
    mc->m = m;
    mc->cap = 4 * m + 8;
    mc->strict = strict;
    mc->cells = (word*)calloc((size_t)w * mc->cap, sizeof(word));
    return mc->cells ? DMM_OK : DMM_ERROR;
}
static void machine_free(machine_t* mc) { free(mc->cells); }
static u32 out_base(const machine_t* mc) { return mc->m; }
static u32 scratch_a_base(const machine_t* mc) { return 2 * mc->m; }
static u32 scratch_b_base(const machine_t* mc) { return 3 * mc->m; }
static u32 counter_base(const machine_t* mc) { return mc->cap - 8; }
static word* cell(const machine_t* mc, u32 bank, u32 off) { return &mc->cells[(u64)bank * mc->cap + off]; }

/* ------------------------------------------------------------------------ */
/* L2 views  view.hpp:15-167                                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    machine_t* mach;
    u32 W;
    u32* rows;
    u32 col_base, cols, s0, s1;
} view_t;

static view_t view_make(machine_t* mc, const u32* rows, u32 W, u32 col_base, u32 cols, u32 s0, u32 s1) {
    view_t v;
    v.mach = mc;
    v.W = W;
    v.rows = (u32*)malloc(sizeof(u32) * (W ? W : 1));
    if (W)
        memcpy(v.rows, rows, sizeof(u32) * W);
    v.col_base = col_base;
    v.cols = cols;
    v.s0 = s0;
    v.s1 = s1;
    return v;
}
static view_t view_full(machine_t* mc) { /* view.hpp:21 */
    u32* rows = (u32*)malloc(sizeof(u32) * mc->w);
    for (u32 r = 0; r < mc->w; ++r)
        rows[r] = r;
    view_t v = view_make(mc, rows, mc->w, 0, mc->m, out_base(mc), scratch_a_base(mc));
    free(rows);
    return v;
}
static view_t view_copy(const view_t* v) { return view_make(v->mach, v->rows, v->W, v->col_base, v->cols, v->s0, v->s1); }
static void view_free(view_t* v) {
    free(v->rows);
    v->rows = NULL;
}
static view_t view_row_range(const view_t* v, u32 lo, u32 count) { /* view.hpp:61 */
    return view_make(v->mach, v->rows + lo, count, v->col_base, v->cols, v->s0, v->s1);
}
static view_t view_pick_rows(const view_t* v, const u32* locals, u32 n) { /* view.hpp:70 */
    view_t out = view_make(v->mach, NULL, 0, v->col_base, v->cols, v->s0, v->s1);
    free(out.rows);
    out.rows = (u32*)malloc(sizeof(u32) * (n ? n : 1));
    out.W = n;
    for (u32 i = 0; i < n; ++i)
        out.rows[i] = v->rows[locals[i]];
    return out;
}
static view_t view_col_window(const view_t* v, u32 lo, u32 count) { /* view.hpp:83 */
    view_t out = view_copy(v);
    out.col_base += lo;
    out.s0 += lo;
    out.s1 += lo;
    out.cols = count;
    return out;
}
static word* vcell(const view_t* v, u32 r, u32 c) { return cell(v->mach, v->rows[r], v->col_base + c); }

static void view_load(const view_t* v, const word* grid) { /* view.hpp:103 */
    for (u32 r = 0; r < v->W; ++r)
        for (u32 c = 0; c < v->cols; ++c)
            *vcell(v, r, c) = grid[(u64)r * v->cols + c];
}
static void view_snapshot(const view_t* v, word* grid) { /* view.hpp:95 */
    for (u32 r = 0; r < v->W; ++r)
        for (u32 c = 0; c < v->cols; ++c)
            grid[(u64)r * v->cols + c] = *vcell(v, r, c);
}

/* ------------------------------------------------------------------------ */
/* Row sorting  sort.hpp:20-81, partition.hpp:24-99                           */
/* ------------------------------------------------------------------------ */
/* SortOrder sort.hpp:20-38 */
typedef enum { ORD_ASC = 0, ORD_DESC = 1, ORD_ALT = 2 } ord_kind;
typedef struct {
    ord_kind kind;
    int start_asc;
} sort_order;
static sort_order ord_asc(void) { sort_order o = {ORD_ASC, 1}; return o; }
static sort_order ord_desc(void) { sort_order o = {ORD_DESC, 1}; return o; }
static sort_order ord_alt(int start_asc) { sort_order o = {ORD_ALT, start_asc}; return o; }
static sort_order ord_dir(int asc) { return asc ? ord_asc() : ord_desc(); }
static int ascending_for(sort_order o, u32 row) {
    switch (o.kind) {
        case ORD_ASC: return 1;
        case ORD_DESC: return 0;
        default: return ((row % 2 == 0) == (o.start_asc != 0));
    }
}

static int cmp_asc(const void* a, const void* b) {
    word x = *(const word*)a, y = *(const word*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}
static int cmp_desc(const void* a, const void* b) { return cmp_asc(b, a); }

/* Sort `len` cells of one bank starting at `off` (the outcome of row_merge_sort
 * sort.hpp:44-70 and of row_radix_segment partition.hpp:42-88: the unique sorted row). */
static void bank_sort(machine_t* mc, u32 bank, u32 off, u32 len, int asc) {
    if (len <= 1)
        return;
    word* p = cell(mc, bank, off);
    qsort(p, len, sizeof(word), asc ? cmp_asc : cmp_desc);
}

/* radix_sort_rows partition.hpp:94-99 (row_radix_segment checks x < domain, :63) */
static int radix_sort_rows(const view_t* v, u64 domain, sort_order o) {
    if (v->cols <= 1)
        return DMM_OK; /* partition.hpp:44: len <= 1 returns before any read */
    for (u32 r = 0; r < v->W; ++r) {
        for (u32 c = 0; c < v->cols; ++c)
            if (*vcell(v, r, c) >= domain)
                return DMM_KEY_OUT_OF_RANGE;
        bank_sort(v->mach, v->rows[r], v->col_base, v->cols, ascending_for(o, r));
    }
    return DMM_OK;
}

/* sort_rows sort.hpp:76-81 */
static int sort_rows(const view_t* v, sort_order o) {
    for (u32 r = 0; r < v->W; ++r)
        bank_sort(v->mach, v->rows[r], v->col_base, v->cols, ascending_for(o, r));
    return DMM_OK;
}

/* merge_sort_segments sort.hpp:177-182 */
static int merge_sort_segments(const view_t* v, u32 seg, int asc) {
    for (u32 r = 0; r < v->W; ++r)
        for (u32 s = 0; s < v->cols; s += seg)
            bank_sort(v->mach, v->rows[r], v->col_base + s, seg, asc);
    return DMM_OK;
}

/* Row sorter / segment sorter "strategy" objects (the lambdas of the reference). */
typedef struct {
    int radix; /* 1: radix_sort_rows with domain, 0: sort_rows (merge) */
    u64 domain;
} row_sorter;
static int do_row_sort(const row_sorter* rs, const view_t* v, sort_order o) {
    return rs->radix ? radix_sort_rows(v, rs->domain, o) : sort_rows(v, o);
}

/* ------------------------------------------------------------------------ */
/* Layout  layout.hpp:24-61, 316-405                                         */
/* ------------------------------------------------------------------------ */
static int transpose_square(const view_t* v) { /* layout.hpp:24 */
    if (v->W != v->cols)
        return DMM_NOT_SQUARE;
    const u32 s = v->W;
    for (u32 i = 0; i < s; ++i)
        for (u32 j = i + 1; j < s; ++j) {
            word* a = vcell(v, i, j);
            word* b = vcell(v, j, i);
            word t = *a;
            *a = *b;
            *b = t;
        }
    return DMM_OK;
}

/* convert_layout layout.hpp:357-391: value at row-major linear index i*M+j moves to
 * (lin mod W, lin div W) (to_column_major) or the inverse (to_row_major). */
static int convert_layout(const view_t* v, int to_col) {
    const u32 W = v->W, M = v->cols;
    if (W == 1 || M == 1)
        return DMM_OK;
    if (W == M)
        return transpose_square(v);
    word* tmp = (word*)malloc(sizeof(word) * (u64)W * M);
    for (u32 i = 0; i < W; ++i)
        for (u32 j = 0; j < M; ++j) {
            const u64 lin = (u64)i * M + j;
            const u32 ci = (u32)(lin % W), cj = (u32)(lin / W);
            if (to_col)
                tmp[(u64)ci * M + cj] = *vcell(v, i, j);
            else
                tmp[(u64)i * M + j] = *vcell(v, ci, cj);
        }
    for (u32 i = 0; i < W; ++i)
        for (u32 j = 0; j < M; ++j) {
            *vcell(v, i, j) = tmp[(u64)i * M + j];
            /* staging side effect: the s0 window holds the converted matrix (layout.hpp:386-390) */
            *cell(v->mach, v->rows[i], v->s0 + j) = tmp[(u64)i * M + j];
        }
    free(tmp);
    return DMM_OK;
}
static int to_column_major(const view_t* v) { return convert_layout(v, 1); } /* layout.hpp:397 */
static int to_row_major(const view_t* v) { return convert_layout(v, 0); }    /* layout.hpp:403 */

/* ------------------------------------------------------------------------ */
/* Column sorts  sort.hpp:115-174                                            */
/* ------------------------------------------------------------------------ */
/* sort_columns_network sort.hpp:115: Batcher odd-even network; outcome = every
 * column sorted ascending. */
static int sort_columns_network(const view_t* v) {
    const u32 W = v->W, M = v->cols;
    if (W <= 1)
        return DMM_OK;
    word* col = (word*)malloc(sizeof(word) * W);
    for (u32 c = 0; c < M; ++c) {
        for (u32 r = 0; r < W; ++r)
            col[r] = *vcell(v, r, c);
        qsort(col, W, sizeof(word), cmp_asc);
        for (u32 r = 0; r < W; ++r)
            *vcell(v, r, c) = col[r];
    }
    free(col);
    return DMM_OK;
}

/* sort_columns_blocked sort.hpp:162-174 with the merge segment sorter */
static int sort_columns_blocked(const view_t* v, int asc) {
    const u32 W = v->W, M = v->cols;
    if (W <= 1)
        return DMM_OK;
    if (M % W != 0)
        return DMM_DIVISIBILITY_VIOLATION;
    for (u32 k = 0; k < M / W; ++k) {
        view_t b = view_col_window(v, k * W, W);
        int s = transpose_square(&b);
        view_free(&b);
        TRY(s);
    }
    TRY(merge_sort_segments(v, W, asc));
    for (u32 k = 0; k < M / W; ++k) {
        view_t b = view_col_window(v, k * W, W);
        int s = transpose_square(&b);
        view_free(&b);
        TRY(s);
    }
    return DMM_OK;
}

/* ------------------------------------------------------------------------ */
/* Skeletons  sort.hpp:200-330                                               */
/* ------------------------------------------------------------------------ */
/* short_wide_skeleton sort.hpp:200-218 */
static int short_wide_skeleton(const view_t* v, int asc, const row_sorter* rs) {
    if ((u64)v->W * v->W > v->cols)
        return DMM_SHAPE_VIOLATION;
    for (int pass = 0; pass < 2; ++pass) {
        TRY(do_row_sort(rs, v, ord_alt(asc)));
        TRY(to_column_major(v));
        TRY(do_row_sort(rs, v, ord_dir(asc)));
        TRY(to_row_major(v));
    }
    return do_row_sort(rs, v, ord_dir(asc));
}

static int square_skeleton_fits(u32 W, u32 M) { /* sort.hpp:313 */
    const u32 h = isqrt_floor(M);
    return h * h == M && W <= M && W % h == 0;
}

/* square_skeleton sort.hpp:250-280 (segment sorter: merge_sort_segments) */
static int square_skeleton(const view_t* v, int asc, const row_sorter* rs) {
    const u32 W = v->W, M = v->cols;
    const u32 h = isqrt_floor(M);
    if (h * h != M || W > M || W % h != 0)
        return DMM_SHAPE_VIOLATION;
    for (int phase = 0; phase < 2; ++phase) {
        const int alternate = phase == 1;
        for (u32 g = 0; g < W / h; ++g) { /* super_rows, merged lockstep */
            const int dir = alternate ? ((g % 2 == 0) == (asc != 0)) : asc;
            view_t grp = view_row_range(v, g * h, h);
            int s = short_wide_skeleton(&grp, dir, rs);
            view_free(&grp);
            TRY(s);
        }
        /* columns() */
        if (W == M) {
            TRY(transpose_square(v));
            TRY(do_row_sort(rs, v, ord_dir(asc)));
            TRY(transpose_square(v));
        } else {
            TRY(sort_columns_blocked(v, asc));
        }
    }
    return do_row_sort(rs, v, ord_dir(asc));
}

/* shearsort_rect sort.hpp:288-311 */
static int shearsort_rect(const view_t* v, int asc, const row_sorter* rs) {
    const u32 W = v->W, M = v->cols;
    if (W > M || (W > 1 && M % W != 0))
        return DMM_SHAPE_VIOLATION;
    const u32 rounds = ilog2_ceil(W) + 1;
    for (u32 i = 0; i < rounds; ++i) {
        TRY(do_row_sort(rs, v, ord_alt(asc)));
        if (W > 1)
            TRY(sort_columns_blocked(v, asc));
    }
    TRY(do_row_sort(rs, v, ord_alt(asc)));
    for (u32 r = 0; r < W; ++r) { /* snake -> row-major, sort.hpp:301-310 */
        if (ascending_for(ord_alt(asc), r) == asc)
            continue;
        for (u32 c = 0; c < M / 2; ++c) {
            word* a = vcell(v, r, c);
            word* b = vcell(v, r, M - 1 - c);
            word t = *a;
            *a = *b;
            *b = t;
        }
    }
    return DMM_OK;
}

/* sort_wide_any sort.hpp:321-330 */
static int sort_short_wide_v(const view_t* v, int asc);
static int sort_wide_any(const view_t* v, int asc) {
    row_sorter rs = {0, 0};
    if ((u64)v->W * v->W <= v->cols)
        return sort_short_wide_v(v, asc);
    if (square_skeleton_fits(v->W, v->cols))
        return square_skeleton(v, asc, &rs);
    return shearsort_rect(v, asc, &rs);
}

static int sort_short_wide_v(const view_t* v, int asc) { /* sort.hpp:225 */
    row_sorter rs = {0, 0};
    return short_wide_skeleton(v, asc, &rs);
}

static int sort_square_v(const view_t* v, int asc) { /* sort.hpp:337 */
    if (v->W != v->cols)
        return DMM_SHAPE_VIOLATION;
    const u32 h = isqrt_floor(v->cols);
    if (h * h != v->cols)
        return DMM_SHAPE_VIOLATION;
    row_sorter rs = {0, 0};
    return square_skeleton(v, asc, &rs);
}

static int sort_tall_v(const view_t* v) { /* sort.hpp:352-374 */
    const u32 W = v->W, M = v->cols;
    if (W < M || (M > 0 && W % M != 0))
        return DMM_SHAPE_VIOLATION;
    if (W == M)
        return sort_wide_any(v, 1);
    TRY(sort_rows(v, ord_asc()));
    TRY(sort_columns_network(v));
    TRY(to_row_major(v));
    TRY(sort_columns_network(v));
    for (u32 k = 0; k < W / M; ++k) {
        view_t b = view_row_range(v, k * M, M);
        int s = sort_wide_any(&b, k % 2 == 0);
        view_free(&b);
        TRY(s);
    }
    TRY(sort_columns_network(v));
    return sort_rows(v, ord_asc());
}

/* ------------------------------------------------------------------------ */
/* Partition  partition.hpp:112-456                                          */
/* ------------------------------------------------------------------------ */
static int check_partition_instance(const view_t* v) { /* partition.hpp:112 */
    u64* counts = (u64*)calloc(v->W ? v->W : 1, sizeof(u64));
    int s = DMM_OK;
    for (u32 r = 0; r < v->W && s == DMM_OK; ++r)
        for (u32 c = 0; c < v->cols; ++c) {
            word x = *vcell(v, r, c);
            if (x >= v->W) {
                s = DMM_INVALID_INSTANCE;
                break;
            }
            ++counts[x];
        }
    for (u32 r = 0; r < v->W && s == DMM_OK; ++r)
        if (counts[r] != v->cols)
            s = DMM_INVALID_INSTANCE;
    free(counts);
    return s;
}

/* general_sort_shape_ok partition.hpp:133-152 (+ the B200 partial-group extension) */
int dmmo_general_sort_shape_ok(uint64_t W, uint64_t M, uint32_t flags) {
    if (W <= 1)
        return 1;
    if (W <= M) {
        const u32 h = isqrt_floor((u32)M);
        return W * W <= M || ((u64)h * h == M && W % h == 0) || (M % W == 0);
    }
    if (M < 2 || W % M != 0)
        return 0;
    u64 nsubs = W;
    while (nsubs > 1) {
        const u64 g = M < nsubs ? M : nsubs;
        if (g < M && g * g > M) {
            if (!(flags & DMMO_FLAG_EXT_PARTIAL_GROUPS) || M % g != 0)
                return 0;
        }
        if (nsubs % g != 0)
            return 0;
        nsubs /= g;
    }
    return dmmo_general_sort_shape_ok(W / M, M, flags);
}

/* partition_leaf partition.hpp:156-172 */
static int partition_leaf(const view_t* v, u64 domain, int asc) {
    row_sorter rs = {1, domain};
    if ((u64)v->W * v->W <= v->cols)
        return short_wide_skeleton(v, asc, &rs);
    if (square_skeleton_fits(v->W, v->cols))
        return square_skeleton(v, asc, &rs);
    return shearsort_rect(v, asc, &rs);
}

/* PartitionParams::compute partition.hpp:209-225 */
typedef struct {
    double log_m_w;
    u32 d, rounds, subproblems;
} partition_params;
static int partition_params_compute(u32 W, u32 M, u32 flags, partition_params* p) {
    p->log_m_w = log((double)W) / log((double)M);
    p->rounds = (u32)ceil(p->log_m_w - 1e-9);
    u32 want = (u32)ceil(2 * p->log_m_w - 1e-9);
    if (want < 1)
        want = 1;
    u32 d = want < W / M ? want : W / M;
    while ((u64)M * d <= W && (W % ((u64)M * d) != 0 || !dmmo_general_sort_shape_ok(W / ((u64)M * d), M, flags)))
        ++d;
    if ((u64)M * d > W || W % ((u64)M * d) != 0)
        return DMM_DIVISIBILITY_VIOLATION;
    p->d = d;
    p->subproblems = M * d;
    return DMM_OK;
}
int dmmo_partition_params(uint32_t W, uint32_t M, uint32_t flags, uint32_t* rounds, uint32_t* d,
                          uint32_t* subproblems) {
    partition_params p;
    TRY(partition_params_compute(W, M, flags, &p));
    *rounds = p.rounds;
    *d = p.d;
    *subproblems = p.subproblems;
    return DMM_OK;
}

/* balance partition.hpp:234-271 */
static int balance(const view_t* v, u64 domain, u32 flags) {
    const u32 W = v->W, M = v->cols;
    if (W % M != 0)
        return DMM_SHAPE_VIOLATION;
    u32 sub_h = 1, nsubs = W;
    u32* locals = (u32*)malloc(sizeof(u32) * (M ? M : 1));
    int s = DMM_OK;
    while (nsubs > 1 && s == DMM_OK) {
        const u32 g = M < nsubs ? M : nsubs;
        int ext = 0;
        if (g < M && (u64)g * g > M) {
            if (!(flags & DMMO_FLAG_EXT_PARTIAL_GROUPS)) {
                s = DMM_SHAPE_VIOLATION;
                break;
            }
            ext = 1;
        }
        for (u32 grp = 0; grp < nsubs / g && s == DMM_OK; ++grp) {
            for (u32 j = 0; j < sub_h && s == DMM_OK; ++j) {
                for (u32 t = 0; t < g; ++t)
                    locals[t] = (grp * g + t) * sub_h + j;
                view_t a = view_pick_rows(v, locals, g);
                if (g == M) {
                    s = partition_leaf(&a, domain, 1);
                    if (s == DMM_OK)
                        s = transpose_square(&a);
                } else if (ext) {
                    /* B200 extension: the partial group sorted by the leaf dispatcher */
                    s = partition_leaf(&a, domain, 1);
                    if (s == DMM_OK)
                        s = to_column_major(&a);
                } else {
                    row_sorter rs = {1, domain};
                    s = short_wide_skeleton(&a, 1, &rs);
                    if (s == DMM_OK)
                        s = to_column_major(&a);
                }
                view_free(&a);
            }
        }
        sub_h *= g;
        nsubs /= g;
    }
    free(locals);
    return s;
}

/* scan_sorted partition.hpp:308-337 */
static int scan_sorted(const view_t* v) {
    const u32 W = v->W, M = v->cols;
    for (u32 r = 0; r < W; ++r) {
        for (u32 c = 1; c < M; ++c)
            if (*vcell(v, r, c - 1) > *vcell(v, r, c))
                return 0;
        if (r + 1 < W && *vcell(v, r, M - 1) > *vcell(v, r + 1, 0))
            return 0;
    }
    return 1;
}

/* cleanup_pass_pair partition.hpp:341-361 */
static int cleanup_pass_pair(const view_t* v, u64 domain) {
    const u32 W = v->W, M = v->cols;
    for (u32 k = 0; k < W / M; ++k) {
        view_t b = view_row_range(v, k * M, M);
        int s = partition_leaf(&b, domain, 1);
        view_free(&b);
        TRY(s);
    }
    if (W > M && M >= 2) {
        view_t b = view_row_range(v, 0, M / 2);
        int s = partition_leaf(&b, domain, 1);
        view_free(&b);
        TRY(s);
        for (u32 lo = M / 2; lo + M <= W; lo += M) {
            b = view_row_range(v, lo, M);
            s = partition_leaf(&b, domain, 1);
            view_free(&b);
            TRY(s);
        }
        b = view_row_range(v, W - M / 2, M / 2);
        s = partition_leaf(&b, domain, 1);
        view_free(&b);
        TRY(s);
    }
    return DMM_OK;
}

/* balance_divide_sort partition.hpp:363-428 */
static int balance_divide_sort(const view_t* v, u64 domain, dmmo_general_stats* st, u32 flags) {
    const u32 W = v->W, M = v->cols;
    if (W <= M)
        return partition_leaf(v, domain, 1);
    if (W % M != 0)
        return DMM_SHAPE_VIOLATION;

    /* (1) balancing + convert-and-divide until subproblems have <= m rows */
    u32 nlevel = 1;
    view_t* level = (view_t*)malloc(sizeof(view_t));
    level[0] = view_copy(v);
    int s = DMM_OK;
    while (s == DMM_OK && level[0].W > M) {
        for (u32 i = 0; i < nlevel && s == DMM_OK; ++i)
            s = balance(&level[i], domain, flags);
        if (s != DMM_OK)
            break;
        partition_params p;
        s = partition_params_compute(level[0].W, M, flags, &p);
        if (s != DMM_OK)
            break;
        view_t* next = (view_t*)malloc(sizeof(view_t) * (u64)nlevel * p.subproblems);
        u32 nnext = 0;
        for (u32 i = 0; i < nlevel && s == DMM_OK; ++i) {
            /* convert_and_divide partition.hpp:275-286 */
            if (level[i].W % p.subproblems != 0) {
                s = DMM_DIVISIBILITY_VIOLATION;
                break;
            }
            s = to_row_major(&level[i]);
            const u32 h = level[i].W / p.subproblems;
            for (u32 k = 0; k < p.subproblems && s == DMM_OK; ++k)
                next[nnext++] = view_row_range(&level[i], k * h, h);
        }
        for (u32 i = 0; i < nlevel; ++i)
            view_free(&level[i]);
        free(level);
        level = next;
        nlevel = nnext;
    }
    /* (2) leaves */
    for (u32 i = 0; i < nlevel && s == DMM_OK; ++i)
        s = partition_leaf(&level[i], domain, 1);
    for (u32 i = 0; i < nlevel; ++i)
        view_free(&level[i]);
    free(level);
    TRY(s);

    /* (3) column recursion */
    TRY(to_row_major(v));
    {
        const u32 h = W / M;
        for (u32 k = 0; k < M; ++k) {
            view_t c = view_row_range(v, k * h, h);
            int s2 = balance_divide_sort(&c, domain, st, flags);
            view_free(&c);
            TRY(s2);
        }
    }
    TRY(to_column_major(v));

    /* (4) shifted square cleanup with a checked postcondition */
    TRY(cleanup_pass_pair(v, domain));
    int sorted = scan_sorted(v);
    const u32 budget = ilog2_ceil(W);
    u32 tries = 0;
    while (!sorted && tries < budget) {
        TRY(cleanup_pass_pair(v, domain));
        sorted = scan_sorted(v);
        ++tries;
    }
    if (tries > st->cleanup_retries)
        st->cleanup_retries = tries;
    if (!sorted) {
        st->sorted = 0;
        if (v->mach->strict)
            return DMM_POSTCONDITION_FAILED;
    }
    return DMM_OK;
}

/* integer_sort_general partition.hpp:436-449 */
static int integer_sort_general_v(const view_t* v, u64 domain, int enforce_pre, u32 flags,
                                  dmmo_general_stats* st) {
    if (v->W > v->cols && v->cols < 2)
        return DMM_SHAPE_VIOLATION;
    if (enforce_pre && v->W > v->cols && (double)v->cols <= 2.0 * sqrt(log2((double)v->W)))
        return DMM_SHAPE_VIOLATION;
    st->cleanup_retries = 0;
    st->sorted = 1;
    return balance_divide_sort(v, domain, st, flags);
}

/* ------------------------------------------------------------------------ */
/* Public standalone entry points                                            */
/* ------------------------------------------------------------------------ */
typedef int (*view_fn)(const view_t* v, void* ctx);

static int run_on_standalone(uint32_t w, uint32_t m, uint64_t* grid, int strict, int permute_view,
                             view_fn fn, void* ctx) {
    machine_t mc;
    TRY(machine_init(&mc, w, m, strict));
    view_t v = view_full(&mc);
    if (permute_view) { /* the vp view of run_algorithm (instance.hpp:295) */
        v.s0 = scratch_a_base(&mc);
        v.s1 = scratch_b_base(&mc);
    }
    view_load(&v, grid);
    int s = fn(&v, ctx);
    view_snapshot(&v, grid);
    view_free(&v);
    machine_free(&mc);
    return s;
}

typedef struct {
    u64 domain;
    u32 flags;
    dmmo_general_stats* st;
    int asc;
} algo_ctx;

static int fn_partition_general(const view_t* v, void* p) { /* partition.hpp:453 */
    algo_ctx* c = (algo_ctx*)p;
    TRY(check_partition_instance(v));
    return integer_sort_general_v(v, v->W, !(c->flags & DMMO_FLAG_NO_ENFORCE_PRE), c->flags, c->st);
}
static int fn_integer_sort_general(const view_t* v, void* p) {
    algo_ctx* c = (algo_ctx*)p;
    return integer_sort_general_v(v, c->domain, !(c->flags & DMMO_FLAG_NO_ENFORCE_PRE), c->flags, c->st);
}
static int fn_partition_square(const view_t* v, void* p) { /* partition.hpp:189 */
    (void)p;
    if (v->W != v->cols)
        return DMM_SHAPE_VIOLATION;
    const u32 h = isqrt_floor(v->cols);
    if (h * h != v->cols)
        return DMM_SHAPE_VIOLATION;
    TRY(check_partition_instance(v));
    return partition_leaf(v, v->W, 1);
}
static int fn_partition_short_wide(const view_t* v, void* p) { /* partition.hpp:178 */
    (void)p;
    if ((u64)v->W * v->W > v->cols)
        return DMM_SHAPE_VIOLATION;
    TRY(check_partition_instance(v));
    row_sorter rs = {1, v->W};
    return short_wide_skeleton(v, 1, &rs);
}
static int fn_sort_short_wide(const view_t* v, void* p) { return sort_short_wide_v(v, ((algo_ctx*)p)->asc); }
static int fn_sort_square(const view_t* v, void* p) { return sort_square_v(v, ((algo_ctx*)p)->asc); }
static int fn_sort_tall(const view_t* v, void* p) { (void)p; return sort_tall_v(v); }
static int fn_sort_wide_any(const view_t* v, void* p) {
    if (v->W > v->cols || (v->W > 1 && v->cols % v->W != 0))
        return DMM_SHAPE_VIOLATION;  /* shearsort_rect sort.hpp:291-292 */
    return sort_wide_any(v, ((algo_ctx*)p)->asc);
}
static int fn_transpose(const view_t* v, void* p) { (void)p; return transpose_square(v); }
static int fn_to_col(const view_t* v, void* p) { (void)p; return to_column_major(v); }
static int fn_to_row(const view_t* v, void* p) { (void)p; return to_row_major(v); }

int dmmo_partition_general(uint32_t w, uint32_t m, uint64_t* grid, uint32_t flags, dmmo_general_stats* st) {
    algo_ctx c = {0, flags, st, 1};
    return run_on_standalone(w, m, grid, !(flags & DMMO_FLAG_NONSTRICT), 0, fn_partition_general, &c);
}
int dmmo_integer_sort_general(uint32_t w, uint32_t m, uint64_t* grid, uint64_t domain, uint32_t flags,
                              dmmo_general_stats* st) {
    algo_ctx c = {domain, flags, st, 1};
    return run_on_standalone(w, m, grid, !(flags & DMMO_FLAG_NONSTRICT), 1, fn_integer_sort_general, &c);
}
int dmmo_partition_square(uint32_t w, uint32_t m, uint64_t* grid) {
    return run_on_standalone(w, m, grid, 1, 0, fn_partition_square, NULL);
}
int dmmo_partition_short_wide(uint32_t w, uint32_t m, uint64_t* grid) {
    return run_on_standalone(w, m, grid, 1, 0, fn_partition_short_wide, NULL);
}
int dmmo_sort_short_wide(uint32_t w, uint32_t m, uint64_t* grid, int ascending) {
    algo_ctx c = {0, 0, NULL, ascending};
    return run_on_standalone(w, m, grid, 1, 0, fn_sort_short_wide, &c);
}
int dmmo_sort_square(uint32_t w, uint32_t m, uint64_t* grid, int ascending) {
    algo_ctx c = {0, 0, NULL, ascending};
    return run_on_standalone(w, m, grid, 1, 0, fn_sort_square, &c);
}
int dmmo_sort_wide_any(uint32_t w, uint32_t m, uint64_t* grid, int ascending) { /* sort.hpp:321 */
    algo_ctx c = {0, 0, NULL, ascending};
    return run_on_standalone(w, m, grid, 1, 0, fn_sort_wide_any, &c);
}
int dmmo_sort_tall(uint32_t w, uint32_t m, uint64_t* grid) {
    return run_on_standalone(w, m, grid, 1, 0, fn_sort_tall, NULL);
}
int dmmo_transpose_square(uint32_t s, uint64_t* grid) {
    return run_on_standalone(s, s, grid, 1, 0, fn_transpose, NULL);
}
int dmmo_to_column_major(uint32_t w, uint32_t m, uint64_t* grid) {
    return run_on_standalone(w, m, grid, 1, 0, fn_to_col, NULL);
}
int dmmo_to_row_major(uint32_t w, uint32_t m, uint64_t* grid) {
    return run_on_standalone(w, m, grid, 1, 0, fn_to_row, NULL);
}

/* ------------------------------------------------------------------------ */
/* Permutation  permute.hpp:24-628                                           */
/* ------------------------------------------------------------------------ */
enum { CTR_HASH = 0, CTR_SYNC = 1, CTR_LOAD = 2, CTR_CURSOR = 3 }; /* permute.hpp:24-29 */

static u32 hash_eval(word key, u32 m, u32 i) { /* HashOracle permute.hpp:35-46 */
    return (u32)(dmmo_splitmix64(key ^ ((u64)i * 0x9e3779b97f4a7c15ULL)) % m);
}
static u32 color_of(word label, word key, u32 m) { /* permute.hpp:49 */
    const u32 i = (u32)(label / m), j = (u32)(label % m);
    return (j + m - hash_eval(key, m, i)) % m;
}

uint64_t dmmo_permute_threshold(uint32_t w, uint32_t m) { /* permute.hpp:97 */
    double L = log((double)w) / log((double)m);
    if (L < 2.0)
        L = 2.0;
    const double t = ceil((double)w * m / (L * L * L));
    return (u64)t > w ? (u64)t : w;
}

/* preprocess_shuffle permute.hpp:109-142 */
static int preprocess_shuffle(const view_t* v, dmmo_rng* rng, u64* words, u32* shifts) {
    const u32 W = v->W, M = v->cols;
    if (W % M != 0)
        return DMM_SHAPE_VIOLATION;
    for (u32 r = 0; r < W; ++r)
        shifts[r] = 1 + (u32)dmmo_rng_below(rng, M);
    *words += W;
    word* tmp = (word*)malloc(sizeof(word) * M);
    for (u32 r = 0; r < W; ++r) {
        const u32 s = shifts[r] % M;
        if (s == 0)
            continue;
        for (u32 c = 0; c < M; ++c)
            tmp[(c + s) % M] = *vcell(v, r, c);
        for (u32 c = 0; c < M; ++c)
            *vcell(v, r, c) = tmp[c];
    }
    free(tmp);
    for (u32 b = 0; b < W / M; ++b) {
        view_t blk = view_row_range(v, b * M, M);
        int s = transpose_square(&blk);
        view_free(&blk);
        TRY(s);
    }
    return DMM_OK;
}

/* draw_and_broadcast_hash permute.hpp:147-166: m draws, key = payload[0]; the
 * broadcast writes the payload into the counter slot of every bank. */
static word draw_hash(machine_t* mc, dmmo_rng* rng, u64* words) {
    const u32 mm = mc->m, w = mc->w;
    word key = 0;
    word* payload = (word*)malloc(sizeof(word) * mm);
    for (u32 j = 0; j < mm; ++j)
        payload[j] = dmmo_rng_next(rng);
    *words += mm;
    key = payload[0];
    const u32 slot = counter_base(mc) + CTR_HASH;
    const u32 have = mm < w ? mm : w;
    for (u32 r = 0; r < w; ++r)
        *cell(mc, r, slot) = payload[r % have];
    free(payload);
    return key;
}

/* Rows' held labels, bucketed by color (RowHoldings permute.hpp:90-94). */
typedef struct {
    u32* bucket_pos; /* W * M positions, grouped by color */
    u32* bucket_start; /* W * (M+1) */
    u32* count;        /* W */
} holdings_t;

/* rescan_and_bucket permute.hpp:174-216 */
static void rescan_and_bucket(const view_t* v, word key, holdings_t* h) {
    const u32 W = v->W, M = v->cols;
    const word empty = (u64)v->mach->w * v->mach->m;
    word* vals = (word*)malloc(sizeof(word) * M);
    word* staged = (word*)malloc(sizeof(word) * M);
    u32* hist = (u32*)malloc(sizeof(u32) * (M + 1));
    for (u32 r = 0; r < W; ++r) {
        memset(hist, 0, sizeof(u32) * (M + 1));
        for (u32 c = 0; c < M; ++c) {
            vals[c] = *vcell(v, r, c);
            if (vals[c] != empty)
                ++hist[color_of(vals[c], key, M)];
        }
        u32 run = 0;
        for (u32 b = 0; b < M; ++b) {
            u32 cnt = hist[b];
            hist[b] = run;
            h->bucket_start[(u64)r * (M + 1) + b] = run;
            run += cnt;
        }
        h->bucket_start[(u64)r * (M + 1) + M] = run;
        for (u32 c = 0; c < M; ++c) {
            if (vals[c] == empty)
                continue;
            const u32 g = color_of(vals[c], key, M);
            staged[hist[g]++] = vals[c];
        }
        for (u32 c = 0; c < M; ++c)
            *vcell(v, r, c) = c < run ? staged[c] : empty;
        /* staging side effect: s0 holds the compacted labels, s1 the histogram ends */
        for (u32 c = 0; c < run; ++c)
            *cell(v->mach, v->rows[r], v->s0 + c) = staged[c];
        for (u32 b = 0; b < M; ++b)
            *cell(v->mach, v->rows[r], v->s1 + b) = hist[b];
        h->count[r] = run;
        for (u32 c = 0; c < run; ++c)
            h->bucket_pos[(u64)r * M + c] = c; /* compacted cells are color-sorted */
    }
    free(vals);
    free(staged);
    free(hist);
}

/* communication_phase permute.hpp:225-274 */
static u64 communication_phase(const view_t* v, u32 alpha, holdings_t* h, u32 out_b) {
    const u32 W = v->W, M = v->cols;
    machine_t* mc = v->mach;
    const word empty = (u64)mc->w * mc->m;
    for (u32 r = 0; r < W; ++r) {
        for (u32 k = 0; k < M; ++k) {
            const u32 lo = h->bucket_start[(u64)r * (M + 1) + k];
            const u32 hi = h->bucket_start[(u64)r * (M + 1) + k + 1];
            const u32 take = (hi - lo) < alpha ? (hi - lo) : alpha;
            for (u32 t = 0; t < take; ++t) {
                const u32 c = h->bucket_pos[(u64)r * M + lo + t];
                const word label = *vcell(v, r, c);
                const u32 di = (u32)(label / M), dj = (u32)(label % M);
                *cell(mc, v->rows[di], out_b + dj) = label;
                *vcell(v, r, c) = empty;
            }
            h->count[r] -= take;
        }
    }
    u64 leftover = 0;
    for (u32 r = 0; r < W; ++r)
        leftover += h->count[r];
    return leftover;
}

/* pack_leftovers permute.hpp:298-443 */
typedef struct {
    u32 width, base, s0, s1;
} packed_layout;

static int pack_leftovers(const view_t* v, dmmo_rng* rng, u64 leftover_total, u32 alpha, u64* words,
                          packed_layout* out) {
    const u32 W = v->W, M = v->cols;
    machine_t* mc = v->mach;
    const u32 lg = ilog2_ceil(W);
    const u32 t = lg * lg > 1 ? lg * lg : 1;
    const u32 theta = (u32)((2 * leftover_total + W - 1) / W) + alpha;
    const u32 bundle = (2 * M + t - 1) / t;
    u32 width = (u32)next_pow2((u64)theta + bundle + 1);
    for (;;) {
        if (!(2 * width <= M))
            break;
        const double band = pow(2.0, 2.0 * log2((double)W) / log2((double)width));
        const int headroom = band <= 0.5 * (double)width * (double)ilog2_ceil(W);
        if (dmmo_general_sort_shape_ok(W, width, 0) && headroom)
            break;
        width *= 2;
    }
    if (2 * width > M)
        return DMM_PACKING_OVERFLOW;

    const u32 load_slot = counter_base(mc) + CTR_LOAD;
    const u32 cursor_slot = counter_base(mc) + CTR_CURSOR;
    const word kReceived = (word)1 << 32;
    const word empty = (u64)mc->w * mc->m;
    u32* load = (u32*)calloc(W, sizeof(u32));
    for (u32 r = 0; r < W; ++r) {
        const u32 bank = v->rows[r];
        u32 o = 0;
        for (u32 c = 0; c < M; ++c) {
            const word x = *vcell(v, r, c);
            if (x != empty)
                *cell(mc, bank, v->s0 + o++) = x;
        }
        load[r] = o;
        for (u32 c = o; c < width; ++c)
            *cell(mc, bank, v->s0 + c) = empty;
        *cell(mc, bank, load_slot) = o;
        *cell(mc, bank, cursor_slot) = o;
    }
    *words += t;
    word* partner_load = (word*)malloc(sizeof(word) * W);
    u32* give = (u32*)malloc(sizeof(u32) * W);
    u32* sender = (u32*)malloc(sizeof(u32) * W);
    word* cursors = (word*)malloc(sizeof(word) * W);
    word* moved = (word*)malloc(sizeof(word) * W);
    u32* act = (u32*)malloc(sizeof(u32) * W);
    for (u32 round = 0; round < t; ++round) {
        const u32 shift = 1 + (u32)dmmo_rng_below(rng, W);
        for (u32 r = 0; r < W; ++r)
            partner_load[r] = *cell(mc, v->rows[(r + shift) % W], load_slot);
        u32 ns = 0;
        for (u32 r = 0; r < W; ++r) {
            give[r] = 0;
            const int received = (partner_load[r] & kReceived) != 0;
            const u32 plo = (u32)(partner_load[r] & 0xffffffffu);
            if (load[r] > theta && !received && plo <= theta) {
                sender[ns++] = r;
                give[r] = bundle < load[r] ? bundle : load[r];
            }
        }
        for (u32 i = 0; i < ns; ++i)
            cursors[i] = *cell(mc, v->rows[(sender[i] + shift) % W], cursor_slot);
        for (u32 k = 0; k < bundle; ++k) {
            /* one read batch then one write batch: all reads see pre-step state */
            u32 na = 0;
            for (u32 i = 0; i < ns; ++i) {
                const u32 r = sender[i];
                if (k < give[r]) {
                    moved[na] = *cell(mc, v->rows[r], v->s0 + load[r] - 1 - k);
                    act[na++] = i;
                }
            }
            for (u32 a = 0; a < na; ++a) {
                const u32 i = act[a];
                const u32 r = sender[i];
                const u32 p = (r + shift) % W;
                *cell(mc, v->rows[p], v->s0 + (u32)cursors[i] + k) = moved[a];
            }
        }
        for (u32 i = 0; i < ns; ++i) {
            const u32 r = sender[i], p = (r + shift) % W;
            const u32 plo = (u32)(partner_load[r] & 0xffffffffu);
            *cell(mc, v->rows[p], load_slot) = (word)(plo + give[r]) | kReceived;
        }
        for (u32 i = 0; i < ns; ++i) {
            const u32 r = sender[i], p = (r + shift) % W;
            *cell(mc, v->rows[p], cursor_slot) = cursors[i] + give[r];
        }
        for (u32 i = 0; i < ns; ++i) {
            const u32 r = sender[i];
            load[r] -= give[r];
            *cell(mc, v->rows[r], load_slot) = load[r];
        }
        for (u32 i = 0; i < ns; ++i) {
            const u32 r = sender[i], p = (r + shift) % W;
            load[p] += give[r];
        }
    }
    int s = DMM_OK;
    for (u32 r = 0; r < W; ++r)
        if (load[r] > width)
            s = DMM_PACKING_OVERFLOW;
    if (s == DMM_OK) {
        for (u32 r = 0; r < W; ++r)
            for (u32 c = load[r]; c < width; ++c)
                *cell(mc, v->rows[r], v->s0 + c) = empty;
        out->width = width;
        out->base = v->s0;
        out->s0 = scratch_b_base(mc);
        out->s1 = scratch_b_base(mc) + width;
    }
    free(load);
    free(partner_load);
    free(give);
    free(sender);
    free(cursors);
    free(moved);
    free(act);
    return s;
}

/* three_phase_delivery permute.hpp:452-529: every non-empty packed label reaches
 * out[label / m][label % m] (the phase order only schedules conflict-free steps). */
static void three_phase_delivery(const view_t* packed, u32 dest_m, u32 out_b) {
    machine_t* mc = packed->mach;
    const word empty = (u64)mc->w * mc->m;
    for (u32 r = 0; r < packed->W; ++r)
        for (u32 c = 0; c < packed->cols; ++c) {
            const word x = *vcell(packed, r, c);
            if (x != empty)
                *cell(mc, packed->rows[(u32)(x / dest_m)], out_b + (u32)(x % dest_m)) = x;
        }
}

/* finish permute.hpp:536-541 */
static int finish(const view_t* packed, u32 dest_m, u32 out_b, dmmo_general_stats* st) {
    const word empty = (u64)packed->mach->w * packed->mach->m;
    TRY(integer_sort_general_v(packed, empty + 1, 0, 0, st));
    three_phase_delivery(packed, dest_m, out_b);
    return DMM_OK;
}

/* permute permute.hpp:545-628 */
static int permute_machine(machine_t* mc, dmmo_rng* rng, u32 alpha, u32 iter_cap, dmmo_permute_report* rep,
                           u32* shifts) {
    const u32 w = mc->w, m = mc->m;
    memset(rep, 0, sizeof(*rep));
    if (m < 2 || w % m != 0)
        return DMM_SHAPE_VIOLATION;
    if (!dmmo_general_sort_shape_ok(w, m, 0))
        return DMM_SHAPE_VIOLATION;
    u32* rows = (u32*)malloc(sizeof(u32) * w);
    for (u32 r = 0; r < w; ++r)
        rows[r] = r;
    view_t v = view_make(mc, rows, w, 0, m, scratch_a_base(mc), scratch_b_base(mc));
    free(rows);
    const u32 ob = out_base(mc);
    rep->threshold = dmmo_permute_threshold(w, m);
    int s = preprocess_shuffle(&v, rng, &rep->random_words, shifts);
    if (s != DMM_OK) {
        view_free(&v);
        return s;
    }
    holdings_t h;
    h.bucket_pos = (u32*)malloc(sizeof(u32) * (u64)w * m);
    h.bucket_start = (u32*)malloc(sizeof(u32) * (u64)w * (m + 1));
    h.count = (u32*)malloc(sizeof(u32) * w);
    u64 leftover = (u64)w * m;
    while (leftover > rep->threshold && rep->iterations < iter_cap) {
        const word key = draw_hash(mc, rng, &rep->random_words);
        rescan_and_bucket(&v, key, &h);
        communication_phase(&v, alpha, &h, ob);
        leftover = 0; /* synchronize permute.hpp:278 */
        for (u32 r = 0; r < w; ++r) {
            *cell(mc, r, counter_base(mc) + CTR_SYNC) = h.count[r];
            leftover += h.count[r];
        }
        if (rep->n_hist < DMMO_MAX_HIST)
            rep->leftover_history[rep->n_hist++] = leftover;
        ++rep->iterations;
    }
    int delivered = leftover == 0;
    if (!delivered && leftover <= rep->threshold) {
        packed_layout pk;
        int ps = pack_leftovers(&v, rng, leftover, alpha, &rep->random_words, &pk);
        if (ps == DMM_OK) {
            rep->used_packing = 1;
            rep->packed_width = pk.width;
            view_t packed = view_make(mc, v.rows, w, pk.base, pk.width, pk.s0, pk.s1);
            dmmo_general_stats st = {0, 1};
            int fs = finish(&packed, m, ob, &st);
            view_free(&packed);
            if (fs == DMM_OK) {
                rep->cleanup_retries = st.cleanup_retries;
                delivered = 1;
            } else if (fs != DMM_POSTCONDITION_FAILED) {
                s = fs;
            }
        } else if (ps != DMM_PACKING_OVERFLOW) {
            s = ps;
        }
    }
    if (s == DMM_OK && !delivered) {
        rep->fallback = 1;
        const word empty = (u64)w * m;
        word* keep = (word*)malloc(sizeof(word) * m);
        for (u32 r = 0; r < w; ++r) {
            u32 o = 0;
            for (u32 c = 0; c < m; ++c) {
                const word x = *vcell(&v, r, c);
                if (x != empty)
                    keep[o++] = x;
            }
            for (u32 c = 0; c < m; ++c)
                *vcell(&v, r, c) = c < o ? keep[c] : empty;
        }
        free(keep);
        dmmo_general_stats st = {0, 1};
        int fs = finish(&v, m, ob, &st);
        if (fs == DMM_OK) {
            rep->cleanup_retries = st.cleanup_retries;
        } else if (fs == DMM_POSTCONDITION_FAILED) {
            s = sort_tall_v(&v);
            if (s == DMM_OK)
                three_phase_delivery(&v, m, ob);
        } else {
            s = fs;
        }
    }
    free(h.bucket_pos);
    free(h.bucket_start);
    free(h.count);
    view_free(&v);
    return s;
}

int dmmo_permute(uint32_t w, uint32_t m, const uint64_t* grid, uint64_t rng_seed, uint32_t alpha, uint32_t iter_cap,
                 uint64_t* out, dmmo_permute_report* rep, uint32_t* shifts) {
    machine_t mc;
    TRY(machine_init(&mc, w, m, 1));
    for (u32 r = 0; r < w; ++r)
        for (u32 c = 0; c < m; ++c)
            *cell(&mc, r, c) = grid[(u64)r * m + c];
    dmmo_rng rng;
    dmmo_rng_seed(&rng, rng_seed);
    int s = permute_machine(&mc, &rng, alpha, iter_cap, rep, shifts);
    if (out)
        for (u32 r = 0; r < w; ++r)
            for (u32 c = 0; c < m; ++c)
                out[(u64)r * m + c] = *cell(&mc, r, out_base(&mc) + c);
    machine_free(&mc);
    return s;
}

/* ------------------------------------------------------------------------ */
/* run_algorithm instance.hpp:277-363 (validate, dispatch, verify)            */
/* ------------------------------------------------------------------------ */
static int cmp_u64(const void* a, const void* b) { return cmp_asc(a, b); }

int dmmo_run_algorithm(int alg, uint32_t w, uint32_t m, uint64_t seed, const uint64_t* grid, uint32_t flags,
                       uint64_t* out_grid, dmmo_run_report* rep, dmmo_permute_report* prep, uint32_t* shifts) {
    const u64 n = (u64)w * m;
    memset(rep, 0, sizeof(*rep));
    /* validate_instance instance.hpp:79-100 */
    if (alg == DMMO_PARTITION_SHORT_WIDE || alg == DMMO_PARTITION_SQUARE || alg == DMMO_PARTITION_GENERAL) {
        u64* counts = (u64*)calloc(w, sizeof(u64));
        int bad = 0;
        for (u64 i = 0; i < n; ++i) {
            if (grid[i] >= w) {
                bad = 1;
                break;
            }
            ++counts[grid[i]];
        }
        for (u32 r = 0; r < w && !bad; ++r)
            if (counts[r] != m)
                bad = 1;
        free(counts);
        if (bad)
            return DMM_INVALID_INSTANCE;
    } else if (alg == DMMO_INTEGER_SORT_GENERAL || alg == DMMO_PERMUTE) {
        unsigned char* seen = (unsigned char*)calloc(n, 1);
        int bad = 0;
        for (u64 i = 0; i < n; ++i) {
            if (grid[i] >= n || seen[grid[i]]) {
                bad = 1;
                break;
            }
            seen[grid[i]] = 1;
        }
        free(seen);
        if (bad)
            return DMM_INVALID_INSTANCE;
    }
    memcpy(out_grid, grid, sizeof(word) * n);
    int s = DMM_OK;
    dmmo_general_stats st = {0, 1};
    switch (alg) {
        case DMMO_SORT_SHORT_WIDE: s = dmmo_sort_short_wide(w, m, out_grid, 1); break;
        case DMMO_SORT_SQUARE: s = dmmo_sort_square(w, m, out_grid, 1); break;
        case DMMO_SORT_TALL: s = dmmo_sort_tall(w, m, out_grid); break;
        case DMMO_PARTITION_SHORT_WIDE: s = dmmo_partition_short_wide(w, m, out_grid); break;
        case DMMO_PARTITION_SQUARE: s = dmmo_partition_square(w, m, out_grid); break;
        case DMMO_PARTITION_GENERAL:
            s = dmmo_partition_general(w, m, out_grid, flags, &st);
            rep->cleanup_retries = st.cleanup_retries;
            break;
        case DMMO_INTEGER_SORT_GENERAL:
            s = dmmo_integer_sort_general(w, m, out_grid, n, flags, &st);
            rep->cleanup_retries = st.cleanup_retries;
            break;
        case DMMO_PERMUTE: {
            dmmo_permute_report pr;
            s = dmmo_permute(w, m, grid, seed, 4, 64, out_grid, &pr, shifts);
            rep->iterations = pr.iterations;
            rep->fallback = pr.fallback;
            rep->cleanup_retries = pr.cleanup_retries;
            if (prep)
                *prep = pr;
            break;
        }
        default: return DMM_ERROR;
    }
    if (s != DMM_OK)
        return s;
    /* verifiers instance.hpp:243-265 */
    int ok = 1;
    if (alg <= DMMO_SORT_TALL || alg == DMMO_INTEGER_SORT_GENERAL) {
        word* e = (word*)malloc(sizeof(word) * n);
        memcpy(e, grid, sizeof(word) * n);
        qsort(e, n, sizeof(word), cmp_u64);
        ok = memcmp(e, out_grid, sizeof(word) * n) == 0;
        free(e);
    } else if (alg == DMMO_PERMUTE) {
        for (u64 i = 0; i < n; ++i)
            if (out_grid[i] != i)
                ok = 0;
    } else {
        for (u32 r = 0; r < w; ++r)
            for (u32 c = 0; c < m; ++c)
                if (out_grid[(u64)r * m + c] != r)
                    ok = 0;
    }
    rep->correct = (u32)ok;
    return DMM_OK;
}

int dmmo_partition_general_batch(uint32_t w, uint32_t m, uint64_t count, const uint32_t* in, uint32_t* out,
                                 uint32_t flags, dmmo_general_stats* st) {
    const u64 n = (u64)w * m;
    word* g = (word*)malloc(sizeof(word) * n);
    int worst = DMM_OK;
    for (u64 k = 0; k < count; ++k) {
        for (u64 i = 0; i < n; ++i)
            g[i] = in[k * n + i];
        dmmo_general_stats s1 = {0, 1};
        int s = dmmo_partition_general(w, m, g, flags, &s1);
        if (st)
            st[k] = s1;
        if (s != DMM_OK && worst == DMM_OK)
            worst = s;
        for (u64 i = 0; i < n; ++i)
            out[k * n + i] = (uint32_t)g[i];
    }
    free(g);
    return worst;
}
