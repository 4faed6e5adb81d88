/*
 * vnm_oracle.c — plain, slow, obviously-correct CPU oracle for the V:N:M sparse linear layer.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path (paper_2410_16135_b200/) never
 * links, imports or calls it, and it shares no source, header, table or helper with csrc/.
 *
 * Citation keys: P:n = /root/reference/PAPER.md line n; S:n = /root/reference/SPEC.md line n.
 * Readings of the paper (Q1..Q18) are listed in DESIGN.md §3.
 *
 * What it computes (step numbers O1..O9 as in DESIGN.md §3):
 *   O1  explicit zero-padding of W (and score) to rows_p x cols_p            (§3 "Acceleration")
 *   O2  importance e = |s|, s = score or float(W) (ABS criterion)            (§3 step 1)
 *   O3  column L1 of e over the V rows of each V x M block, fp32, summed in the
 *       canonical stride-halving tree order (reading Q3)                      (§3 step 2)
 *   O4  keep the 4 columns of largest L1; ties -> smaller column index      (§3 step 2)
 *   O5  per row keep the 2 largest e among the kept 4; ties -> smaller index (§3 step 3)
 *   O6  pack: A_n (2 values per block per row, left to right), A_i1 (4 column
 *       indices per block, ascending), A_i2 (2-bit positions, nibble lo|hi<<2) (App. A)
 *   O7  unpack                                                               (App. A)
 *   O8  Y^T[o][t] = sum_k x[k][t] * W'[o][k] in fp64, plus A = sum_k |x w'|   (Y = X W'^T, W' = W (.) M)
 *   O9  the same product computed from the packed arrays only (gather x rows) (App. A)
 *
 * Packed layout (identical to include/vnm.h, but written here independently):
 *   rows_p = ceil(rows/V)*V, cols_p = ceil(cols/M)*M, nb = cols_p/M, nb_pad = ceil(nb/8)*8
 *   values  bf16 [rows_p][2*nb_pad]     pad blocks: 0
 *   col_idx u8   [rows_p/V][nb_pad][4]  pad blocks: 0,1,2,3
 *   meta    u32  [rows_p][nb_pad/8]     nibble (b%8) of word b/8 = lo | hi<<2 ; pad blocks: 0x4
 *   mask    u32  [rows_p][ceil(cols_p/32)], bit c%32 of word c/32; bits >= cols_p are 0
 *
 * Compiled with -O2 -ffp-contract=off -fno-fast-math (see build.sh); OpenMP only over independent
 * V-blocks / output rows, never inside a reduction.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define VNMO_OK 0
#define VNMO_ERR_ARG (-1)
#define VNMO_ERR_SHAPE (-2)

typedef struct {
    int32_t rows, cols, V, M;
    int32_t rows_p, cols_p, nb, nb_pad;
    int32_t ld_val, ld_meta, ld_mask;
} vnmo_geom;

static float bf16_bits_to_float(uint16_t h) {
    uint32_t u = ((uint32_t)h) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return f;
}

static int32_t ceil_to(int32_t a, int32_t m) { return ((a + m - 1) / m) * m; }

int vnmo_geometry(int32_t rows, int32_t cols, int32_t V, int32_t M, vnmo_geom* g) {
    if (!g) return VNMO_ERR_ARG;
    if (rows < 0 || cols < 0 || V < 1 || M < 4) return VNMO_ERR_SHAPE;
    g->rows = rows; g->cols = cols; g->V = V; g->M = M;
    g->rows_p = ceil_to(rows, V);
    g->cols_p = ceil_to(cols, M);
    g->nb = g->cols_p / M;
    g->nb_pad = ceil_to(g->nb, 8);
    g->ld_val = 2 * g->nb_pad;
    g->ld_meta = ceil_to(g->nb_pad / 8, 4);  /* DESIGN.md reading Q20: rows padded to 16 B */
    g->ld_mask = (g->cols_p + 31) / 32;
    return VNMO_OK;
}

/* O1 + O2: the padded importance matrix E[rows_p][cols_p], e = |s|, zero outside the logical extent. */
static float* importance_padded(const uint16_t* W, int64_t ldw, const float* score, int64_t lds,
                                const vnmo_geom* g) {
    float* E = (float*)calloc((size_t)g->rows_p * (size_t)g->cols_p, sizeof(float));
    if (!E) return NULL;
    for (int32_t r = 0; r < g->rows; ++r)
        for (int32_t c = 0; c < g->cols; ++c) {
            float s = score ? score[(int64_t)r * lds + c] : bf16_bits_to_float(W[(int64_t)r * ldw + c]);
            E[(int64_t)r * g->cols_p + c] = fabsf(s);
        }
    return E;
}

/* O3: L1 of column c of block (vb, b): stride-halving tree over the V rows (zero-padded to a power of
 * two, which adds exact zeros):  for stride = P/2, P/4, ..., 1:  s[r] = s[r] + s[r + stride], r < stride. */
static float column_l1_tree(const float* E, const vnmo_geom* g, int32_t vb, int32_t b, int32_t c) {
    int32_t P = 1;
    while (P < g->V) P <<= 1;
    float* s = (float*)calloc((size_t)P, sizeof(float));
    for (int32_t r = 0; r < g->V; ++r)
        s[r] = E[(int64_t)(vb * g->V + r) * g->cols_p + (int64_t)b * g->M + c];
    for (int32_t stride = P / 2; stride >= 1; stride /= 2)
        for (int32_t r = 0; r < stride; ++r)
            s[r] = s[r] + s[r + stride];
    float out = s[0];
    free(s);
    return out;
}

/* O4: the 4 columns of largest L1, ties toward the smaller column index; returned ascending. */
static void top4_columns(const float* L, int32_t M, uint8_t kept[4]) {
    int chosen[64] = {0};
    for (int k = 0; k < 4; ++k) {
        int best = -1;
        for (int c = 0; c < M; ++c) {
            if (chosen[c]) continue;
            if (best < 0 || L[c] > L[best]) best = c;  /* strict '>' keeps the smaller index on ties */
        }
        chosen[best] = 1;
    }
    int n = 0;
    for (int c = 0; c < M; ++c)
        if (chosen[c]) kept[n++] = (uint8_t)c;
}

/* O5: among the 4 kept positions of one row, the 2 of largest e, ties toward the smaller position. */
static void top2_positions(const float e4[4], uint8_t* lo, uint8_t* hi) {
    int first = 0;
    for (int j = 1; j < 4; ++j)
        if (e4[j] > e4[first]) first = j;
    int second = -1;
    for (int j = 0; j < 4; ++j) {
        if (j == first) continue;
        if (second < 0 || e4[j] > e4[second]) second = j;
    }
    *lo = (uint8_t)(first < second ? first : second);
    *hi = (uint8_t)(first < second ? second : first);
}

/* S_{V:N:M} (§3): writes the mask bits, and optionally kept[rows_p/V][nb][4] and
 * pos[rows_p][nb][2] (the intermediate decisions, for tests). */
int vnmo_prune(const uint16_t* W, int64_t ldw, const float* score, int64_t lds,
               int32_t rows, int32_t cols, int32_t V, int32_t M,
               uint32_t* mask, uint8_t* kept_out, uint8_t* pos_out) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    if (M > 64) return VNMO_ERR_SHAPE;
    if (!mask || (!W && !score)) return VNMO_ERR_ARG;
    float* E = importance_padded(W, ldw, score, lds, &g);
    if (!E) return VNMO_ERR_ARG;
    memset(mask, 0, sizeof(uint32_t) * (size_t)g.rows_p * (size_t)g.ld_mask);
    const int32_t nvb = g.rows_p / V;
#pragma omp parallel for schedule(static)
    for (int32_t vb = 0; vb < nvb; ++vb) {
        float L[64];
        for (int32_t b = 0; b < g.nb; ++b) {
            for (int32_t c = 0; c < M; ++c) L[c] = column_l1_tree(E, &g, vb, b, c);
            uint8_t kept[4];
            top4_columns(L, M, kept);
            if (kept_out)
                for (int j = 0; j < 4; ++j) kept_out[((int64_t)vb * g.nb + b) * 4 + j] = kept[j];
            for (int32_t i = 0; i < V; ++i) {
                int32_t r = vb * V + i;
                float e4[4];
                for (int j = 0; j < 4; ++j) e4[j] = E[(int64_t)r * g.cols_p + (int64_t)b * M + kept[j]];
                uint8_t lo, hi;
                top2_positions(e4, &lo, &hi);
                if (pos_out) {
                    pos_out[((int64_t)r * g.nb + b) * 2 + 0] = lo;
                    pos_out[((int64_t)r * g.nb + b) * 2 + 1] = hi;
                }
                int32_t c0 = b * M + kept[lo], c1 = b * M + kept[hi];
                mask[(int64_t)r * g.ld_mask + c0 / 32] |= 1u << (c0 % 32);
                mask[(int64_t)r * g.ld_mask + c1 / 32] |= 1u << (c1 % 32);
            }
        }
    }
    free(E);
    return VNMO_OK;
}

static int mask_bit(const uint32_t* mask, const vnmo_geom* g, int32_t r, int32_t c) {
    return (int)((mask[(int64_t)r * g->ld_mask + c / 32] >> (c % 32)) & 1u);
}

/* O6: pack.  Returns 0, or 1 + (vb*nb + b) of the first block whose mask is not a valid V:N:M mask
 * (a row without exactly 2 bits, more than 4 columns carrying bits); if every block is valid but a
 * bit is set at a column >= cols_p, 1 + rows_p/V*nb.  A_i1 = the columns carrying the block's bits, ascending; when fewer
 * than 4 columns carry bits it is completed with the lowest-index remaining columns (reading Q19). */
int vnmo_pack(const uint16_t* W, int64_t ldw, const uint32_t* mask,
              int32_t rows, int32_t cols, int32_t V, int32_t M,
              uint16_t* values, uint8_t* col_idx, uint32_t* meta) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    if (M > 64) return VNMO_ERR_SHAPE;
    if (!W || !mask || !values || !col_idx || !meta) return VNMO_ERR_ARG;
    const int32_t nvb = g.rows_p / V;
    int64_t first_bad = -1;
    for (int32_t vb = 0; vb < nvb && first_bad < 0; ++vb) {
        for (int32_t b = 0; b < g.nb_pad; ++b) {
            uint8_t ci[4] = {0, 1, 2, 3};
            if (b < g.nb) {
                int used[64] = {0};
                int nused = 0;
                for (int32_t i = 0; i < V; ++i) {
                    int cnt = 0;
                    for (int32_t c = 0; c < M; ++c)
                        if (mask_bit(mask, &g, vb * V + i, b * M + c)) { cnt++; if (!used[c]) { used[c] = 1; nused++; } }
                    if (cnt != 2) { first_bad = (int64_t)vb * g.nb + b; break; }
                }
                if (first_bad >= 0) break;
                if (nused > 4) { first_bad = (int64_t)vb * g.nb + b; break; }
                /* complete to 4 columns with the lowest unused indices, then list ascending */
                for (int32_t c = 0; c < M && nused < 4; ++c)
                    if (!used[c]) { used[c] = 1; nused++; }
                int n = 0;
                for (int32_t c = 0; c < M; ++c)
                    if (used[c]) ci[n++] = (uint8_t)c;
            }
            for (int j = 0; j < 4; ++j) col_idx[((int64_t)vb * g.nb_pad + b) * 4 + j] = ci[j];
            for (int32_t i = 0; i < V; ++i) {
                int32_t r = vb * V + i;
                uint8_t p[2] = {0, 1};
                uint16_t v[2] = {0, 0};
                if (b < g.nb) {
                    int n = 0;
                    for (int j = 0; j < 4; ++j) {
                        int32_t c = b * M + ci[j];
                        if (mask_bit(mask, &g, r, c)) {
                            p[n] = (uint8_t)j;
                            v[n] = (r < rows && c < cols) ? W[(int64_t)r * ldw + c] : (uint16_t)0;
                            n++;
                        }
                    }
                }
                values[(int64_t)r * g.ld_val + 2 * b + 0] = v[0];
                values[(int64_t)r * g.ld_val + 2 * b + 1] = v[1];
                uint32_t nib = (uint32_t)p[0] | ((uint32_t)p[1] << 2);
                uint32_t* w = &meta[(int64_t)r * g.ld_meta + b / 8];
                if (b % 8 == 0) *w = 0;
                *w |= nib << (4 * (b % 8));
            }
        }
    }
    /* words past the nb_pad/8 block words of a row (Q20): eight pad blocks, nibble 0x4 each */
    for (int32_t r = 0; r < g.rows_p; ++r)
        for (int32_t w = g.nb_pad / 8; w < g.ld_meta; ++w) meta[(int64_t)r * g.ld_meta + w] = 0x44444444u;
    if (first_bad >= 0) return (int)(1 + first_bad);
    /* bits beyond cols_p (checked after the blocks: the status is the lowest error index) */
    for (int32_t r = 0; r < g.rows_p; ++r)
        for (int32_t c = g.cols_p; c < g.ld_mask * 32; ++c)
            if (mask_bit(mask, &g, r, c)) return 1 + nvb * g.nb;
    return VNMO_OK;
}

/* O7: unpack the packed arrays into the dense masked weight W' (bf16 bits) [rows_p][cols_p]. */
int vnmo_unpack(const uint16_t* values, const uint8_t* col_idx, const uint32_t* meta,
                int32_t rows, int32_t cols, int32_t V, int32_t M, uint16_t* Wout) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    memset(Wout, 0, sizeof(uint16_t) * (size_t)g.rows_p * (size_t)g.cols_p);
    for (int32_t r = 0; r < g.rows_p; ++r)
        for (int32_t b = 0; b < g.nb; ++b) {
            uint32_t nib = (meta[(int64_t)r * g.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
            uint32_t lo = nib & 3u, hi = nib >> 2;
            if (lo >= hi) return VNMO_ERR_ARG;
            const uint8_t* ci = &col_idx[((int64_t)(r / V) * g.nb_pad + b) * 4];
            for (int j = 0; j < 3; ++j)
                if (ci[j] >= ci[j + 1]) return VNMO_ERR_ARG;
            if (ci[3] >= M) return VNMO_ERR_ARG;
            Wout[(int64_t)r * g.cols_p + b * M + ci[lo]] = values[(int64_t)r * g.ld_val + 2 * b + 0];
            Wout[(int64_t)r * g.cols_p + b * M + ci[hi]] = values[(int64_t)r * g.ld_val + 2 * b + 1];
        }
    return VNMO_OK;
}

/* O8: Y^T[o][t] = sum_k x[k][t] * W'[o][k] in fp64 (k ascending) and A[o][t] = sum_k |x[k][t] W'[o][k]|.
 * XT: bf16 [cols][ldx] (feature-major); Wm: bf16 [rows][ldw]; outputs [rows][T]. */
int vnmo_gemm_ref(const uint16_t* XT, int64_t ldx, int32_t T, const uint16_t* Wm, int64_t ldw,
                  int32_t rows, int32_t cols, double* YT, double* AT) {
    if (!XT || !Wm || !YT) return VNMO_ERR_ARG;
#pragma omp parallel for schedule(static)
    for (int32_t o = 0; o < rows; ++o) {
        double* y = &YT[(int64_t)o * T];
        double* a = AT ? &AT[(int64_t)o * T] : NULL;
        for (int32_t t = 0; t < T; ++t) { y[t] = 0.0; if (a) a[t] = 0.0; }
        for (int32_t k = 0; k < cols; ++k) {
            double w = (double)bf16_bits_to_float(Wm[(int64_t)o * ldw + k]);
            if (w == 0.0) continue; /* exact: adding +-0 products changes nothing but the sign of zero */
            const uint16_t* x = &XT[(int64_t)k * ldx];
            for (int32_t t = 0; t < T; ++t) {
                double p = (double)bf16_bits_to_float(x[t]) * w;
                y[t] += p;
                if (a) a[t] += fabs(p);
            }
        }
    }
    return VNMO_OK;
}

/* O8 on sampled outputs: for each pair i, Y[i] = sum_k x[k][t_i] W'[o_i][k], A[i] likewise. */
int vnmo_gemm_ref_sampled(const uint16_t* XT, int64_t ldx, const uint16_t* Wm, int64_t ldw, int32_t cols,
                          const int32_t* o_idx, const int32_t* t_idx, int64_t n, double* Y, double* A) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double y = 0.0, a = 0.0;
        for (int32_t k = 0; k < cols; ++k) {
            double p = (double)bf16_bits_to_float(XT[(int64_t)k * ldx + t_idx[i]]) *
                       (double)bf16_bits_to_float(Wm[(int64_t)o_idx[i] * ldw + k]);
            y += p;
            a += fabs(p);
        }
        Y[i] = y;
        if (A) A[i] = a;
    }
    return VNMO_OK;
}

/* O9: Y^T from the packed arrays only: for each row o and block b, gather the two x rows
 * b*M + col_idx[o/V][b][pos] and multiply by the stored values (App. A).
 * x rows at k >= cols are zero (implicit padding).  Output [rows][T] fp64. */
int vnmo_spmm_packed(const uint16_t* XT, int64_t ldx, int32_t T,
                     const uint16_t* values, const uint8_t* col_idx, const uint32_t* meta,
                     int32_t rows, int32_t cols, int32_t V, int32_t M, double* YT) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
#pragma omp parallel for schedule(static)
    for (int32_t o = 0; o < rows; ++o) {
        double* y = &YT[(int64_t)o * T];
        for (int32_t t = 0; t < T; ++t) y[t] = 0.0;
        for (int32_t b = 0; b < g.nb; ++b) {
            uint32_t nib = (meta[(int64_t)o * g.ld_meta + b / 8] >> (4 * (b % 8))) & 0xFu;
            const uint8_t* ci = &col_idx[((int64_t)(o / V) * g.nb_pad + b) * 4];
            for (int i = 0; i < 2; ++i) {
                uint32_t pos = i == 0 ? (nib & 3u) : (nib >> 2);
                int32_t k = b * M + ci[pos];
                if (k >= cols) continue;
                double w = (double)bf16_bits_to_float(values[(int64_t)o * g.ld_val + 2 * b + i]);
                const uint16_t* x = &XT[(int64_t)k * ldx];
                for (int32_t t = 0; t < T; ++t) y[t] += (double)bf16_bits_to_float(x[t]) * w;
            }
        }
    }
    return VNMO_OK;
}

/* helper for tests: W (.) mask as bf16 bits [rows][cols] (logical extent). */
int vnmo_apply_mask(const uint16_t* W, int64_t ldw, const uint32_t* mask, int32_t rows, int32_t cols,
                    int32_t V, int32_t M, uint16_t* Wm) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    for (int32_t r = 0; r < rows; ++r)
        for (int32_t c = 0; c < cols; ++c)
            Wm[(int64_t)r * cols + c] = mask_bit(mask, &g, r, c) ? W[(int64_t)r * ldw + c] : (uint16_t)0;
    return VNMO_OK;
}

/* retained score: sum of e over mask bits, fp64 (order irrelevant for the test values). */
double vnmo_retained_score(const float* score, int64_t lds, const uint32_t* mask,
                           int32_t rows, int32_t cols, int32_t V, int32_t M) {
    vnmo_geom g;
    if (vnmo_geometry(rows, cols, V, M, &g)) return -1.0;
    double s = 0.0;
    for (int32_t r = 0; r < rows; ++r)
        for (int32_t c = 0; c < cols; ++c)
            if (mask_bit(mask, &g, r, c)) s += fabs((double)score[(int64_t)r * lds + c]);
    return s;
}

/* ---------------------------------------------------------------------------------------------------
 * RIA importance, the step before the path for TS1/TS3 masks:
 *   Eq. (1):  RIA_ij = ( |W_ij| / sum_r |W_rj| + |W_ij| / sum_c |W_ic| ) * ( ||X_j||_2 )^a
 * with the SPEC reading of the activation index (input channel j = column of W) and of
 * zero sums (a fraction with a zero denominator is 0).  Computed in fp64 and rounded to fp32 once
 * (the precision is not fixed by the paper; reading Q21).
 *   vnmo_act_norms:  norms[j] = sqrt( sum_t x[j][t]^2 ), X^T bf16 [cols][ldx] (feature-major)
 *   vnmo_ria:        score fp32 [rows][lds]; act == NULL means ||X_j|| = 1 for every j (S:166 default)
 * ------------------------------------------------------------------------------------------------- */
int vnmo_act_norms(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, double* norms) {
    if (!XT || !norms || cols < 0 || T < 0 || ldx < T) return VNMO_ERR_ARG;
    for (int32_t j = 0; j < cols; ++j) {
        double s = 0.0;
        for (int32_t t = 0; t < T; ++t) {
            const double x = (double)bf16_bits_to_float(XT[(int64_t)j * ldx + t]);
            s += x * x;
        }
        norms[j] = sqrt(s);
    }
    return VNMO_OK;
}

int vnmo_ria(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, const double* act, double a,
             float* score, int64_t lds, double* score64 /* nullable: the fp64 values before rounding */) {
    if (!W || !score || rows < 0 || cols < 0 || ldw < cols || lds < cols) return VNMO_ERR_ARG;
    double* colsum = (double*)calloc((size_t)cols + 1, sizeof(double));
    double* rowsum = (double*)calloc((size_t)rows + 1, sizeof(double));
    if (!colsum || !rowsum) { free(colsum); free(rowsum); return VNMO_ERR_ARG; }
    for (int32_t i = 0; i < rows; ++i)
        for (int32_t j = 0; j < cols; ++j) {
            const double w = fabs((double)bf16_bits_to_float(W[(int64_t)i * ldw + j]));
            rowsum[i] += w;   /* sum_c |W_ic|: output channel i */
            colsum[j] += w;   /* sum_r |W_rj|: input channel j  */
        }
    for (int32_t i = 0; i < rows; ++i)
        for (int32_t j = 0; j < cols; ++j) {
            const double w = fabs((double)bf16_bits_to_float(W[(int64_t)i * ldw + j]));
            const double f1 = colsum[j] > 0.0 ? w / colsum[j] : 0.0;
            const double f2 = rowsum[i] > 0.0 ? w / rowsum[i] : 0.0;
            const double act_j = act ? act[j] : 1.0;
            const double s = (f1 + f2) * pow(act_j, a);
            score[(int64_t)i * lds + j] = (float)s;
            if (score64) score64[(int64_t)i * cols + j] = s;
        }
    free(colsum);
    free(rowsum);
    return VNMO_OK;
}

/* ---------------------------------------------------------------------------------------------------
 * Channel-permutation gain scores: the cost matrix of the linear sum assignment
 * that approximates the input-permutation step, Eq. (7) `eq:admm1` (LSA modelling P:213):
 *   cost[j][b*M + s] = sum over V-row stripes of the retained score contributed by channel j when it
 *   replaces the occupant of slot s of column block b (every other column frozen) and the block is
 *   re-pruned by S_{V:N:M} (column L1 top-4, then per-row top-2; §3, the same decision rules
 *   and the same fp32 stride-halving L1 as vnmo_prune).
 * "Contributed by channel j" = the sum of e_j over the rows that keep slot s (reading Q22), so
 * that with the identity assignment the costs add up to the retained score of the actual pruning.
 * score fp32 [rows][lds] (e = |score|, zero-padded to rows_p x cols_p); cost fp64 [cols_p][cols_p].
 * ------------------------------------------------------------------------------------------------- */
int vnmo_permute_gain(const float* score, int64_t lds, int32_t rows, int32_t cols, int32_t V, int32_t M,
                      double* cost) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    if (!score || !cost || M > 64) return VNMO_ERR_ARG;
    float* E = importance_padded(NULL, 0, score, lds, &g);
    if (!E) return VNMO_ERR_ARG;
    const int32_t K = g.cols_p, nvb = g.rows_p / V;
    int32_t P = 1;
    while (P < V) P <<= 1;
#pragma omp parallel for schedule(dynamic)
    for (int32_t j = 0; j < K; ++j) {
        float* s = (float*)malloc(sizeof(float) * (size_t)P);
        float* col = (float*)malloc(sizeof(float) * (size_t)V * (size_t)M);  /* hypothetical block [V][M] */
        float L[64];
        for (int32_t b = 0; b < g.nb; ++b)
            for (int32_t sl = 0; sl < M; ++sl) {
                double acc = 0.0;
                for (int32_t vb = 0; vb < nvb; ++vb) {
                    for (int32_t i = 0; i < V; ++i)
                        for (int32_t c = 0; c < M; ++c)
                            col[i * M + c] = E[(int64_t)(vb * V + i) * K + (c == sl ? j : b * M + c)];
                    for (int32_t c = 0; c < M; ++c) {  /* O3: the stride-halving tree of the block's columns */
                        for (int32_t r = 0; r < P; ++r) s[r] = r < V ? col[r * M + c] : 0.0f;
                        for (int32_t stride = P / 2; stride >= 1; stride /= 2)
                            for (int32_t r = 0; r < stride; ++r) s[r] = s[r] + s[r + stride];
                        L[c] = s[0];
                    }
                    uint8_t kept[4];
                    top4_columns(L, M, kept);
                    int ks = -1;
                    for (int q = 0; q < 4; ++q)
                        if (kept[q] == sl) ks = q;
                    if (ks < 0) continue;  /* slot s pruned in this stripe */
                    for (int32_t i = 0; i < V; ++i) {
                        float e4[4];
                        for (int q = 0; q < 4; ++q) e4[q] = col[i * M + kept[q]];
                        uint8_t lo, hi;
                        top2_positions(e4, &lo, &hi);
                        if (lo == ks || hi == ks) acc += (double)col[i * M + sl];
                    }
                }
                cost[(int64_t)j * K + (int64_t)b * M + sl] = acc;
            }
        free(s);
        free(col);
    }
    free(E);
    return VNMO_OK;
}

/* ------------------------------------------------------------------------------------------------------------
 * Output-channel permutation gain (Eq. (8) `eq:admm2`, §4.2: P_o^{k+1} =
 * argmax_{P_o} sum RIA(S_{V:N:M}(P_o W P_i^k)), "approximately modeled as the traditional linear sum assignment
 * problem"; "V:N:M sparsity allows both input and output CP to affect the retained norm";
 * SPEC solve_output_perm S:382-389; reading Q23).
 *
 * cost[i][g*V + s] = the retained score that ROW i contributes when it replaces the occupant of slot s of V-row
 * stripe g (every other row frozen) and the stripe is re-pruned by S_{V:N:M}: in every column block b the stripe's
 * 4 columns of largest L1 (fp32, the canonical stride-halving tree over the stripe's V rows with row i at position
 * s; ties -> smaller column) are kept, then row i keeps the 2 largest e among them (ties -> smaller position);
 * the contribution is the sum over blocks (ascending) of those 2 kept e (ascending column) in fp64.  With every
 * row in its own slot the costs add up to the retained score of the actual pruning.
 * score fp32 [rows][lds] (e = |score|, zero-padded to rows_p x cols_p); cost fp64 [rows_p][rows_p].
 * ------------------------------------------------------------------------------------------------------------ */
int vnmo_permute_gain_out(const float* score, int64_t lds, int32_t rows, int32_t cols, int32_t V, int32_t M,
                          double* cost) {
    vnmo_geom g;
    int st = vnmo_geometry(rows, cols, V, M, &g);
    if (st) return st;
    if (!score || !cost || M > 64) return VNMO_ERR_ARG;
    float* E = importance_padded(NULL, 0, score, lds, &g);
    if (!E) return VNMO_ERR_ARG;
    const int32_t K = g.cols_p, R = g.rows_p;
    int32_t P = 1;
    while (P < V) P <<= 1;
#pragma omp parallel for schedule(dynamic)
    for (int32_t i = 0; i < R; ++i) {
        float* s = (float*)malloc(sizeof(float) * (size_t)P);
        float* blk = (float*)malloc(sizeof(float) * (size_t)V * (size_t)M);  /* the hypothetical stripe block [V][M] */
        float L[64];
        for (int32_t gs = 0; gs < R; ++gs) {
            const int32_t vb = gs / V, sl = gs % V;
            double acc = 0.0;
            for (int32_t b = 0; b < g.nb; ++b) {
                for (int32_t r = 0; r < V; ++r)
                    for (int32_t c = 0; c < M; ++c)
                        blk[r * M + c] = E[(int64_t)(r == sl ? i : vb * V + r) * K + (int64_t)b * M + c];
                for (int32_t c = 0; c < M; ++c) {  /* O3: the stride-halving tree of the block's column */
                    for (int32_t r = 0; r < P; ++r) s[r] = r < V ? blk[r * M + c] : 0.0f;
                    for (int32_t stride = P / 2; stride >= 1; stride /= 2)
                        for (int32_t r = 0; r < stride; ++r) s[r] = s[r] + s[r + stride];
                    L[c] = s[0];
                }
                uint8_t kept[4];
                top4_columns(L, M, kept);
                float e4[4];
                for (int q = 0; q < 4; ++q) e4[q] = blk[sl * M + kept[q]];
                uint8_t lo, hi;
                top2_positions(e4, &lo, &hi);
                acc += (double)e4[lo];
                acc += (double)e4[hi];
            }
            cost[(int64_t)i * R + gs] = acc;
        }
        free(s);
        free(blk);
    }
    free(E);
    return VNMO_OK;
}
