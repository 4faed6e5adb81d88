/*
 * vnm.h — C ABI of the B200-native V:N:M sparse linear layer (arXiv 2410.16135).
 *
 * The method (§3 "Preliminary"; App. A):
 *   S_{V:N:M}: within every V x M block of W keep the 4 columns whose L1 norm of importance scores is
 *   largest, then keep the 2 largest scores of each row among those 4.  The deployment
 *   path pads W, converts it to the compressed form A_n / A_i1 / A_i2, and runs
 *   the V:N:M SpMM on sparse tensor cores.
 *
 * Conventions (all calls):
 *   - Every data pointer is a DEVICE pointer owned by the caller (e.g. a torch tensor); the library
 *     allocates no device memory and keeps no device state (TMA descriptors are encoded on the host per call,
 *     passed as kernel parameters).
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *   - Argument / shape / alignment errors are detected on the host and returned before any launch.
 *     Data-dependent errors (a mask that violates the V:N:M pattern) are written to `d_status`.
 *   - bf16 tensors are passed as uint16_t bit patterns.  Leading dimensions (ld*) are in ELEMENTS.
 *   - Inputs must be finite; NaN/Inf behaviour is unspecified.
 *   - Identical inputs give byte-identical outputs.
 *   - Thread-safe.
 *
 * Padding: W, score and X^T are read with their logical extents and are zero outside;
 * all packed outputs use the padded geometry of vnm_geom.  Padded rows/columns are pruned like real
 * ones (their scores are 0), pad blocks (nb <= b < nb_pad) hold values 0, col_idx {0,1,2,3} and the
 * 2:4 nibble 0x4; mask bits at columns >= cols_p are 0.  See DESIGN.md §4 for every layout.
 */
#ifndef VNM_H_
#define VNM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* vnm_stream_t; /* == cudaStream_t */

typedef enum {
    VNM_OK = 0,
    VNM_ERR_ARG = -1,         /* NULL pointer where one is required, bad enum value              */
    VNM_ERR_SHAPE = -2,       /* V, M, rows, cols, T, ld out of range                            */
    VNM_ERR_ALIGN = -3,       /* pointer not 16-byte aligned / ld not a multiple of 8 (4 for fp32) */
    VNM_ERR_UNSUPPORTED = -4, /* valid per the method but not implemented (e.g. vnm_spmm V != 64)  */
    VNM_ERR_CUDA = -5         /* a CUDA launch / driver call failed                              */
} vnm_status;

typedef enum { VNM_F32 = 0, VNM_BF16 = 1 } vnm_dtype;

/* Padded geometry.  N (=2) is implicit ("N≡2").
 *   rows_p = ceil(rows/V)*V      cols_p = ceil(cols/M)*M      nb = cols_p/M (column blocks per row)
 *   nb_pad = ceil(nb/8)*8        (one u32 of metadata = 8 blocks = one 32-wide sparse MMA K step)
 *   ld_val = 2*nb_pad (bf16)     ld_meta = ceil(nb_pad/8 / 4)*4 (u32, rows of 16 B multiples)
 *   ld_mask = ceil(cols_p/32) (u32)                                                                  */
typedef struct {
    int32_t rows, cols, V, M;
    int32_t rows_p, cols_p, nb, nb_pad;
    int32_t ld_val, ld_meta, ld_mask;
} vnm_geom;

/* The compressed form (App. A).  Borrowed device pointers:
 *   values  (A_n)  bf16 [rows_p][ld_val]       the 2 kept values of each block of each row, left to right
 *   col_idx (A_i1) u8   [rows_p/V][nb_pad][4]  the block's 4 column indices (0..M-1), strictly ascending
 *   meta    (A_i2) u32  [rows_p][ld_meta]      nibble (b%8) of word b/8 = pos_lo | pos_hi<<2, pos in 0..3
 *                                              indexes col_idx, pos_lo < pos_hi; words nb_pad/8 ..
 *                                              ld_meta-1 of a row hold 0x44444444 (reading Q20)
 * A_i1 lists the columns that carry the block's nonzeros; when fewer than 4 do (always possible,
 * e.g. V = 1) it is completed with the lowest-index remaining columns (reading Q19), so the
 * packed form is a function of the mask alone.                                                        */
typedef struct {
    vnm_geom g;
    uint16_t* values;
    uint8_t* col_idx;
    uint32_t* meta;
    /* Optional tensor-core form of the same weights (NULL if absent), filled by vnm_pack_tc; used by
     * vnm_spmm for large T when 4 <= M <= 8 (DESIGN.md §6 "window form").  Every V x M block becomes an
     * 8-row window of X^T (the block's M channels followed by 8-M channels of the next block) holding two
     * 2:4 groups (channels 0-3 and 4-7); the row's two nonzeros sit in their own channels, the other
     * positions carry zero values.  This lets M = 128 sparse MMAs share one dense, TMA-loaded X^T tile
     * instead of gathering per V-block.  Any 32 <= V <= 128: each row's metadata selects within the window, so rows
 * of different V-blocks share the tile.  Layouts (rows_w = ceil(rows_p/128)*128, bpm = M == 4 ? 8 : 4
     * blocks per MMA, n_mma_w = nb_pad/bpm, n_stage_w = ceil(n_mma_w/4)):
     *   values_tc bf16 [rows_w][16*n_mma_w]       4 values per block (M >= 5: lo pair, hi pair); = A_n for M = 4
     *   meta_tc   u32  [rows_w/128][n_stage_w][128][4]   2:4 metadata of MMA (stage*4 + k) in the M = 128
     *             TMEM lane order (lane L holds rows (L%8)+16(L/16) and +8, K-groups 4((L/8)%2)..+3).
     * For M % 4 == 0 with M > 8 (e.g. 64:2:16) the tensor-core form is the NATURAL 2:4 form instead: a
     * block is a whole number of 4-channel groups, so each group holds at most the row's 2 nonzeros and the
     * masked W is 2:4-sparse in channel order; values_tc / meta_tc are the M = 4 layouts above over the
     * groups (2 values per group, zero-completed; nb_pad -> ceil(cols_p/4 / 8)*8 groups).
     * For the other 8 < M < 16 (e.g. the paper's 128:2:9 / 10 / 11 / 13, tab:bs-sped P:656-665) it is the
     * WINDOW-16 form: every block is a 16-row window of X^T (the block's M channels and 16-M of the next) as
     * four 2:4 groups, zero-completed like the window form; MMA 2j + h reads the half-windows h (groups 2h,
     * 2h+1) of blocks 4j .. 4j+3, so n_mma_w = nb_pad/2 and values_tc holds 8 values per block (half 0 of
     * blocks 4j.. at MMA 2j, half 1 at MMA 2j + 1), meta_tc the same lane layout.                          */
    uint16_t* values_tc;
    uint32_t* meta_tc;
} vnm_packed;

/* Host, pure.  Ranges: rows, cols >= 0; V a power of two in [1, 256]; 4 <= M <= 32.
 * VNM_ERR_SHAPE otherwise.                                                                             */
vnm_status vnm_geometry(int32_t rows, int32_t cols, int32_t V, int32_t M, vnm_geom* out);

/* Bytes of one buffer for geometry g: which = 0 values, 1 col_idx, 2 meta, 3 mask, 4 values_tc, 5 meta_tc
 * (4 and 5 are 0 when the tensor-core form does not apply: V < 32, V > 128, or M > 16 with M % 4 != 0).
 * 0 on bad input.                                                                                     */
size_t vnm_bytes(const vnm_geom* g, int which);

/* S_{V:N:M} (§3) -> mask bits.
 *   W      bf16 [g->rows][ldw], 16-B aligned, ldw % 8 == 0, ldw >= cols
 *   score  fp32 [g->rows][lds] or NULL (NULL = ABS criterion, e = |W|); 16-B aligned, lds % 4 == 0
 *   mask   u32  [rows_p][ld_mask] (written completely)
 * Importance e = |score| (or |W|); column L1 summed in fp32 in the canonical stride-halving tree order
 * (Q3); ties at both steps go to the smaller index.                                */
vnm_status vnm_prune(const uint16_t* W, int64_t ldw, const float* score, int64_t lds, const vnm_geom* g,
                     uint32_t* mask, vnm_stream_t stream);

/* Compress W with a given mask into A_n / A_i1 / A_i2.
 *   W, ldw as above; mask u32 [rows_p][ld_mask]; out->g must equal *g and its pointers must be set.
 *   d_status: NULL or one int32 in device memory; receives 0 if the mask is a valid V:N:M mask, else
 *   1 + (vb*nb + b) of the first (lowest-index) invalid block (a row without exactly 2 bits in the
 *   block, or more than 4 columns carrying bits), or 1 + (rows_p/V)*nb if a bit is set at a column
 *   >= cols_p.  The packed outputs are unspecified when the mask is invalid.                            */
vnm_status vnm_compress(const uint16_t* W, int64_t ldw, const uint32_t* mask, const vnm_geom* g,
                        vnm_packed* out, int32_t* d_status, vnm_stream_t stream);

/* Fused vnm_prune + vnm_compress in one pass over W (byte-identical outputs).  mask may be NULL.
 * If out->values_tc / out->meta_tc are set (32 <= V <= 128, and M < 16 or M % 4 == 0) the tensor-core form is
 * written too: the window form (M <= 8), the window-16 form (other M < 16) and the natural 2:4 form at M = 16 in
 * the same pass (32 <= V <= 128), the other natural 2:4 forms (M % 4 == 0) by a second launch
 * (identical to vnm_pack_tc of the result).                                                             */
vnm_status vnm_prune_compress(const uint16_t* W, int64_t ldw, const float* score, int64_t lds,
                              const vnm_geom* g, vnm_packed* out, uint32_t* mask, vnm_stream_t stream);

/* vnm_prune_compress of n weights in ONE launch (e.g. every linear layer of a model at a mask update: the
 * mask + compression pass is re-run for all layers at once).  Entry i has the meaning of one
 * vnm_prune_compress call: W[i] / ldw[i] / score[i] (NULL: ABS) / lds[i] / out[i] (out[i]->g is the geometry)
 * / mask[i] (NULL: none).  Outputs are byte-identical to n separate calls.  1 <= n <= 8 weights sharing one
 * (V, M) run as one kernel when 32 <= V <= 128 and M <= 8; other batches run as n launches on `stream`.
 * Errors: VNM_ERR_ARG (n < 1 or n > 64, NULL arrays), else the first failing entry's status (nothing launched). */
vnm_status vnm_prune_compress_batched(int32_t n, const uint16_t* const* W, const int64_t* ldw,
                                      const float* const* score, const int64_t* lds, vnm_packed* const* out,
                                      uint32_t* const* mask, vnm_stream_t stream);

/* Fill P->values_tc / P->meta_tc (caller-allocated, vnm_bytes 4 / 5) from the canonical A_n / A_i1 / A_i2
 * of P.  VNM_ERR_UNSUPPORTED unless 32 <= V <= 128 and (M < 16 or M % 4 == 0); VNM_ERR_ARG if a tc pointer
 * is NULL.                                                                                            */
vnm_status vnm_pack_tc(const vnm_packed* P, vnm_stream_t stream);

/* The V:N:M SpMM (App. A):  Y^T[o][t] = sum_k W'[o][k] * X^T[k][t],  W' = unpack(P).
 *   XT  bf16 [P->g.cols][ldx]  feature-major activations (tokens contiguous), 16-B aligned, ldx % 8 == 0
 *   T   tokens, 0 <= T <= ldx
 *   YT  [P->g.rows][ldy]  fp32 (y_dtype VNM_F32) or bf16 (VNM_BF16, round-to-nearest-even), 16-B aligned,
 *       ldy % 8 == 0, ldy >= T; only rows < g.rows and columns < T are written.
 * bf16 x bf16 products, fp32 accumulation on the sparse tensor cores (tcgen05.mma.sp).
 * Supported: 1 <= T <= 32 with V >= 16 and any M; V = 64, 128, 256 with any M at any T (e.g. the paper's 128:2:M,
 * SURVEY §8(f) NEXT-1); 32 <= V <= 128 at any T when the tensor-core form is present (M < 16, or M % 4 == 0;
 * the window-16 form with a Y^T row that is not a multiple of 16 bytes takes the small-T / gather plan);
 * VNM_ERR_UNSUPPORTED otherwise.
 * Plans: tensor-core form present and T > 64 (or V != 64 beyond the small-T range) -> a window-form kernel (dense
 * X^T tiles by TMA; a Y^T row of T tokens that is not a multiple of 16 bytes takes the pair kernel whose stores are
 * element-wise at the tail, so nothing past column T is ever written):
 * CTA pairs with the row pair's A resident for short K (tcgen05.mma.sp.cta_group::2, M = 256), CTA pairs
 * streaming A, or single CTAs (M = 128) — chosen by shape from measurements;
 * 1 <= T <= 32, V >= 16, any M -> the small-T kernel (canonical A_n / A_i1 / A_i2 streamed by TMA, warp-level sparse
 * MMAs whose B fragments are gathered from a dense X^T slice by ldmatrix, stream-K over (128-row group, 32-block
 * stage) units); otherwise (V = 64) the gather kernel (M = 64 sparse MMAs on the 4 kept X^T rows of each block,
 * 16-byte cp.async gathers).
 * workspace: optional device scratch (16-B aligned) for the split-K plans; pass NULL/0 to let the library run
 * without it (the small-T plan then gives every CTA whole row groups).  vnm_spmm_workspace_bytes(g, T) is the
 * size a call can use.  Layout: a fixed 16 KB region of completion tickets at offset 0, fp32 partials after it.
 * The tickets must be zero when a call starts: zero the workspace once with vnm_spmm_workspace_init (or allocate
 * it zero-filled); every completed call leaves the tickets zero again (the partials are not cleared and need not
 * be), so ONE workspace sized for the largest (g, T) serves all later calls of any geometry ordered on the stream
 * (no per-call memset).  Re-initialise after a failed launch; use one workspace per concurrently running call. */
vnm_status vnm_spmm(const uint16_t* XT, int64_t ldx, int32_t T, const vnm_packed* P, void* YT, int64_t ldy,
                    vnm_dtype y_dtype, void* workspace, size_t workspace_bytes, vnm_stream_t stream);

size_t vnm_spmm_workspace_bytes(const vnm_geom* g, int32_t T);

/* n INDEPENDENT vnm_spmm problems sharing T and y_dtype (a grouped SpMM, e.g. the q / k / v projections or the
 * gate / up projections of one decode step — layers whose inputs do not depend on each other's outputs):
 * entry i has the meaning of vnm_spmm(XT[i], ldx[i], T, P[i], YT[i], ldy[i], y_dtype, ...).  Consecutive groups
 * of up to 4 problems that all take the small-T plan (1 <= T <= 32, V >= 16) with one V class (all V >= 64, or
 * equal V) run as ONE launch of the small-T kernel over the concatenated (problem, row group, stage) unit list —
 * one prologue, one pipeline fill and one stream-K tail for the group instead of one per layer; any other group
 * runs as one vnm_spmm per problem, in order, on `stream`.  Results are identical to n vnm_spmm calls up to the
 * fp32 summation order of the K pieces (deterministic for a given batch).  workspace: as for vnm_spmm, sized by
 * vnm_spmm_batched_workspace_bytes (one workspace serves the whole call).
 * flags: 0, or VNM_SPMM_WEIGHTS_READY — the caller guarantees every P[i]'s arrays were completely written before
 * the kernel that precedes this call on `stream` began (e.g. weights pruned once, or at least two launches
 * earlier): the small-T launch then issues the weight loads of its first pipeline fill before waiting for that
 * kernel (programmatic dependent launch), hiding them behind its tail; X^T, Y^T and the workspace are still only
 * touched after the wait.  Errors: VNM_ERR_ARG (n < 1 or n > 64, NULL arrays, unknown flag bits), else the first
 * invalid entry's vnm_spmm status (nothing launched).                                                   */
#define VNM_SPMM_WEIGHTS_READY 1u
vnm_status vnm_spmm_batched(int32_t n, const uint16_t* const* XT, const int64_t* ldx, int32_t T,
                            const vnm_packed* const* P, void* const* YT, const int64_t* ldy, vnm_dtype y_dtype,
                            uint32_t flags, void* workspace, size_t workspace_bytes, vnm_stream_t stream);
size_t vnm_spmm_batched_workspace_bytes(int32_t n, const vnm_geom* const* g, int32_t T);

/* Zero-fill a vnm_spmm workspace (asynchronous on stream).  VNM_ERR_ARG if ws is NULL with bytes > 0.     */
vnm_status vnm_spmm_workspace_init(void* ws, size_t bytes, vnm_stream_t stream);

/* ---- RIA importance: the score pre-pass for vnm_prune / vnm_prune_compress.
 * Eq. (1), §3 P:86-90:
 *     RIA_ij = ( |W_ij| / sum_r |W_rj| + |W_ij| / sum_c |W_ic| ) * ( ||X_j||_2 )^a
 * Readings (Q16, Q21): ||X_j|| is the L2 norm over tokens of INPUT channel j (the column of W,
 * SPEC S:165); a zero row / column sum makes its fraction 0; fp32 arithmetic.
 *
 * vnm_act_norms: norms[j] = ||X^T[j][0..T)||_2 for j < cols.  XT bf16 [cols][ldx] (16-B aligned), norms fp32
 *   [cols] (4-B aligned, caller-owned).
 * vnm_ria_score: score fp32 [rows][lds] (16-B aligned, lds % 4 == 0) from W bf16 [rows][ldw] (16-B aligned,
 *   ldw % 8 == 0); act_norms fp32 [cols] or NULL (all ones: the activation factor is 1); a >= 0
 *   (0.5 in the cited RIA work).  workspace: caller-owned device scratch of at least
 *   vnm_ria_workspace_bytes(rows, cols) bytes, 16-B aligned.  Deterministic (fixed summation order).  */
vnm_status vnm_act_norms(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, float* norms, vnm_stream_t stream);
size_t vnm_ria_workspace_bytes(int32_t rows, int32_t cols);
vnm_status vnm_ria_score(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, const float* act_norms, float a,
                         float* score, int64_t lds, void* workspace, size_t workspace_bytes, vnm_stream_t stream);

/* ---- Channel-permutation gain scores: the cost matrix of the linear sum assignment
 * that approximates the input-permutation step of the V:N:M-specific channel permutation, Eq. (7)
 * `eq:admm1` (§4.2; "approximately modeled as the traditional linear sum assignment
 * problem").  The Hungarian solve stays with the caller (host).
 *   cost[j][b*M + s] = sum over the V-row stripes of the retained score that input channel j contributes when
 *   it replaces the occupant of slot s of column block b (every other column frozen) and the block is
 *   re-pruned by S_{V:N:M} (same tie rules and fp32 L1 tree as vnm_prune); "contributes" = the sum
 *   of e_j = |score[.][j]| over the rows that keep slot s (reading Q22).  With the identity
 *   assignment the costs add up to the retained score of the pruned matrix.
 *   score fp32 [g->rows][lds] (4-B aligned), cost fp32 [g->cols_p][ldc], ldc >= cols_p (caller-owned);
 *   workspace >= vnm_permute_gain_workspace_bytes(g), 16-B aligned.  V <= 128, any M (VNM_ERR_UNSUPPORTED for
 *   V = 256).  Deterministic (fp32 sums in stripe order).                                              */
size_t vnm_permute_gain_workspace_bytes(const vnm_geom* g);
vnm_status vnm_permute_gain(const float* score, int64_t lds, const vnm_geom* g, float* cost, int64_t ldc,
                            void* workspace, size_t workspace_bytes, vnm_stream_t stream);

/* ---- The OUTPUT-channel half of the V:N:M-specific channel permutation: the LSA cost of
 * Eq. (8) `eq:admm2` (§4.2; "V:N:M sparsity allows both input and output CP to affect the
 * retained norm").
 *   cost[i][g*V + s] = the retained score ROW i contributes when it replaces the occupant of slot s of V-row
 *   stripe g (every other row frozen) and the stripe is re-pruned by S_{V:N:M} (same tie rules and fp32
 *   L1 tree as vnm_prune): in each column block row i keeps its 2 largest |score| among the stripe's 4 kept columns
 *   (reading Q23).  With the identity assignment the costs add up to the retained score.
 *   score fp32 [g->rows][lds] (4-B aligned), cost fp32 [g->rows_p][ldc], ldc >= rows_p (caller-owned).  V <= 128,
 *   any M (VNM_ERR_UNSUPPORTED for V = 256).  Deterministic (fp32 sums in column-block order).               */
vnm_status vnm_permute_gain_out(const float* score, int64_t lds, const vnm_geom* g, float* cost, int64_t ldc,
                                vnm_stream_t stream);

/* Human-readable text of a status (static storage).                                                   */
const char* vnm_status_string(vnm_status s);

/* Number of kernel launches the library issued since load (for the bench's gpu_launches count).       */
uint64_t vnm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* VNM_H_ */
