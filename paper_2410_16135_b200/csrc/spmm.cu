// spmm.cu — the V:N:M SpMM  Y^T = W' X^T  on the 5th-generation sparse tensor cores (SURVEY §8(a)
// rows a6-a8; §3 "Acceleration of V:N:M sparsity" P:106-109 and App. A: "retrieve the
// retained weights and the corresponding tiles of the input matrix B ... align the data layout with
// that of a 2:4-sparse MM").
//
// Work unit (tile) = one V-block (64 rows of W) x NT tokens.  K is walked in stages of 32 column blocks
// (4 sparse MMAs of logical K = 32 = 8 blocks each).  Persistent CTAs (one per SM) walk the tiles in
// token-tile-major order so the CTAs resident at any time share X^T rows in L2.  Warp roles:
//   warps 8-15 gather: the 4 kept X^T rows of each block (A_i1) -> the stage's B tile, written straight
//              into the MN-major 128B-swizzled UMMA layout by 16-byte cp.async (zero fill past T tokens and
//              past the logical channels: the implicit padding of P:107-108); each thread's copies arrive
//              on the stage barrier asynchronously (cp.async.mbarrier.arrive.noinc).  TMA tile::gather4 was
//              measured at only 7-15 B/clk/SM (csrc/probes2.cu MB3b) and is not used;
//   warp 16    TMA: the stage's A_n tile (64 x 64 bf16, 128B swizzle, K-major);
//   warps 4-7  metadata: A_i2 words -> TMEM in the M=64 sparse-metadata layout (tcgen05.st);
//   warp 17    one thread issues tcgen05.mma.sp.cta_group::1.kind::f16 M=64 N=NT into TMEM;
//   warps 0-3  epilogue: tcgen05.ld -> fp32 / bf16 -> Y^T.
// Two accumulators share TMEM columns: accumulator a (a = tile parity) and its metadata live in lanes
// 16a..16a+15 of every 32-lane sub-partition, so the epilogue of tile i overlaps the MMAs of tile i+1.
//
// TMEM layouts (measured on B200 by csrc/probes*.cu):
//   D (M=64):  row m -> lane 16a + (m % 16) + 32 * (m / 16), column n.
//   E (M=64):  nibble (row m, K-group g) = nibble 4*((m/8)%2) + g%4 of the word at lane
//              16a + (m % 8) + 8*(g/4) + 32*(m/16), column e_col + id2 (e_col even).
//   D and E must carry the same lane offset (0 or 16).
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kV = 64;
constexpr int kBlocksPerStage = 32;
constexpr int kMmaPerStage = kBlocksPerStage / 8;
constexpr int kKRowsPerStage = 4 * kBlocksPerStage;  // 128 gathered X^T rows per stage
constexpr int kGatherWarps = 8;
constexpr int kEpiWarp0 = 0, kMetaWarp0 = 4, kGatherWarp0 = 8, kProdWarp = 16, kMmaWarp = 17;
constexpr int kThreads = 32 * 18;
constexpr uint32_t kMetaCol = 256;
constexpr uint32_t kABytes = kV * 128;

struct SpmmArgs {
    const uint16_t* XT;
    int64_t ldx;
    int32_t cols;
    const uint8_t* col_idx;
    const uint32_t* meta;
    void* YT;
    int64_t ldy;
    int32_t T;
    int32_t y_bf16;
    int32_t rows, M, nb_pad, ld_meta, nvb, ntt, ntiles;
    // split-K (small T): unit u = (tile u / ks_n, K-slice u % ks_n of sps stages); partial sums go to
    // ws[k][row][t] (fp32) and a second kernel adds the ks_n slices in order (deterministic)
    int32_t ks_n, sps, nunits;
    float* ws;
};

template <int NT>
struct Cfg {
    static constexpr int kBBytes = kKRowsPerStage * NT * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = NT == 256 ? 3 : (NT == 128 ? 5 : 8);
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 512;
};

// arrive on `bar` once every cp.async this thread issued so far has landed (count pre-set in mbar_init)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1)
    vnm_spmm_kernel(const __grid_constant__ CUtensorMap tmap_a, const SpmmArgs a) {
    using C = Cfg<NT>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + S * kABytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* meta_ready = empty + S;
    uint64_t* tmem_full = meta_ready + S;  // [2]
    uint64_t* tmem_empty = tmem_full + 2;  // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int n_mma = a.ld_meta;
    const int n_stage = (n_mma + kMmaPerStage - 1) / kMmaPerStage;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 32 * kGatherWarps + 1);
            mbar_init(&empty[s], 1);
            mbar_init(&meta_ready[s], 4);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tmem_full[i], 1);
            mbar_init(&tmem_empty[i], 4);
        }
        fence_mbar_init();
    }
    if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
    if (warp == kProdWarp && lane == 0) tma_prefetch_desc(&tmap_a);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp >= kGatherWarp0 && warp < kGatherWarp0 + kGatherWarps) {
        // ------------------------------------------------------------ gather producers (B = kept X^T rows)
        // Warp pw owns blocks 4pw..4pw+3 of every stage (gathered rows 16pw..16pw+15); each lane moves 16 B
        // (8 tokens) per cp.async, zero-filled past T (tokens) and past cols (padded channels).
        constexpr int CPR = NT / 8;       // 16-byte chunks per gathered row
        constexpr int RPI = 32 / CPR;     // rows per warp instruction
        const int pw = warp - kGatherWarp0;
        const int sub = lane / CPR, ch = lane % CPR;
        const uint32_t dst_chunk = (ch / 8) * (kKRowsPerStage * 128);
        int q = 0;
        for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
            const int tile = u / a.ks_n, k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
            const int vb = tile % a.nvb, n0 = (tile / a.nvb) * NT;
            const uint32_t* ci_vb = reinterpret_cast<const uint32_t*>(a.col_idx) + static_cast<int64_t>(vb) * a.nb_pad;
            int tok_bytes = (a.T - (n0 + 8 * ch)) * 2;
            tok_bytes = tok_bytes < 0 ? 0 : (tok_bytes > 16 ? 16 : tok_bytes);
            const uint16_t* xt_tok = a.XT + n0 + 8 * ch;
            // A_i1 words of this warp's 4 blocks, loaded two stages ahead (the load latency is not exposed)
            auto load_ci = [&](int ks) -> uint32_t {
                const int blk_l = ks * kBlocksPerStage + 4 * pw + (lane & 3);
                return (ks < k1 && blk_l < a.nb_pad) ? __ldg(ci_vb + blk_l) : 0xFFFFFFFFu;
            };
            uint32_t ci_n1 = load_ci(k0), ci_n2 = load_ci(k0 + 1);
            for (int ks = k0; ks < k1; ++ks, ++q) {
                const int s = q % S;
                const uint32_t ph = (q / S) & 1;
                const uint32_t ci = ci_n1;
                ci_n1 = ci_n2;
                ci_n2 = load_ci(ks + 2);
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* bst = sB + s * C::kBBytes + dst_chunk;
#pragma unroll
                for (int it = 0; it < 16 / RPI; ++it) {
                    const int rl = it * RPI + sub;             // 0..15 within the warp's rows
                    const int r = 16 * pw + rl;                // gathered row of the stage (0..127)
                    const uint32_t cw = __shfl_sync(0xffffffffu, ci, rl >> 2);
                    const int blk = ks * kBlocksPerStage + (r >> 2);
                    const int krow = blk * a.M + static_cast<int>((cw >> (8 * (r & 3))) & 0xFFu);
                    const bool ok = cw != 0xFFFFFFFFu && krow < a.cols;
                    const int bytes = ok ? tok_bytes : 0;
                    const uint16_t* src = bytes ? xt_tok + static_cast<int64_t>(krow) * a.ldx : a.XT;
                    cp_async_16(bst + (r >> 3) * 1024 + sw128_offset(r & 7, (ch & 7) * 16), src,
                                static_cast<uint32_t>(bytes));
                }
                cp_async_arrive_noinc(&full[s]);
            }
        }
    } else if (warp == kProdWarp) {
        // ------------------------------------------------------------ TMA producer (A_n)
        if (lane == 0) {
            int q = 0;
            for (int u = blockIdx.x; u < a.nunits; u += gridDim.x) {
                const int tile = u / a.ks_n, k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
                const int vb = tile % a.nvb;
                for (int ks = k0; ks < k1; ++ks, ++q) {
                    const int s = q % S;
                    const uint32_t ph = (q / S) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    mbar_arrive_expect_tx(&full[s], kABytes);
                    tma_load_2d(sA + s * kABytes, &tmap_a, ks * (2 * kBlocksPerStage), vb * kV, &full[s]);
                }
            }
        }
    } else if (warp == kMmaWarp) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int q = 0, tl = 0;
            const uint32_t idesc0 = idesc_bf16(64, NT, true, 0, true);
            const uint32_t idesc1 = idesc_bf16(64, NT, true, 1, true);
            for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
                const int k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
                const int acc = tl & 1;
                const uint32_t aph = (tl >> 1) & 1;
                mbar_wait(&tmem_empty[acc], aph ^ 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + ((16u * acc) << 16);
                for (int ks = k0; ks < k1; ++ks, ++q) {
                    const int s = q % S;
                    const uint32_t ph = (q / S) & 1;
                    mbar_wait(&full[s], ph);
                    mbar_wait(&meta_ready[s], ph);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(sA + s * kABytes);
                    const uint32_t b_base = smem_u32(sB + s * C::kBBytes);
#pragma unroll
                    for (int k = 0; k < kMmaPerStage; ++k) {
                        const int mi = ks * kMmaPerStage + k;
                        if (mi < n_mma) {
                            const uint64_t ad = sdesc(a_base + 32 * k, 16, 1024, kLayoutSW128);
                            const uint64_t bd = sdesc(b_base + 4096 * k, kKRowsPerStage * 128, 1024, kLayoutSW128);
                            const uint32_t e = d_tmem + kMetaCol + 4 * s + (k & ~1);
                            mma_sp_bf16(d_tmem, ad, bd, e, (k & 1) ? idesc1 : idesc0, mi > k0 * kMmaPerStage ? 1u : 0u);
                        }
                    }
                    mma_commit(&empty[s]);
                }
                mma_commit(&tmem_full[acc]);
            }
        }
    } else if (warp >= kMetaWarp0 && warp < kMetaWarp0 + 4) {
        // ------------------------------------------------------------ metadata -> TMEM
        // The slot of stage s is reused only after the MMAs that read it completed (empty[s]); lanes of the
        // other accumulator's half are written with a don't-care pattern (no in-flight MMA reads slot s).
        const int qd = warp - kMetaWarp0;  // TMEM sub-partition (== warp % 4)
        const int ml = lane % 16, mh = ml / 8;
        int q = 0, tl = 0;
        for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
            const int tile = u / a.ks_n, k0 = (u % a.ks_n) * a.sps, k1 = min(k0 + a.sps, n_stage);
            const int vb = tile % a.nvb;
            const int acc = tl & 1;
            const int row_a = vb * kV + 16 * qd + (ml % 8);
            const uint32_t* ma = a.meta + static_cast<int64_t>(row_a) * a.ld_meta;
            const uint32_t* mb = ma + 8 * static_cast<int64_t>(a.ld_meta);
            const bool mine = (lane / 16) == acc;  // lanes 16*acc .. +15 carry this tile's metadata
            // the A_i2 words of a stage, loaded two stages ahead (the load latency is not exposed)
            struct Words {
                uint32_t a[kMmaPerStage], b[kMmaPerStage];
            };
            auto load_words = [&](int ks) -> Words {
                Words r;
#pragma unroll
                for (int k = 0; k < kMmaPerStage; ++k) {
                    const int mi = ks * kMmaPerStage + k;
                    const bool ok = mine && ks < k1 && mi < n_mma;
                    r.a[k] = ok ? __ldg(ma + mi) : 0x44444444u;
                    r.b[k] = ok ? __ldg(mb + mi) : 0x44444444u;
                }
                return r;
            };
            Words n1 = load_words(k0), n2 = load_words(k0 + 1);
            for (int ks = k0; ks < k1; ++ks, ++q) {
                const int s = q % S;
                const uint32_t ph = (q / S) & 1;
                const Words cur = n1;
                n1 = n2;
                n2 = load_words(ks + 2);
                uint32_t w[kMmaPerStage];
#pragma unroll
                for (int k = 0; k < kMmaPerStage; ++k)
                    w[k] = ((cur.a[k] >> (16 * mh)) & 0xFFFFu) | (((cur.b[k] >> (16 * mh)) & 0xFFFFu) << 16);
                mbar_wait(&empty[s], ph ^ 1);
                tmem_st_32x32b_x4(tmem + ((32 * qd) << 16) + kMetaCol + 4 * s, w[0], w[1], w[2], w[3]);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&meta_ready[s]);
            }
        }
    } else if (warp < kEpiWarp0 + 4) {
        // ------------------------------------------------------------ epilogue
        const int qd = warp - kEpiWarp0;
        int tl = 0;
        for (int u = blockIdx.x; u < a.nunits; u += gridDim.x, ++tl) {
            const int tile = u / a.ks_n, kspl = u % a.ks_n;
            const int vb = tile % a.nvb, n0 = (tile / a.nvb) * NT;
            const int acc = tl & 1;
            const uint32_t aph = (tl >> 1) & 1;
            mbar_wait(&tmem_full[acc], aph);
            tc_fence_after();
            const bool mine = (lane / 16) == acc;
            const int row = vb * kV + 16 * qd + (lane % 16);
            const bool row_ok = mine && row < a.rows;
#pragma unroll 1
            for (int c = 0; c < NT; c += 16) {
                uint32_t v[16];
                tmem_ld_32x32b_x16(tmem + ((32 * qd) << 16) + c, v);
                tmem_wait_ld();
                const int tcol = n0 + c;
                if (row_ok && tcol < a.T) {
                    if (a.ks_n > 1) {  // fp32 partial of K-slice kspl
                        float* y = a.ws + (static_cast<int64_t>(kspl) * a.rows + row) * a.T + tcol;
#pragma unroll
                        for (int k = 0; k < 16; ++k)
                            if (tcol + k < a.T) y[k] = __uint_as_float(v[k]);
                    } else if (!a.y_bf16) {
                        float* y = reinterpret_cast<float*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                        if (tcol + 16 <= a.T) {
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                reinterpret_cast<uint4*>(y)[k] =
                                    make_uint4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 16; ++k)
                                if (tcol + k < a.T) y[k] = __uint_as_float(v[k]);
                        }
                    } else {
                        uint16_t* y = reinterpret_cast<uint16_t*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                        uint32_t pk[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            __nv_bfloat162 h =
                                __floats2bfloat162_rn(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]));
                            pk[k] = *reinterpret_cast<uint32_t*>(&h);
                        }
                        if (tcol + 16 <= a.T) {
                            reinterpret_cast<uint4*>(y)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                            reinterpret_cast<uint4*>(y)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                        } else {
#pragma unroll
                            for (int k = 0; k < 16; ++k)
                                if (tcol + k < a.T) y[k] = static_cast<uint16_t>((pk[k >> 1] >> (16 * (k & 1))) & 0xFFFFu);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[acc]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) tmem_dealloc(tmem, 512);
}

// Y^T[row][t] = sum over the ks K-slices, in slice order (deterministic), then fp32 or bf16 (RNE)
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, int ks, int rows, int T, void* YT, int64_t ldy,
                                     int y_bf16) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(rows) * T) return;
    const int row = static_cast<int>(idx / T), t = static_cast<int>(idx % T);
    float acc = ws[idx];
    for (int k = 1; k < ks; ++k) acc += ws[static_cast<int64_t>(k) * rows * T + idx];
    if (y_bf16) {
        reinterpret_cast<__nv_bfloat16*>(YT)[static_cast<int64_t>(row) * ldy + t] = __float2bfloat16_rn(acc);
    } else {
        reinterpret_cast<float*>(YT)[static_cast<int64_t>(row) * ldy + t] = acc;
    }
}

// ------------------------------------------------------------------ host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return static_cast<EncodeTiledFn>(nullptr);
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

bool encode_2d(CUtensorMap* tm, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
               uint32_t box_inner, uint32_t box_outer) {
    EncodeTiledFn enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Split K when the tiles cannot fill the GPU: minimise (waves of units) x (stages per unit + 1 for the
// per-unit epilogue / pipeline refill), K-slices of at least 2 stages.
int choose_ksplit(int ntiles, int n_stage) {
    const int G = num_sms();
    if (ntiles >= 2 * G) return 1;
    int best = 1;
    long best_cost = static_cast<long>((ntiles + G - 1) / G) * (n_stage + 1);
    for (int ks = 2; ks <= 16 && 2 * ks <= n_stage; ++ks) {
        const int sps = (n_stage + ks - 1) / ks;
        const long cost = static_cast<long>((ntiles * ks + G - 1) / G) * (sps + 1);
        if (cost < best_cost) {
            best_cost = cost;
            best = ks;
        }
    }
    return best;
}

template <int NT>
int launch_nt(const SpmmLaunch& L, const CUtensorMap& ta, SpmmArgs a, cudaStream_t st) {
    auto k = vnm_spmm_kernel<NT>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NT>::kSmem) != cudaSuccess)
        return kLaunchCudaError;
    a.ntt = (L.T + NT - 1) / NT;
    a.ntiles = a.nvb * a.ntt;
    const int n_stage = (a.ld_meta + kMmaPerStage - 1) / kMmaPerStage;
    a.ks_n = 1;
    if (L.workspace) {
        const int ks = choose_ksplit(a.ntiles, n_stage);
        if (ks > 1 && L.workspace_bytes >= static_cast<size_t>(ks) * a.rows * L.T * 4) {
            a.ks_n = ks;
            a.ws = static_cast<float*>(L.workspace);
        }
    }
    a.sps = (n_stage + a.ks_n - 1) / a.ks_n;
    a.ks_n = (n_stage + a.sps - 1) / a.sps;  // no empty slices
    a.nunits = a.ntiles * a.ks_n;
    const int grid = a.nunits < num_sms() ? a.nunits : num_sms();
    k<<<grid, kThreads, Cfg<NT>::kSmem, st>>>(ta, a);
    count_launch();
    if (a.ks_n > 1) {
        const int64_t n = static_cast<int64_t>(a.rows) * L.T;
        splitk_reduce_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(a.ws, a.ks_n, a.rows, L.T, a.YT, a.ldy,
                                                                                    a.y_bf16);
        count_launch();
    }
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

size_t spmm_workspace_bytes(const vnm_geom& g, int32_t T) {
    if (g.V != kV || T <= 0 || T > 64 || g.nb_pad == 0) return 0;  // split-K serves the small-T (gather) plan
    const int n_stage = (g.ld_meta + kMmaPerStage - 1) / kMmaPerStage;
    const int ks = choose_ksplit(g.rows_p / kV, n_stage);
    return ks > 1 ? static_cast<size_t>(ks) * g.rows * T * 4 : 0;
}

int launch_spmm(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (g.V != kV) return kLaunchUnsupported;
    if (g.nb_pad == 0) {  // K == 0: Y = 0
        const size_t es = L.y_dtype == VNM_BF16 ? 2 : 4;
        return cudaMemset2DAsync(L.YT, static_cast<size_t>(L.ldy) * es, 0, static_cast<size_t>(L.T) * es, g.rows,
                                 stream) == cudaSuccess ? 0 : kLaunchCudaError;
    }
    // A_n: [rows_p][ld_val] bf16, box 64 values x 64 rows, 128B swizzle (values past ld_val zero-filled).
    CUtensorMap ta;
    if (!encode_2d(&ta, L.P->values, static_cast<uint64_t>(g.ld_val), static_cast<uint64_t>(g.rows_p),
                   static_cast<uint64_t>(g.ld_val) * 2, 64, 64))
        return kLaunchCudaError;
    SpmmArgs a;
    a.XT = L.XT;
    a.ldx = L.ldx;
    a.cols = g.cols;
    a.col_idx = L.P->col_idx;
    a.meta = L.P->meta;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.T = L.T;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.M = g.M;
    a.nb_pad = g.nb_pad;
    a.ld_meta = g.ld_meta;
    a.nvb = g.rows_p / kV;
    a.ntt = 0;
    a.ntiles = 0;
    if (L.T > 128) return launch_nt<256>(L, ta, a, stream);
    if (L.T > 64) return launch_nt<128>(L, ta, a, stream);
    return launch_nt<64>(L, ta, a, stream);
}

}  // namespace vnm
