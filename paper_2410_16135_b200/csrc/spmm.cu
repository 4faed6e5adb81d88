// spmm.cu — the V:N:M SpMM  Y^T = W' X^T  on the 5th-generation sparse tensor cores (SURVEY §8(a)
// rows a6-a8; §3 "Acceleration of V:N:M sparsity" P:106-109 and App. A: "retrieve the
// retained weights and the corresponding tiles of the input matrix B ... align the data layout with
// that of a 2:4-sparse MM").
//
// One CTA computes one output tile = one V-block (V = 64 rows of W) x NT tokens.  K is walked in
// stages of 32 column blocks (= 4 sparse MMAs of logical K = 32, 8 blocks each):
//   warp 4     TMA: the stage's A_n tile (64 rows x 64 bf16 = 128 B rows, 128B swizzle, K-major);
//   warps 0-3  gather: the 4 kept X^T rows of each block (A_i1) -> the stage's B tile, MN-major,
//              128B swizzle, 16-byte cp.async with zero fill (tokens >= T, channels >= K: padding);
//              and the 2:4 metadata (A_i2) words -> TMEM in the M=64 sparse-metadata layout;
//   warp 5     one thread issues tcgen05.mma.sp.cta_group::1.kind::f16 (M=64, N=NT) into a TMEM fp32
//              accumulator and commits each stage back to the producers;
//   warps 0-3  epilogue: tcgen05.ld -> fp32 / bf16 -> Y^T rows.
//
// TMEM layouts used here were measured on B200 by csrc/probes.cu:
//   D (M=64):  row m -> lane (m % 16) + 32 * (m / 16), column n.
//   E (M=64):  the nibble of (row m, K-group g) is nibble 4*((m/8)%2) + g%4 of the 32-bit word at
//              lane (m % 8) + 8*(g/4) + 32*(m/16), column e_addr + id2 (e_addr even).
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "ptx.cuh"
#include "vnm_internal.h"

namespace vnm {
namespace {

constexpr int kV = 64;                       // rows per MMA (V-block)
constexpr int kBlocksPerStage = 32;          // column blocks per pipeline stage
constexpr int kMmaPerStage = kBlocksPerStage / 8;
constexpr int kKRowsPerStage = 4 * kBlocksPerStage;  // gathered X^T rows per stage (128)
constexpr int kThreads = 192;                // warps 0-3 gather/meta/epilogue, 4 TMA, 5 MMA
constexpr uint32_t kMetaCol = 256;
constexpr uint32_t kABytes = kV * 128;       // 64 rows x 64 bf16

struct SpmmArgs {
    const uint16_t* XT;
    int64_t ldx;
    int32_t T;
    const uint8_t* col_idx;
    const uint32_t* meta;
    void* YT;
    int64_t ldy;
    int32_t y_bf16;
    int32_t rows, cols, M, nb_pad, ld_meta;
};

template <int NT>
struct Cfg {
    static constexpr int kBBytes = kKRowsPerStage * NT * 2;
    static constexpr int kStageBytes = kABytes + kBBytes;
    static constexpr int kStages = NT == 256 ? 3 : (NT == 128 ? 4 : 6);
    static constexpr int kSmem = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) vnm_spmm_kernel(const __grid_constant__ CUtensorMap tmap_a,
                                                               const SpmmArgs a) {
    using C = Cfg<NT>;
    constexpr int S = C::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;                            // S x 8 KB
    uint8_t* sB = smem + S * kABytes;              // S x kBBytes
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * C::kStageBytes);
    uint64_t* empty = full + S;
    uint64_t* tmem_full = empty + S;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int vb = blockIdx.x;
    const int n0 = blockIdx.y * NT;
    const int n_mma = a.ld_meta;                   // nb_pad / 8
    const int n_stage = (n_mma + kMmaPerStage - 1) / kMmaPerStage;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 128 + 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 5) tmem_alloc(tmem_slot, 512);
    if (warp == 4 && lane == 0) tma_prefetch_desc(&tmap_a);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 4) {
        // ------------------------------------------------------------ gather + metadata producers
        const int t = threadIdx.x;  // 0..127
        constexpr int kChunks = NT / 8;                  // 16-byte chunks per gathered row
        constexpr int kRowsPerPass = 128 / kChunks;      // rows covered by one pass of 128 threads
        const int ch = t % kChunks;
        const int r_first = t / kChunks;
        const int nc = ch / 8, cw = ch % 8;              // 64-token chunk, 16-B chunk within it
        const int tok = n0 + ch * 8;
        int tok_bytes = (a.T - tok) * 2;
        tok_bytes = tok_bytes < 0 ? 0 : (tok_bytes > 16 ? 16 : tok_bytes);
        const uint8_t* ci_vb = a.col_idx + static_cast<int64_t>(vb) * a.nb_pad * 4;
        // metadata lane role (lanes 0..15 of each 32-lane sub-partition are used for M = 64)
        const int ml = lane % 16, mh = ml / 8;
        const int row_a = vb * kV + 16 * warp + (ml % 8), row_b = row_a + 8;
        const uint32_t* meta_a = a.meta + static_cast<int64_t>(row_a) * a.ld_meta;
        const uint32_t* meta_b = a.meta + static_cast<int64_t>(row_b) * a.ld_meta;
        constexpr int LAG = 1;
        for (int it = 0; it < n_stage; ++it) {
            const int s = it % S;
            const uint32_t ph = (it / S) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* bst = sB + s * C::kBBytes;
            const int blk0 = it * kBlocksPerStage;
#pragma unroll 4
            for (int r = r_first; r < kKRowsPerStage; r += kRowsPerPass) {
                const int blk = blk0 + r / 4;
                const int krow = (blk < a.nb_pad) ? blk * a.M + ci_vb[blk * 4 + (r % 4)] : a.cols;
                const int bytes = krow < a.cols ? tok_bytes : 0;
                const uint16_t* src = bytes ? a.XT + static_cast<int64_t>(krow) * a.ldx + tok : a.XT;
                uint8_t* dst = bst + nc * (kKRowsPerStage * 128) + (r / 8) * 1024 + sw128_offset(r % 8, cw * 16);
                cp_async_16(dst, src, static_cast<uint32_t>(bytes));
            }
            cp_async_commit();
            // metadata of the stage's (up to) 4 MMAs -> TMEM columns kMetaCol + 4 s + k
            {
                uint32_t w[kMmaPerStage];
#pragma unroll
                for (int k = 0; k < kMmaPerStage; ++k) {
                    const int mi = it * kMmaPerStage + k;
                    uint32_t wa = 0x44444444u, wb = 0x44444444u;
                    if (mi < n_mma) {
                        wa = __ldg(meta_a + mi);
                        wb = __ldg(meta_b + mi);
                    }
                    w[k] = ((wa >> (16 * mh)) & 0xFFFFu) | (((wb >> (16 * mh)) & 0xFFFFu) << 16);
                    if (lane >= 16) w[k] = 0x44444444u;
                }
                tmem_st_32x32b_x4(tmem + ((32 * warp) << 16) + kMetaCol + 4 * s, w[0], w[1], w[2], w[3]);
                tmem_wait_st();
            }
            if (it >= LAG) {
                cp_async_wait<LAG>();
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(&full[(it - LAG) % S]);
            }
        }
        cp_async_wait<0>();
        fence_proxy_async_smem();
        tc_fence_before();
        for (int it = n_stage - LAG < 0 ? 0 : n_stage - LAG; it < n_stage; ++it) mbar_arrive(&full[it % S]);

        // ------------------------------------------------------------ epilogue
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = vb * kV + 16 * warp + lane;  // valid for lane < 16
        const bool row_ok = lane < 16 && row < a.rows;
#pragma unroll 1
        for (int c = 0; c < NT; c += 16) {
            uint32_t v[16];
            tmem_ld_32x32b_x16(tmem + ((32 * warp) << 16) + c, v);
            tmem_wait_ld();
            const int tcol = n0 + c;
            if (row_ok && tcol < a.T) {
                if (!a.y_bf16) {
                    float* y = reinterpret_cast<float*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                    if (tcol + 16 <= a.T) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            reinterpret_cast<uint4*>(y)[q] = make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    } else {
                        for (int q = 0; q < 16 && tcol + q < a.T; ++q) y[q] = __uint_as_float(v[q]);
                    }
                } else {
                    uint16_t* y = reinterpret_cast<uint16_t*>(a.YT) + static_cast<int64_t>(row) * a.ldy + tcol;
                    uint32_t pk[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(v[2 * q]), __uint_as_float(v[2 * q + 1]));
                        pk[q] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    if (tcol + 16 <= a.T) {
                        reinterpret_cast<uint4*>(y)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        reinterpret_cast<uint4*>(y)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    } else {
                        for (int q = 0; q < 16 && tcol + q < a.T; ++q)
                            y[q] = static_cast<uint16_t>((pk[q / 2] >> (16 * (q % 2))) & 0xFFFFu);
                    }
                }
            }
        }
    } else if (warp == 4) {
        // ------------------------------------------------------------ TMA producer for A_n
        if (lane == 0) {
            for (int it = 0; it < n_stage; ++it) {
                const int s = it % S;
                const uint32_t ph = (it / S) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                mbar_arrive_expect_tx(&full[s], kABytes);
                tma_load_2d(sA + s * kABytes, &tmap_a, it * (2 * kBlocksPerStage), vb * kV, &full[s]);
            }
        }
    } else {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc0 = idesc_bf16(64, NT, true, 0, true);
            const uint32_t idesc1 = idesc_bf16(64, NT, true, 1, true);
            for (int it = 0; it < n_stage; ++it) {
                const int s = it % S;
                const uint32_t ph = (it / S) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA + s * kABytes);
                const uint32_t b_base = smem_u32(sB + s * C::kBBytes);
#pragma unroll
                for (int k = 0; k < kMmaPerStage; ++k) {
                    const int mi = it * kMmaPerStage + k;
                    if (mi < n_mma) {
                        const uint64_t ad = sdesc(a_base + 32 * k, 16, 1024, kLayoutSW128);
                        const uint64_t bd = sdesc(b_base + 4096 * k, kKRowsPerStage * 128, 1024, kLayoutSW128);
                        const uint32_t e = tmem + kMetaCol + 4 * s + (k & ~1);
                        mma_sp_bf16(tmem, ad, bd, e, (k & 1) ? idesc1 : idesc0, mi > 0 ? 1u : 0u);
                    }
                }
                mma_commit(&empty[s]);
            }
            mma_commit(tmem_full);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 5) tmem_dealloc(tmem, 512);
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

template <int NT>
int launch_nt(const SpmmLaunch& L, const CUtensorMap& tm, const SpmmArgs& a, cudaStream_t st) {
    auto k = vnm_spmm_kernel<NT>;
    if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NT>::kSmem) != cudaSuccess)
        return kLaunchCudaError;
    dim3 grid(L.P->g.rows_p / kV, (L.T + NT - 1) / NT);
    k<<<grid, kThreads, Cfg<NT>::kSmem, st>>>(tm, a);
    count_launch();
    return cudaGetLastError() == cudaSuccess ? 0 : kLaunchCudaError;
}

}  // namespace

size_t spmm_workspace_bytes(const vnm_geom&, int32_t) { return 0; }

int launch_spmm(const SpmmLaunch& L, cudaStream_t stream) {
    const vnm_geom& g = L.P->g;
    if (g.V != kV) return kLaunchUnsupported;
    if (g.nb_pad == 0) {  // K == 0: Y = 0
        const size_t es = L.y_dtype == VNM_BF16 ? 2 : 4;
        return cudaMemset2DAsync(L.YT, static_cast<size_t>(L.ldy) * es, 0, static_cast<size_t>(L.T) * es, g.rows,
                                 stream) == cudaSuccess ? 0 : kLaunchCudaError;
    }
    EncodeTiledFn enc = get_encode();
    if (!enc) return kLaunchCudaError;
    // A_n tensor map: [rows_p][ld_val] bf16, box 64 values x 64 rows, 128B swizzle
    CUtensorMap tm;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(g.ld_val), static_cast<cuuint64_t>(g.rows_p)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(g.ld_val) * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, L.P->values, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return kLaunchCudaError;
    SpmmArgs a;
    a.XT = L.XT;
    a.ldx = L.ldx;
    a.T = L.T;
    a.col_idx = L.P->col_idx;
    a.meta = L.P->meta;
    a.YT = L.YT;
    a.ldy = L.ldy;
    a.y_bf16 = L.y_dtype == VNM_BF16;
    a.rows = g.rows;
    a.cols = g.cols;
    a.M = g.M;
    a.nb_pad = g.nb_pad;
    a.ld_meta = g.ld_meta;
    if (L.T > 128) return launch_nt<256>(L, tm, a, stream);
    if (L.T > 64) return launch_nt<128>(L, tm, a, stream);
    return launch_nt<64>(L, tm, a, stream);
}

}  // namespace vnm
