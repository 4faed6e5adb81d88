// vnm_internal.h — host-side glue between the C ABI (api.cpp) and the kernels (prune.cu, spmm.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../../include/vnm.h"

namespace vnm {

constexpr size_t kMaxSmem = 227 * 1024;
// every vnm_spmm workspace starts with this ticket region (small-T plan: zero between calls); plans that keep
// other scratch there (split-K partials) place it after the region, so one workspace serves every plan
constexpr size_t kWsTicketBytes = 16 * 1024;

// Tuning / tracing switches from the environment, read ONCE per call site and process (a function-local static
// inside a unique lambda), so the hot path makes no getenv calls.  Timing ablations (VNM_ABL, which make the
// results invalid) exist only in builds compiled with -DVNM_ABLATIONS.
#define VNM_ENV_INT(name, dflt)                                                                     \
    ([] {                                                                                           \
        static const int v_ = [] { const char* e_ = getenv(name); return e_ ? atoi(e_) : (dflt); }(); \
        return v_;                                                                                  \
    }())
#ifdef VNM_ABLATIONS
#define VNM_ABLATION_FLAGS() VNM_ENV_INT("VNM_ABL", 0)
#else
#define VNM_ABLATION_FLAGS() 0
#endif
constexpr int kLaunchUnsupported = 1;
constexpr int kLaunchCudaError = 2;

void count_launch();

struct PruneLaunch {
    const vnm_geom* g;
    const uint16_t* W;
    int64_t ldw;
    const float* score;      // null => ABS
    int64_t lds;
    const uint32_t* mask_in; // non-null => compress from this mask
    uint32_t* mask_out;      // may be null
    uint16_t* values;        // may be null (mask only)
    uint8_t* col_idx;
    uint32_t* meta;
    int32_t* status;         // compress only, may be null
    uint16_t* values_tc = nullptr;  // optional fused window form (prune_compress)
    uint32_t* meta_tc = nullptr;
};
int launch_prune_pack(const PruneLaunch& L, cudaStream_t stream);
int launch_prune2(const PruneLaunch& L, cudaStream_t stream);  // V >= 32 (prune2.cu)
int launch_prune2_batch(const PruneLaunch* Ls, int n, cudaStream_t stream);  // n <= 8 weights, one (V, M)

struct SpmmLaunch {
    const vnm_packed* P;
    const uint16_t* XT;
    int64_t ldx;
    int32_t T;
    void* YT;
    int64_t ldy;
    vnm_dtype y_dtype;
    void* workspace;
    size_t workspace_bytes;
};
int launch_spmm(const SpmmLaunch& L, cudaStream_t stream);
int launch_spmm_tc(const SpmmLaunch& L, cudaStream_t stream);   // window form (values_tc / meta_tc), 1 CTA
int launch_spmm_tc2(const SpmmLaunch& L, cudaStream_t stream);  // window form on CTA pairs (M = 256)
// pairs, K-ring; mode 1 resident A (short K), 0 streamed A, -1 resident when it fits (spmm_tc3.cu)
int launch_spmm_tc3(const SpmmLaunch& L, int mode, cudaStream_t stream);
int launch_pack_tc(const vnm_packed& P, cudaStream_t stream);
int launch_pack_nat24(const vnm_packed& P, cudaStream_t stream);  // M % 4 == 0, M > 8: natural 2:4 form
size_t spmm_workspace_bytes(const vnm_geom& g, int32_t T);
// small-T plan (spmm_smallt.cu): 1 <= T <= 32, V >= 16, any M; canonical A_n / A_i1 / A_i2 only
bool spmm_smallt_applies(const vnm_geom& g, int32_t T);
size_t spmm_smallt_workspace_bytes(const vnm_geom& g, int32_t T);
int launch_spmm_smallt(const SpmmLaunch& L, cudaStream_t stream);
// n (<= 4) independent problems of one T, y dtype and V class in ONE launch (vnm_spmm_batched); the workspace of
// Ls[0] serves the launch
bool spmm_smallt_batch_applies(const vnm_geom* const* gs, int n, int32_t T);
size_t spmm_smallt_batch_workspace_bytes(const vnm_geom* const* gs, int n, int32_t T);
// flags & 1: the packed weights were written before the previous kernel on the stream began (VNM_SPMM_WEIGHTS_READY)
int launch_spmm_smallt_batch(const SpmmLaunch* Ls, int n, uint32_t flags, cudaStream_t stream);

// RIA importance (ria.cu)
size_t ria_workspace_bytes(int32_t rows, int32_t cols);
int launch_ria(const uint16_t* W, int64_t ldw, int32_t rows, int32_t cols, const float* act, float a, float* score,
               int64_t lds, void* ws, cudaStream_t st);
int launch_act_norms(const uint16_t* XT, int64_t ldx, int32_t cols, int32_t T, float* norms, cudaStream_t st);

// channel-permutation gain scores (permute.cu)
size_t permute_gain_workspace_bytes(const vnm_geom& g);
int launch_permute_gain(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc, void* ws,
                        cudaStream_t st);
int launch_permute_gain_out(const float* score, int64_t lds, const vnm_geom& g, float* cost, int64_t ldc,
                            cudaStream_t st);  // permute_out.cu

}  // namespace vnm
