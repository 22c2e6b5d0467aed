// spa_band_sim.cu -- fused simulate step: channel draw ->
// Sum-Product decode -> error counters in one band-kernel launch, without the
// frames x n x 4-byte LLR buffer.  The prologue draws R exactly as
// ldpc_channel (Eq. 4; channel_common.cuh), so the decode and the
// counters equal ldpc_channel + ldpc_decode + ldpc_count_errors bit for bit.
// Gallager (3,6) codes whose frame fits one SM (C1-C4 lengths).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {
using namespace band;
#include "channel_common.cuh"
#include "band_kernel.cuh"

template <int B0, int MODE>
void *gen_pair(bool et) {
    return et ? reinterpret_cast<void *>(&band_kernel<6, 3, B0, true, MODE, 0, true>)
              : reinterpret_cast<void *>(&band_kernel<6, 3, B0, false, MODE, 0, true>);
}
// the same arithmetic as the ldpc_decode kernel it stands in for
void *pick_gen_kernel(int n, int wr, int wc, int b0, bool et, int mode, int max_iter) {
    if (wr != 6 || wc != 3 || (mode != 0 && mode != 2)) return nullptr;
    if (band_novote(n, wr, wc, max_iter, et)) {
        if (n == 96 && b0 == 1 && mode == 0)
            return reinterpret_cast<void *>(&band_kernel<6, 3, 1, false, 0, 96, true, 0, true>);
        return nullptr;
    }
    if (n == 16200 && b0 == 3 && mode == 2)         // C4, n compiled in as in ldpc_decode
        return et ? reinterpret_cast<void *>(&band_kernel<6, 3, 3, true, 2, 16200, true>)
                  : reinterpret_cast<void *>(&band_kernel<6, 3, 3, false, 2, 16200, true>);
    switch (b0) {
        case 1: return mode ? gen_pair<1, 2>(et) : gen_pair<1, 0>(et);
        case 2: return mode ? gen_pair<2, 2>(et) : gen_pair<2, 0>(et);
        case 3: return mode ? gen_pair<3, 2>(et) : gen_pair<3, 0>(et);
    }
    return nullptr;
}
}  // namespace
}  // namespace ldpc

extern "C" ldpc_status ldpc_decode_simulate(const ldpc_code *code, uint64_t seed, int64_t frame0, int64_t frames,
                                            double sigma, const uint32_t *d_info, const uint32_t *d_cw,
                                            const ldpc_decode_opts *opts, uint32_t *d_bits, uint8_t *d_syndrome_ok,
                                            int32_t *d_iters, int64_t *d_counters6, void *d_ws, size_t ws_bytes,
                                            void *stream) {
    if (!code || !opts || frames < 0 || frame0 < 0 || !(sigma > 0.0)) return LDPC_ERR_ARG;
    if (!code->d_buf || !code->bound_G) return LDPC_ERR_STATE;
    if (opts->max_iter < 1) return LDPC_ERR_ARG;
    if (frames == 0) return LDPC_OK;
    if (!d_info || !d_cw || !d_bits || !d_syndrome_ok || !d_iters || !d_counters6) return LDPC_ERR_ARG;
    const int v = opts->variant;
    if (v != 0 && v != 3 && v != 4 && v != 6) return LDPC_ERR_UNSUPPORTED;
    ldpc::BandPlan bp;
    if (!ldpc::band_plan(*code, frames, opts->early_term != 0, v, bp, opts->max_iter, false)) return LDPC_ERR_UNSUPPORTED;
    // the rows per thread of the band plan ldpc_decode runs (its row stride is
    // bp.threads), so the fused kernel decodes every row, with the same warps
    const int b0 = bp.b0;
    void *k = ldpc::pick_gen_kernel(code->n, code->wr, code->wc, b0, opts->early_term != 0, bp.mode, opts->max_iter);
    if (!k) return LDPC_ERR_UNSUPPORTED;
    if (!ldpc::ensure_smem_attribute(k, bp.smem)) return LDPC_ERR_CUDA;
    if (!d_ws || ws_bytes < bp.ws_bytes) return LDPC_ERR_ARG;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ldpc::BandArgs a{};
    a.code = code->dev;
    a.llr = nullptr;
    a.frames = frames;
    a.max_iter = opts->max_iter;
    a.early_term = opts->early_term ? 1 : 0;
    a.bits = d_bits;
    a.syn_ok = d_syndrome_ok;
    a.iters = d_iters;
    a.posterior = nullptr;
    a.frame_counter = static_cast<unsigned long long *>(d_ws);
    a.r_global = bp.r_in_smem ? nullptr : reinterpret_cast<float *>(static_cast<char *>(d_ws) + 256);
    a.r_in_smem = bp.r_in_smem ? 1 : 0;
    a.row_stride = bp.threads;
    a.seed = seed;
    a.frame0 = frame0;
    a.sigma = sigma;
    a.cw = d_cw;
    a.info = d_info;
    a.counters = reinterpret_cast<unsigned long long *>(d_counters6);
    if (cudaMemsetAsync(d_ws, 0, 8, s) != cudaSuccess) return LDPC_ERR_CUDA;
    void *args[] = {&a};
    const cudaError_t e = cudaLaunchKernel(k, dim3(unsigned(bp.grid)), dim3(unsigned(bp.threads)), args, bp.smem, s);
    return e == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}
