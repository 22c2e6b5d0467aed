// debug_probe.cu -- diagnostics that run the throughput decoders' OWN device
// code (band_common.cuh) on caller-supplied inputs, for the exhaustive
// accuracy sweeps in tests/test_gpu_parity.py:
//   ldpc_debug_psi       psi and each of its tiers, elementwise;
//   ldpc_debug_check_row check_row<D, VOTE> (Eq. 5) on rows.
// Nothing here is on the decode path; the functions probed are the very
// inline functions every band / exchange / edge kernel calls.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {
using namespace band;

// tier: 0 psi (both regimes, selected per element), 1 psi_small, 2 psi_large,
// 3 psi_deep_large, 4 psi_deep_small, 5 psi_row<1, LARGE_FIRST = true, VOTE>
// (the first psi of a row: the warp votes pick the tier), 6 psi_row<1, false,
// VOTE> (the second psi).
__global__ void psi_probe_kernel(const float *y, float *out, int64_t count, int tier) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x) {
        const float v = y[i];
        float r;
        switch (tier) {
            case 0: r = psi(v); break;
            case 1: r = psi_small(v); break;
            case 2: r = psi_large(v); break;
            case 3: r = psi_deep_large(v); break;
            case 4: r = psi_deep_small(v); break;
            case 5: {
                const float in[1] = {v};
                float o[1];
                psi_row<1, true, true>(in, o);
                r = o[0];
                break;
            }
            default: {
                const float in[1] = {v};
                float o[1];
                psi_row<1, false, true>(in, o);
                r = o[0];
                break;
            }
        }
        out[i] = r;
    }
}

// One thread per row of D inputs x'_j = L'_v - E'_cv (log2 units); writes
// the row's D new E'_cv exactly as check_row<D, VOTE> computes them in the
// decoders, including (VOTE) the saturation and clamp tiers; the clamp-tier
// magnitudes come from clamp_row_mags, as in band_kernel.
template <int D, bool VOTE>
__global__ void check_row_probe_kernel(const float *x, float *e, int64_t rows) {
    __shared__ float cm[D];
    if constexpr (VOTE && has_clamp_tier<D>()) {
        if (threadIdx.x < 32) {
            float m[D];
            clamp_row_mags<D>(m);
            if (threadIdx.x == 0)
                for (int j = 0; j < D; ++j) cm[j] = m[j];
        }
        __syncthreads();
    }
    for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
        float xi[D], eo[D];
#pragma unroll
        for (int j = 0; j < D; ++j) xi[j] = x[r * D + j];
        check_row<D, VOTE>(xi, eo, (VOTE && has_clamp_tier<D>()) ? cm : nullptr);
#pragma unroll
        for (int j = 0; j < D; ++j) e[r * D + j] = eo[j];
    }
}

template <int D>
void *check_probe(bool vote) {
    return vote ? reinterpret_cast<void *>(&check_row_probe_kernel<D, true>)
                : reinterpret_cast<void *>(&check_row_probe_kernel<D, false>);
}

}  // namespace
}  // namespace ldpc

extern "C" {

ldpc_status ldpc_debug_psi(const float *d_y, float *d_out, int64_t count, int32_t tier, void *stream) {
    if (count < 0 || tier < 0 || tier > 6 || (count > 0 && (!d_y || !d_out))) return LDPC_ERR_ARG;
    if (count == 0) return LDPC_OK;
    const int grid = int(std::min<int64_t>((count + 255) / 256, 148 * 32));
    ldpc::psi_probe_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(d_y, d_out, count, tier);
    return cudaGetLastError() == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

ldpc_status ldpc_debug_check_row(const float *d_x, float *d_e, int64_t rows, int32_t degree, int32_t vote,
                                 void *stream) {
    if (rows < 0 || (rows > 0 && (!d_x || !d_e))) return LDPC_ERR_ARG;
    void *k = nullptr;
    switch (degree) {
        case 2: k = ldpc::check_probe<2>(vote != 0); break;
        case 3: k = ldpc::check_probe<3>(vote != 0); break;
        case 4: k = ldpc::check_probe<4>(vote != 0); break;
        case 6: k = ldpc::check_probe<6>(vote != 0); break;
        case 12: k = ldpc::check_probe<12>(vote != 0); break;
        default: return LDPC_ERR_UNSUPPORTED;
    }
    if (rows == 0) return LDPC_OK;
    const int grid = int(std::min<int64_t>((rows + 255) / 256, 148 * 8));
    void *args[] = {&d_x, &d_e, &rows};
    cudaError_t err = cudaLaunchKernel(k, dim3(unsigned(grid)), dim3(256u), args, 0, static_cast<cudaStream_t>(stream));
    return err == cudaSuccess ? LDPC_OK : LDPC_ERR_CUDA;
}

}  // extern "C"
