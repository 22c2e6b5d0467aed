// microbench_cluster.cu -- how many thread-block clusters of size C fit the
// B200 at one CTA per SM (the C5 exchange kernels use ~163-195 KB of shared
// memory per CTA), and which SMs a full launch places them on (the SMs of one
// cluster share a GPC).  Prints, for C = 1..16, cudaOccupancyMaxActiveClusters
// and the SMs covered; then the SM ids of every cluster of a C = 2 launch
// (pairs) grouped by GPC as inferred from a C = 16 launch.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/microbench_cluster tools/microbench_cluster.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <set>
#include <vector>

__global__ void where_kernel(int *smid_out, int *cl_out) {
    extern __shared__ char smem[];
    if (threadIdx.x == 0) {
        unsigned s, c;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
        asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(c));
        smid_out[blockIdx.x] = int(s);
        cl_out[blockIdx.x] = int(c);
        smem[0] = 1;
    }
    // hold the SM long enough that every cluster is resident at once
    long long t0 = clock64();
    while (clock64() - t0 < 20000000) {
    }
}

int main() {
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(where_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    cudaFuncSetAttribute(where_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("SMs %d, one CTA per SM (%zu KB smem)\n", sms, smem / 1024);
    int *d_sm, *d_cl;
    cudaMalloc(&d_sm, 4096 * 4);
    cudaMalloc(&d_cl, 4096 * 4);
    for (int C = 1; C <= 16; ++C) {
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(C);
        int ncl = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, where_kernel, &cfg);
        if (e != cudaSuccess) {
            printf("C=%2d occupancy error %s\n", C, cudaGetErrorString(e));
            cudaGetLastError();
            continue;
        }
        cfg.gridDim = dim3(ncl * C);
        e = cudaLaunchKernelEx(&cfg, where_kernel, d_sm, d_cl);
        cudaDeviceSynchronize();
        std::vector<int> hs(ncl * C), hc(ncl * C);
        cudaMemcpy(hs.data(), d_sm, 4 * hs.size(), cudaMemcpyDeviceToHost);
        cudaMemcpy(hc.data(), d_cl, 4 * hc.size(), cudaMemcpyDeviceToHost);
        std::set<int> used(hs.begin(), hs.end());
        printf("C=%2d max active clusters %3d -> %3d SMs (%zu distinct)%s\n", C, ncl, ncl * C, used.size(),
               e == cudaSuccess ? "" : " launch failed");
        if (C == 16 || C == 8 || C == 9 || C == 10 || C == 12) {
            for (int k = 0; k < ncl; ++k) {
                printf("   cluster %2d:", k);
                for (int i = 0; i < C; ++i) printf(" %3d", hs[k * C + i]);
                printf("\n");
            }
        }
    }
    return 0;
}
