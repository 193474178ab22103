// microbenchmark: cost of cooperative_groups cluster.sync() vs a grid-wide
// atomic barrier, for cluster sizes 2..16 (nvcc -arch=sm_100a)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cs(int iters, unsigned long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) cl.sync();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

__global__ void k_cs_raw(int iters, unsigned long long *out) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

__global__ void k_cs_relaxed(int iters, unsigned long long *out) {
    unsigned long long t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) {
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
    }
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = t1 - t0;
}

template <typename K>
void run(const char *name, K kern, int cs, int nt) {
    unsigned long long *d, h = 0;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(nt);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    const int iters = 10000;
    cudaLaunchKernelEx(&cfg, kern, iters, d);
    cudaLaunchKernelEx(&cfg, kern, iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-10s cluster %2d x %3d threads: %s  %.3f us per barrier\n", name, cs, nt, cudaGetErrorString(e), h * 1e-3 / iters);
    cudaFree(d);
}

int main() {
    for (int cs : {2, 4, 8, 16})
        for (int nt : {32, 256}) {
            run("cg", k_cs, cs, nt);
            run("raw", k_cs_raw, cs, nt);
            run("relaxed", k_cs_relaxed, cs, nt);
        }
    return 0;
}
