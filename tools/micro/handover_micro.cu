// Step-boundary cost on B200 (diagnostic micro): a chain of 148 x 1024-thread CTAs with
// ~174 KB of shared memory (one CTA per SM, like the fused step kernel), each "step" a
// light touch of global memory.  Compares
//   (a) one kernel per step, 32 launches captured in a CUDA graph, plain stream order
//   (b) the same with programmatic dependent launch (griddepcontrol.wait / launch_dependents)
//   (c) one persistent launch, 32 steps separated by an in-kernel grid barrier
//       (a monotonic global counter: red.release.gpu + ld.acquire.gpu spin)
//   (d) as (c) with 2-CTA clusters and the cooperative attribute
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/micro/handover_micro.bin tools/micro/handover_micro.cu
#include <cstdio>
#include <cstdint>

constexpr int STEPS = 32;
constexpr size_t SMEM = 174 * 1024;

__device__ __forceinline__ void touch(uint32_t *g, uint32_t step) {
    extern __shared__ uint32_t sm[];
    sm[threadIdx.x] = step;
    __syncthreads();
    g[blockIdx.x * 1024 + threadIdx.x] += sm[(threadIdx.x + 1) & 1023];
}

__global__ void __launch_bounds__(1024) k_step(uint32_t *g, uint32_t step, int pdl) {
    if (pdl) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    }
    touch(g, step);
}

__device__ __forceinline__ void grid_barrier(unsigned int *ctr, unsigned int target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
        unsigned int v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory"); } while (v < target);
    }
    __syncthreads();
}

__global__ void __launch_bounds__(1024) k_persistent(uint32_t *g, unsigned int *ctr, unsigned int base) {
    for (uint32_t s = 0; s < STEPS; ++s) {
        touch(g, s);
        grid_barrier(ctr, base + (s + 1) * gridDim.x);
    }
}

int main() {
    uint32_t *g;
    unsigned int *ctr;
    cudaMalloc(&g, 148 * 1024 * 4);
    cudaMalloc(&ctr, 4);
    cudaMemset(g, 0, 148 * 1024 * 4);
    cudaMemset(ctr, 0, 4);
    cudaFuncSetAttribute(k_step, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    cudaFuncSetAttribute(k_persistent, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int pdl = 0; pdl < 2; ++pdl) {
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int k = 0; k < STEPS; ++k) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = 148; cfg.blockDim = 1024; cfg.dynamicSmemBytes = SMEM; cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
            cudaLaunchKernelEx(&cfg, k_step, g, (uint32_t)k, pdl);
        }
        cudaStreamEndCapture(s, &gr);
        cudaGraphInstantiate(&ge, gr, 0);
        for (int w = 0; w < 20; ++w) cudaGraphLaunch(ge, s);
        cudaEventRecord(e0, s);
        for (int r = 0; r < 100; ++r) cudaGraphLaunch(ge, s);
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("(%c) kernel per step, graph%s: %.2f us per step\n", pdl ? 'b' : 'a', pdl ? " + PDL" : "", ms * 1e3 / (100 * STEPS));
    }
    for (int cl = 1; cl <= 2; ++cl) {
        unsigned int base = 0;
        cudaMemset(ctr, 0, 4);
        auto launch = [&]() {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = 148; cfg.blockDim = 1024; cfg.dynamicSmemBytes = SMEM; cfg.stream = s;
            cudaLaunchAttribute at[2];
            int na = 0;
            at[na].id = cudaLaunchAttributeCooperative; at[na].val.cooperative = 1; ++na;
            if (cl > 1) { at[na].id = cudaLaunchAttributeClusterDimension; at[na].val.clusterDim.x = cl; at[na].val.clusterDim.y = 1; at[na].val.clusterDim.z = 1; ++na; }
            cfg.attrs = at; cfg.numAttrs = na;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k_persistent, g, ctr, base);
            if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
            base += STEPS * 148;
        };
        for (int w = 0; w < 20; ++w) launch();
        cudaEventRecord(e0, s);
        for (int r = 0; r < 100; ++r) launch();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("(%c) persistent, grid barrier, cluster %d: %.2f us per step\n", cl == 1 ? 'c' : 'd', cl, ms * 1e3 / (100 * STEPS));
    }
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
