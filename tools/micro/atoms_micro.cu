// Shared-memory reduction throughput vs bank-conflict structure (diagnostic micro).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/atoms_micro tools/micro/atoms_micro.cu
// Every lane issues ITER x 8 red.shared.add.u32 into a TW-word tile; the address pattern:
//   mode 0: uniformly random word            (the delivery's case: random targets)
//   mode 1: random word in the lane's bank   (conflict-free: bank = lane)
//   mode 2: random word, bank = lane / 2     (2-way)
//   mode 3: random word, bank = lane & 15    (2-way, half banks)
// plus the same with 16 active lanes (mode 4: random).
#include <cstdio>
#include <cstdint>

constexpr int ITER = 2048;

__global__ void __launch_bounds__(1024) k_atoms(int mode, uint32_t TW, unsigned long long *clk) {
    extern __shared__ uint32_t cnt[];
    for (uint32_t x = threadIdx.x; x < TW; x += blockDim.x) cnt[x] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    uint32_t s = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 0x85EBCA6Bu;
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(cnt);
    const uint32_t rows = TW / 32;
    long long c0 = clock64();
    if (mode == 4 && lane >= 16) { /* idle lanes */ }
    else
    for (int it = 0; it < ITER; ++it) {
        uint32_t a[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s = s * 1664525u + 1013904223u;
            uint32_t w;
            if (mode == 0 || mode == 4) w = __umulhi(s, TW);
            else if (mode == 1) w = __umulhi(s, rows) * 32u + lane;
            else if (mode == 2) w = __umulhi(s, rows) * 32u + (lane >> 1);
            else w = __umulhi(s, rows) * 32u + (lane & 15u);
            a[k] = base + 4u * w;
        }
        asm volatile(
            "red.shared.add.u32 [%0], 1;\n\tred.shared.add.u32 [%1], 1;\n\t"
            "red.shared.add.u32 [%2], 1;\n\tred.shared.add.u32 [%3], 1;\n\t"
            "red.shared.add.u32 [%4], 1;\n\tred.shared.add.u32 [%5], 1;\n\t"
            "red.shared.add.u32 [%6], 1;\n\tred.shared.add.u32 [%7], 1;"
            :: "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]) : "memory");
    }
    __syncthreads();
    long long c1 = clock64();
    if (threadIdx.x == 0) atomicAdd(clk, (unsigned long long)(c1 - c0));
    if (cnt[threadIdx.x] == 0xFFFFFFFF) clk[1] = 1;
}

// the same address generation without the reductions (ALU cost)
__global__ void __launch_bounds__(1024) k_alu(uint32_t TW, unsigned long long *clk) {
    uint32_t s = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x * 0x85EBCA6Bu, acc = 0;
    long long c0 = clock64();
    for (int it = 0; it < ITER; ++it)
#pragma unroll
        for (int k = 0; k < 8; ++k) { s = s * 1664525u + 1013904223u; acc += __umulhi(s, TW); }
    __syncthreads();
    long long c1 = clock64();
    if (threadIdx.x == 0) atomicAdd(clk, (unsigned long long)(c1 - c0));
    if (acc == 0x12345) clk[1] = acc;
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 16);
    const uint32_t TW = 18752;
    cudaFuncSetAttribute(k_atoms, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const char *names[] = {"random", "conflict-free", "bank=lane/2", "bank=lane&15", "random, 16 lanes"};
    for (int bs : {1024, 512}) {
        for (int mode = 0; mode < 5; ++mode) {
            cudaMemset(d, 0, 16);
            k_atoms<<<148, bs, TW * 4>>>(mode, TW, d);
            cudaMemset(d, 0, 16);
            k_atoms<<<148, bs, TW * 4>>>(mode, TW, d);
            unsigned long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double cyc = (double)h / 148.0;
            const double ev = (double)bs * (mode == 4 ? 0.5 : 1.0) * ITER * 8;
            printf("block %4d %-18s %8.0f cyc/CTA  %.2f events/clk/SM  %.2f clk per warp-instr\n", bs, names[mode], cyc,
                   ev / cyc, cyc / (ev / (mode == 4 ? 16 : 32)));
        }
        cudaMemset(d, 0, 16);
        k_alu<<<148, bs>>>(TW, d);
        unsigned long long h;
        cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
        printf("block %4d address ALU only     %8.0f cyc/CTA\n", bs, (double)h / 148.0);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
