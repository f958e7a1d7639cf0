// PCIe write-rate probe (B200 box): device -> page-locked host, by the copy engine
// and by SM stores into the mapped host buffer, for the access shapes the direct
// readback can use. nvcc -O3 -gencode arch=compute_100a,code=sm_100a pcie_write_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

// contiguous copy, grid-stride, 16 B per lane
__global__ void copy_contig(const uint4* __restrict__ src, uint4* dst, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) dst[i] = __ldcg(src + i);
}
// super-tile shape: one warp per 64x64 RGB8 tile (64 rows of 192 B, row pitch W*3)
__global__ void copy_super(const uint8_t* src, uint8_t* dst, int W, int H, int nsx, int nsy) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int s = warp; s < nsx * nsy; s += nw) {
        const int sy = s / nsx, sx = s % nsx;
        const size_t o0 = 3 * ((size_t)sy * 64 * W + (size_t)sx * 64);
        for (int i = lane; i < 12 * 64; i += 32) {
            const int r = i / 12, c = i % 12;
            const size_t o = o0 + (size_t)r * W * 3 + 16 * c;
            *reinterpret_cast<uint4*>(dst + o) = __ldcg(reinterpret_cast<const uint4*>(src + o));
        }
    }
}
// row shape: one warp per super-tile row (64 image rows, contiguous)
__global__ void copy_rows(const uint4* src, uint4* dst, size_t per, int nrows) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < nrows; r += nw)
        for (size_t i = lane; i < per; i += 32) dst[r * per + i] = __ldcg(src + r * per + i);
}

int main() {
    const int W = 3840, H = 2176; // 34 super-tile rows
    const size_t bytes = (size_t)W * H * 3;
    uint8_t *d, *h;
    CK(cudaMalloc(&d, bytes));
    CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
    uint8_t* hd;
    CK(cudaHostGetDevicePointer((void**)&hd, h, 0));
    CK(cudaMemset(d, 1, bytes));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto rate = [&](const char* name, auto fn) {
        for (int k = 0; k < 3; ++k) fn();
        cudaEventRecord(a);
        const int reps = 10;
        for (int k = 0; k < reps; ++k) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-44s %7.3f ms  %6.1f GB/s\n", name, ms / reps, bytes / (ms / reps * 1e6));
    };
    rate("copy engine cudaMemcpyAsync", [&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost); });
    for (int blocks : {148, 592, 2368})
        for (int thr : {128, 512}) {
            char nm[96];
            snprintf(nm, sizeof nm, "SM contiguous 16B/lane, %d x %d", blocks, thr);
            rate(nm, [&] { copy_contig<<<blocks, thr>>>((const uint4*)d, (uint4*)hd, bytes / 16); });
        }
    for (int warps : {8, 32, 128, 592, 2368}) {
        char nm[96];
        snprintf(nm, sizeof nm, "SM super-tiles (192 B rows), %d warps", warps);
        rate(nm, [&] { copy_super<<<(warps + 3) / 4, 128>>>(d, hd, W, H, W / 64, H / 64); });
    }
    for (int warps : {4, 8, 16, 34}) {
        char nm[96];
        snprintf(nm, sizeof nm, "SM super-tile rows (737 KB), %d warps", warps);
        rate(nm, [&] { copy_rows<<<(warps + 3) / 4, 128>>>((const uint4*)d, (uint4*)hd, (size_t)W * 64 * 3 / 16, H / 64); });
    }
    CK(cudaGetLastError());
    return 0;
}
