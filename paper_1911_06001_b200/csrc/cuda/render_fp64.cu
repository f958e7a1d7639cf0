// FP64 parity instantiation of the frame and traversal kernels
// (compiled with -fmad=false: no FMA contraction, like the reference x86-64 build, so
// every operation rounds exactly as the CPU renderer does).
#include "frame_kernel.cuh"
#include "traverse_kernel.cuh"

namespace vxa {

namespace {
template <bool A, bool H> void* frame_fn() { return reinterpret_cast<void*>(&frame_kernel<double, A, H ? 1 : 0, false>); }
void* pick(bool aov, bool hbo, bool /*compact: FP64 keeps the general words*/, bool direct = false) {
    if (direct) return reinterpret_cast<void*>(&frame_kernel<double, false, 0, false, true>); // direct readback
    if (aov) return hbo ? frame_fn<true, true>() : frame_fn<true, false>();
    return hbo ? frame_fn<false, true>() : frame_fn<false, false>();
}
} // namespace

cudaError_t launch_super_cull(const FrameParams<double>& p, uint16_t* list, uint32_t* count, uint32_t* done,
                              cudaStream_t s) {
    const uint32_t n_mine = p.n_tiles / kTilesPerSuper;
    if (n_mine == 0) return cudaSuccess;
    super_cull_kernel<double><<<n_mine, 128, 0, s>>>(p, list, count, done);
    return cudaGetLastError();
}

cudaError_t launch_frame_f64(const FrameParams<double>& p, bool aov, bool hbo, const FrameLaunch& l) {
    void* args[] = {const_cast<FrameParams<double>*>(&p)};
    return cudaLaunchKernel(pick(aov, hbo, p.compact != 0, p.super_done != nullptr), dim3(l.grid), dim3(kBlock), args, frame_smem_bytes_f64(p.max_depth), l.stream);
}

size_t frame_smem_bytes_f64(uint32_t max_depth) {
    return 0;
}

int frame_blocks_per_sm_f64(bool aov, int hbo, bool compact, uint32_t max_depth) {
    int b = 0;
    void* fn = pick(aov, hbo, compact);
    const size_t smem = frame_smem_bytes_f64(max_depth);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kBlock, smem) != cudaSuccess) return 1;
    return b > 0 ? b : 1;
}

cudaError_t launch_traverse_f64(const DevModel& m, const TraverseRayIn* rays, uint32_t n, TraverseRayOut* out,
                                VisitOut* log, uint32_t log_cap, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    traverse_kernel<double><<<(n + 127) / 128, 128, 0, s>>>(m, rays, n, out, log, log_cap);
    return cudaGetLastError();
}

} // namespace vxa
