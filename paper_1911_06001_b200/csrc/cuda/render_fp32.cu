// Production FP32 instantiation of the frame and traversal kernels
// (compiled with FMA contraction enabled: -fmad=true).
#include "frame_kernel.cuh"
#include "traverse_kernel.cuh"

namespace vxa {

namespace {
template <bool A, int H, bool K> void* frame_fn() { return reinterpret_cast<void*>(&frame_kernel<float, A, H, K>); }
template <bool A, bool K> void* pick_h(int hbo) {
    return hbo == 2 ? frame_fn<A, 2, K>() : hbo == 1 ? frame_fn<A, 1, K>() : frame_fn<A, 0, K>();
}
// hbo: 0 none, 1 48-byte records, 2 16-byte records
void* pick(bool aov, int hbo, bool compact, bool direct = false) {
    if (direct) // direct synchronous readback (vxa_render: no AOV, no hit buffer)
        return compact ? reinterpret_cast<void*>(&frame_kernel<float, false, 0, true, true>)
                       : reinterpret_cast<void*>(&frame_kernel<float, false, 0, false, true>);
    if (aov) return compact ? pick_h<true, true>(hbo) : pick_h<true, false>(hbo);
    return compact ? pick_h<false, true>(hbo) : pick_h<false, false>(hbo);
}
int hbo_mode(const FrameParams<float>& p, bool hbo) { return hbo ? (p.hbo_compact ? 2 : 1) : 0; }
} // namespace

cudaError_t launch_frame_f32(const FrameParams<float>& p, bool aov, bool hbo, const FrameLaunch& l) {
    void* args[] = {const_cast<FrameParams<float>*>(&p)};
#if VXA_PDL
    if (p.super_list != nullptr) { // behind the pre-pass: programmatic dependent launch
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(l.grid);
        cfg.blockDim = dim3(kBlock);
        cfg.dynamicSmemBytes = frame_smem_bytes_f32(p.max_depth);
        cfg.stream = l.stream;
        cudaLaunchAttribute attr{};
        attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr.val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = &attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelExC(&cfg, pick(aov, hbo_mode(p, hbo), p.compact != 0, p.super_done != nullptr), args);
    }
#endif
    return cudaLaunchKernel(pick(aov, hbo_mode(p, hbo), p.compact != 0, p.super_done != nullptr), dim3(l.grid), dim3(kBlock), args,
                            frame_smem_bytes_f32(p.max_depth), l.stream);
}

cudaError_t launch_super_cull(const FrameParams<float>& p, uint16_t* list, uint32_t* count, uint32_t* done,
                              cudaStream_t s) {
    const uint32_t n_mine = p.n_tiles / kTilesPerSuper;
    if (n_mine == 0) return cudaSuccess;
    super_cull_kernel<float><<<n_mine, 128, 0, s>>>(p, list, count, done);
    return cudaGetLastError();
}

size_t frame_smem_bytes_f32(uint32_t max_depth) {
    return kStackBytes * kBlock * stack_levels(max_depth) + 4u * VXA_SMEM_TOP;
}

int frame_blocks_per_sm_f32(bool aov, int hbo, bool compact, uint32_t max_depth) {
    int b = 0;
    void* fn = pick(aov, hbo, compact);
    const size_t smem = frame_smem_bytes_f32(max_depth);
    if (smem > 48 * 1024) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, kBlock, smem) != cudaSuccess) return 1;
    return b > 0 ? b : 1;
}

cudaError_t launch_traverse_f32(const DevModel& m, const TraverseRayIn* rays, uint32_t n, TraverseRayOut* out,
                                VisitOut* log, uint32_t log_cap, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    traverse_kernel<float><<<(n + 127) / 128, 128, 0, s>>>(m, rays, n, out, log, log_cap);
    return cudaGetLastError();
}

} // namespace vxa
