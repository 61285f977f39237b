// compute-sanitizer synccheck control: a minimal, correct mbarrier handoff
// in the decode GEMV's pattern (thread 0 inits, fence + __syncthreads, warp 0
// arrives, warp 1 waits on parity 0). If synccheck reports "Missing init"
// here too, its report on sgemv_kernel's red_full barriers is a tool
// limitation, not a kernel defect.
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(int* out) {
    __shared__ __align__(8) uint64_t bar[4];
    __shared__ float buf[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar[i])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 0) {
        buf[lane] = (float)lane;
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
    } else if (warp == 1) {
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                su32(&bar[0])),
            "r"(0)
            : "memory");
        out[blockIdx.x * 32 + lane] = (int)buf[lane];
    }
}

// the decode GEMV's reduction handoff: 8 consumer warps wait red_empty (fresh
// barrier, parity 1), write a buffer, arrive on red_full (count 8); one
// epilogue warp per barrier waits red_full and re-arms red_empty (count 1);
// griddepcontrol as in the kernel; 2 rounds per barrier
template <bool PDL, bool FRESH_ODD_WAIT>
__global__ void __launch_bounds__(416, 1) probe2(float* out, int ne) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t full_bar[16];
    __shared__ __align__(8) uint64_t empty_bar[16];
    __shared__ __align__(8) uint64_t red_full[4];
    __shared__ __align__(8) uint64_t red_empty[4];
    float* red = reinterpret_cast<float*>(sm);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < 16; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full_bar[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty_bar[s])), "r"(8));
        }
        for (int e = 0; e < ne; ++e) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&red_full[e])), "r"(8));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&red_empty[e])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (PDL) {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    auto wait = [](uint64_t* b, uint32_t par) {
        asm volatile(
            "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                su32(b)),
            "r"(par)
            : "memory");
    };
    auto arrive = [](uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); };
    if (warp >= 9) {
        const int e = warp - 9;
        if (e >= ne) return;
        uint32_t ph = 0;
        for (int i = e; i < 2 * ne; i += ne) {
            wait(&red_full[e], ph);
            ph ^= 1u;
            float acc = 0.f;
            for (int w = 0; w < 8; ++w) acc += red[(e * 8 + w) * 32 + lane];
            __syncwarp();
            if (lane == 0) arrive(&red_empty[e]);
            out[(blockIdx.x * 2 * ne + i) * 32 + lane] = acc;
        }
        return;
    }
    if (warp == 8) {  // producer: nothing to stream here
        __syncwarp();
    }
    if (warp == 8) return;
    uint32_t rph[4] = {0, 0, 0, 0};
    for (int i = 0; i < 2 * ne; ++i) {
        const int e = i % ne;
        // first use of each buffer: either the parity-1 wait on the fresh
        // barrier (passes at once: the CUTLASS producer-start idiom) or no wait
        if (FRESH_ODD_WAIT || i >= ne) wait(&red_empty[e], rph[e] ^ 1u);
        rph[e] ^= 1u;
        red[(e * 8 + warp) * 32 + lane] = (float)(i + warp);
        __syncwarp();
        if (lane == 0) arrive(&red_full[e]);
    }
}

int main() {
    int* d;
    cudaMalloc(&d, 4 * 32 * 4);
    probe<<<4, 64>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    int h[32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mbar probe: %s, out[31] = %d\n", cudaGetErrorString(e), h[31]);
    float* o2;
    cudaMalloc(&o2, 8 * 8 * 32 * 4);
    auto run = [&](auto kern, const char* name, int dyn) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
        kern<<<8, 416, dyn>>>(o2, 4);
        cudaError_t er = cudaDeviceSynchronize();
        float h2[32];
        cudaMemcpy(h2, o2, sizeof h2, cudaMemcpyDeviceToHost);
        printf("probe2 %s dyn %d: %s, out[0] = %.0f (expect 28)\n", name, dyn, cudaGetErrorString(er), h2[0]);
    };
    run(probe2<true, true>, "PDL fresh-parity-1-wait", 200 * 1024);
    run(probe2<true, false>, "PDL no-first-wait", 200 * 1024);
    return 0;
}
