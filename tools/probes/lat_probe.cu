// Latency of a dependent read right after a PDL dependency release, as a
// function of how much weight prefetch the dependent kernel's CTAs issued
// before griddepcontrol.wait (the stream-K GEMV's ring fill).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat_probe lat_probe.cu -lcuda
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared.b64 [%0], %1;" ::"r"(su(b)), "r"(n)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t tx) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

// A: 148 CTAs, big smem, staggered finish; writes X (rows x 8192 floats)
__global__ void writer(float* X, int n, int stagger_ns) {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    unsigned long long t0 = gt();
    while (gt() - t0 < 20000ull + (unsigned long long)blockIdx.x * stagger_ns) {}
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) X[i] = (float)i;
}

// B: prefetch `pre` bytes of W per CTA, wait, then read X (TMA, `xb` bytes) and one plain load
__global__ void reader(const float* X, int xb, const char* W, int pre, unsigned long long* tr, int mode) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar[2];
    if (threadIdx.x == 0) {
        mb_init(&bar[0], 1);
        mb_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    unsigned long long* t = tr + blockIdx.x * 8;
    if (threadIdx.x == 0) {
        t[0] = gt();
        if (pre > 0) {
            mb_expect(&bar[0], pre);
            for (int o = 0; o < pre; o += 32768)
                bulk(sm + 65536 + o, W + (size_t)blockIdx.x * (1 << 22) + o, min(32768, pre - o), &bar[0]);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        t[1] = gt();
        if (mode == 0) {
            mb_expect(&bar[1], xb);
            bulk(sm, X + (size_t)(blockIdx.x % 4) * (xb / 4), xb, &bar[1]);
            mb_wait(&bar[1], 0);
        } else {
            volatile float v = __ldcg(X + (blockIdx.x % 4) * 1024);
            (void)v;
        }
        t[2] = gt();
        float v2 = __ldcg(X + 17 + blockIdx.x);  // second, dependent-free load
        t[3] = gt() + (v2 == -1.f ? 1 : 0);
        if (pre > 0) mb_wait(&bar[0], 0);
        t[4] = gt();
    }
}

int main() {
    const int nX = 4 * 6 * 2048;  // 4 chunks x 6 rows x 2048 floats
    float* X;
    char* W;
    unsigned long long* tr;
    cudaMalloc(&X, nX * 4);
    cudaMalloc(&W, (size_t)148 << 22);
    cudaMemset(W, 1, (size_t)148 << 22);
    cudaMalloc(&tr, 148 * 8 * 8);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(writer, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int mode = 0; mode < 2; ++mode)
        for (int pre : {0, 32768, 65536, 131072}) {
            std::vector<double> d1, d2, d3, d4;
            for (int rep = 0; rep < 20; ++rep) {
                cudaMemsetAsync(tr, 0, 148 * 64, s);
                writer<<<148, 256, smem, s>>>(X, nX, 20);
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = 148;
                cfg.blockDim = 128;
                cfg.dynamicSmemBytes = smem;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, reader, (const float*)X, 6 * 2048 * 4, (const char*)W, pre, tr, mode);
                std::vector<unsigned long long> h(148 * 8);
                cudaMemcpyAsync(h.data(), tr, 148 * 64, cudaMemcpyDeviceToHost, s);
                cudaStreamSynchronize(s);
                if (rep < 3) continue;
                for (int b = 0; b < 148; ++b) {
                    const unsigned long long* t = &h[b * 8];
                    d1.push_back((t[1] - t[0]) / 1e3);
                    d2.push_back((t[2] - t[1]) / 1e3);
                    d3.push_back((t[3] - t[2]) / 1e3);
                    d4.push_back((t[4] - t[0]) / 1e3);
                }
            }
            auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
            auto mx = [](std::vector<double> v) { return *std::max_element(v.begin(), v.end()); };
            printf("%s pre %6d B/CTA: wait %.2f us | x read after dep: median %.2f max %.2f us | 2nd load %.2f us | prefetch landed %.2f us\n",
                   mode == 0 ? "TMA 48KB x" : "1 ld.cg   ", pre, med(d1), med(d2), mx(d2), med(d3), med(d4));
        }
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
