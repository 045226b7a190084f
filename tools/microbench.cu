// microbench.cu -- inter-SM communication latency on the B200 (design input
// for the TILED engine's boundary exchange).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long *p)
{
    return *(const volatile unsigned long long *)p;
}
__device__ __forceinline__ void st_volatile(unsigned long long *p, unsigned long long v)
{
    *(volatile unsigned long long *)p = v;
}
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p)
{
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v)
{
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// two CTAs (blockIdx 0 and `peer`) bounce a counter; thread 0 of each
template <int MODE>
__global__ void pingpong(unsigned long long *slots, int iters, int peer, long long *out)
{
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x == 0 ? 0 : (blockIdx.x == (unsigned)peer ? 1 : -1);
    if (me < 0) return;
    unsigned long long *mine = slots + me * 32, *theirs = slots + (1 - me) * 32;
    long long t0 = clock64();
    for (int k = 1; k <= iters; ++k) {
        if (me == 0) {
            if (MODE == 0) st_relaxed(mine, k); else if (MODE == 1) st_volatile(mine, k); else st_release(mine, k);
            unsigned long long v;
            do { v = MODE == 0 ? ld_relaxed(theirs) : MODE == 1 ? ld_volatile(theirs) : ld_acquire(theirs); } while (v != (unsigned long long)k);
        } else {
            unsigned long long v;
            do { v = MODE == 0 ? ld_relaxed(theirs) : MODE == 1 ? ld_volatile(theirs) : ld_acquire(theirs); } while (v != (unsigned long long)k);
            if (MODE == 0) st_relaxed(mine, k); else if (MODE == 1) st_volatile(mine, k); else st_release(mine, k);
        }
    }
    long long t1 = clock64();
    if (me == 0) out[0] = t1 - t0;
}

// single-thread dependent L2 load chain (pointer chase within L2)
__global__ void l2chase(const unsigned *next, int iters, long long *out, unsigned *sink)
{
    unsigned p = 0;
    long long t0 = clock64();
    for (int k = 0; k < iters; ++k) p = __ldcg(next + p);
    long long t1 = clock64();
    out[1] = t1 - t0;
    *sink = p;
}

int main()
{
    unsigned long long *slots;
    long long *out, h[4];
    unsigned *next, *sink;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaMalloc(&slots, 4096);
    cudaMalloc(&out, 64);
    cudaMalloc(&sink, 4);
    const int n = 1 << 22;
    cudaMalloc(&next, n * 4);
    unsigned *hn = new unsigned[n];
    for (int i = 0; i < n; ++i) hn[i] = (unsigned)(((long long)i * 1000003 + 12345) % n);   // a long cycle
    cudaMemcpy(next, hn, n * 4, cudaMemcpyHostToDevice);
    const int iters = 20000;
    for (int peer : {1, sms / 2, sms - 1}) {
        for (int mode = 0; mode < 3; ++mode) {
            cudaMemset(slots, 0, 4096);
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) pingpong<0><<<sms, 32>>>(slots, iters, peer, out);
            if (mode == 1) pingpong<1><<<sms, 32>>>(slots, iters, peer, out);
            if (mode == 2) pingpong<2><<<sms, 32>>>(slots, iters, peer, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
            printf("pingpong mode %s peer %3d: round trip %.1f ns (event), %.0f SM clk (clock64)\n",
                   mode == 0 ? "relaxed " : mode == 1 ? "volatile" : "rel/acq ", peer, ms * 1e6 / iters,
                   (double)h[0] / iters);
        }
    }
    l2chase<<<1, 1>>>(next, 100000, out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("dependent __ldcg chase: %.0f SM clk per load\n", (double)h[1] / 100000);
    printf("sm clock rate attr %d kHz, %s\n", clk, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
