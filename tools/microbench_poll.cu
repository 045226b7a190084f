#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long *p)
{ unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory"); return v; }
__device__ __forceinline__ void st_relaxed(unsigned long long *p, unsigned long long v)
{ asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory"); }
__device__ __forceinline__ unsigned long long ld_rlx_nomem(const unsigned long long *p)
{ unsigned long long v; asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p)); return v; }

// serial poll (baseline)
__device__ __forceinline__ void wait_serial(const unsigned long long *p, unsigned long long k)
{ while (ld_relaxed(p) != k) {} }
// pipelined poll: W loads in flight, round robin
template <int W>
__device__ __forceinline__ void wait_pipe(const unsigned long long *p, unsigned long long k, int gap)
{
    unsigned long long v[W];
#pragma unroll
    for (int j = 0; j < W; ++j) { v[j] = ld_rlx_nomem(p); if (gap) { long long c = clock64(); while (clock64() - c < gap) {} } }
    while (true) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
            if (v[j] == k) return;
            v[j] = ld_rlx_nomem(p);
        }
    }
}

template <int MODE>
__global__ void pingpong(unsigned long long *slots, int iters, int peer, long long *out, int gap)
{
    if (threadIdx.x != 0) return;
    const int me = blockIdx.x == 0 ? 0 : (blockIdx.x == (unsigned)peer ? 1 : -1);
    if (me < 0) return;
    unsigned long long *mine = slots + me * 32, *theirs = slots + (1 - me) * 32;
    long long t0 = clock64();
    for (int k = 1; k <= iters; ++k) {
        if (me == 0) {
            st_relaxed(mine, k);
            if (MODE == 0) wait_serial(theirs, k); else if (MODE == 1) wait_pipe<4>(theirs, k, gap); else wait_pipe<8>(theirs, k, gap);
        } else {
            if (MODE == 0) wait_serial(theirs, k); else if (MODE == 1) wait_pipe<4>(theirs, k, gap); else wait_pipe<8>(theirs, k, gap);
            st_relaxed(mine, k);
        }
    }
    long long t1 = clock64();
    if (me == 0) out[0] = t1 - t0;
}

// DSMEM ping-pong inside a cluster of 2
__global__ void __cluster_dims__(2, 1, 1) dsmem_pp(int iters, long long *out)
{
    __shared__ volatile unsigned long long box;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned r = cl.block_rank();
    if (threadIdx.x == 0) box = 0;
    cl.sync();
    if (threadIdx.x == 0) {
        unsigned long long *peer = cl.map_shared_rank((unsigned long long *)&box, r ^ 1);
        long long t0 = clock64();
        for (int k = 1; k <= iters; ++k) {
            if (r == 0) {
                asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(peer)), "l"((unsigned long long)k) : "memory");
                while (box != (unsigned long long)k) {}
            } else {
                while (box != (unsigned long long)k) {}
                asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(peer)), "l"((unsigned long long)k) : "memory");
            }
        }
        long long t1 = clock64();
        if (r == 0) out[2] = t1 - t0;
    }
    cl.sync();
}

int main()
{
    unsigned long long *slots; long long *out, h[4];
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&slots, 4096); cudaMalloc(&out, 64);
    const int iters = 20000;
    for (int peer : {1, sms / 2, sms - 1}) {
        for (int mode = 0; mode < 3; ++mode) for (int gap : {0, 40, 80}) {
            if (mode == 0 && gap) continue;
            cudaMemset(slots, 0, 4096);
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            if (mode == 0) pingpong<0><<<sms, 32>>>(slots, iters, peer, out, gap);
            if (mode == 1) pingpong<1><<<sms, 32>>>(slots, iters, peer, out, gap);
            if (mode == 2) pingpong<2><<<sms, 32>>>(slots, iters, peer, out, gap);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(h, out, 8, cudaMemcpyDeviceToHost);
            printf("global pingpong %s gap %2d peer %3d: round trip %.1f ns, %.0f clk\n", mode == 0 ? "serial" : mode == 1 ? "pipe4 " : "pipe8 ", gap, peer, ms * 1e6 / iters, (double)h[0] / iters);
        }
    }
    {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        dsmem_pp<<<2, 32>>>(iters, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        printf("dsmem pingpong cluster2: round trip %.1f ns, %.0f clk (%s)\n", ms * 1e6 / iters, (double)h[2] / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
