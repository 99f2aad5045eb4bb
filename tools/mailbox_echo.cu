// Mailbox latency probe (measurement only): a one-warp server echoes requests
// through pinned host memory, with and without a system-scope fence, against
// an empty launch + stream sync.  nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o scratch/mailbox_echo tools/mailbox_echo.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <atomic>
#include <chrono>
#include <vector>
#include <algorithm>
struct MB { uint32_t req_seq; int32_t req[6]; uint32_t req_seq2; uint32_t pad0[8]; uint32_t done_seq; uint32_t pad1[15]; int32_t out[260]; };
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void server(MB* mb, int mode, uint64_t* dev_t) {
    const int lane = threadIdx.x;
    uint32_t last = 0;
    const uint4* req4 = reinterpret_cast<const uint4*>(mb);
    for (;;) {
        uint32_t w0 = 0, w7 = 0;
        if (lane == 0) {
            uint4 a, b;
            asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w) : "l"(req4) : "memory");
            asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(b.x), "=r"(b.y), "=r"(b.z), "=r"(b.w) : "l"(req4 + 1) : "memory");
            w0 = a.x; w7 = b.w;
        }
        w0 = __shfl_sync(~0u, w0, 0); w7 = __shfl_sync(~0u, w7, 0);
        if (w0 == last || w7 != w0) continue;
        if (w0 == 0xFFFFFFFFu) return;
        if (lane < 5) {
            asm volatile("st.volatile.global.v4.u32 [%0], {%1, %1, %1, %1};" :: "l"(reinterpret_cast<uint4*>(mb->out) + lane), "r"(w0) : "memory");
        }
        if (mode == 1) __threadfence_system();
        __syncwarp();
        if (lane == 0) *reinterpret_cast<volatile uint32_t*>(&mb->done_seq) = w0;
        last = w0;
    }
}
int main() {
    MB* mb; cudaHostAlloc(&mb, sizeof(MB), cudaHostAllocMapped); memset(mb, 0, sizeof(MB));
    for (int mode = 0; mode < 2; ++mode) {
        memset(mb, 0, sizeof(MB));
        cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        server<<<1, 32, 0, st>>>(mb, mode, nullptr);
        volatile MB* v = mb;
        std::vector<double> ts;
        for (uint32_t seq = 1; seq <= 20000; ++seq) {
            auto t0 = std::chrono::steady_clock::now();
            v->req[0] = seq;
            std::atomic_thread_fence(std::memory_order_seq_cst);
            v->req_seq = seq;
            std::atomic_thread_fence(std::memory_order_seq_cst);
            v->req_seq2 = seq;
            std::atomic_thread_fence(std::memory_order_seq_cst);
            while (v->done_seq != seq) {}
            auto t1 = std::chrono::steady_clock::now();
            if (seq > 1000) ts.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
        }
        v->req_seq = 0xFFFFFFFFu; std::atomic_thread_fence(std::memory_order_seq_cst); v->req_seq2 = 0xFFFFFFFFu;
        cudaStreamSynchronize(st);
        std::sort(ts.begin(), ts.end());
        printf("mode %d (fence.sys %s): median %.2f us p10 %.2f p90 %.2f\n", mode, mode ? "yes" : "no", ts[ts.size()/2], ts[ts.size()/10], ts[ts.size()*9/10]);
    }
    // launch + sync latency for reference
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    std::vector<double> ts;
    for (int i = 0; i < 5000; ++i) {
        auto t0 = std::chrono::steady_clock::now();
        server<<<1, 32, 0, st>>>(mb, 0, nullptr);  // exits immediately: req_seq = STOP
        cudaStreamSynchronize(st);
        auto t1 = std::chrono::steady_clock::now();
        if (i > 500) ts.push_back(std::chrono::duration<double, std::micro>(t1 - t0).count());
    }
    std::sort(ts.begin(), ts.end());
    printf("empty launch + stream sync: median %.2f us\n", ts[ts.size()/2]);
    return 0;
}
