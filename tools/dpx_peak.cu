// DPX add-min throughput on this GPU (for bench.py's roofline_alu): every
// thread runs independent chains of __viaddmin_u16x2 (VIADDMNMX.U16x2, two
// 16-bit relaxations per instruction) or __viaddmin_u32; reports
// instructions per clock per SM and relaxations per second.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dpx_peak tools/dpx_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <bool U16>
__global__ void dpx_kernel(unsigned *out, int iters, unsigned w) {
    constexpr int C = 8;   // independent chains per thread
    unsigned d[C], x[C];
    for (int c = 0; c < C; ++c) {
        d[c] = 0x7fff7fffu ^ (threadIdx.x * 7 + c);
        x[c] = threadIdx.x * 13 + c * 3;
    }
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (U16) d[c] = __viaddmin_u16x2(x[c], w, d[c]);
            else d[c] = __viaddmin_u32(x[c], w, d[c]);
            x[c] ^= d[c];
        }
    }
    unsigned r = 0;
    for (int c = 0; c < C; ++c) r ^= d[c];
    if (r == 0x12345678u) out[0] = r;   // keep the chains alive
}

int main() {
    int dev = 0, nsm = 0, clk = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);   // kHz
    unsigned *out;
    cudaMalloc(&out, 4);
    const int iters = 1 << 14, threads = 1024, blocks = nsm * 2;
    for (int pass = 0; pass < 2; ++pass) {
        for (int u16 = 0; u16 < 2; ++u16) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            if (u16) dpx_kernel<true><<<blocks, threads>>>(out, 16, 5u);
            else dpx_kernel<false><<<blocks, threads>>>(out, 16, 5u);
            cudaEventRecord(a);
            if (u16) dpx_kernel<true><<<blocks, threads>>>(out, iters, 5u | (5u << 16));
            else dpx_kernel<false><<<blocks, threads>>>(out, iters, 5u);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            const double instr = (double)blocks * threads * iters * 8;   // thread-level DPX ops
            const double per_clk_sm = instr / 32.0 / (ms * 1e-3) / (clk * 1e3) / nsm;   // warp instr / clk / SM
            if (pass)
                printf("{\"op\": \"%s\", \"ms\": %.3f, \"warp_instr_per_clk_per_sm\": %.3f, \"lane_ops_per_clk_per_sm\": %.1f, "
                       "\"relaxations_per_s\": %.4g, \"clock_khz\": %d, \"sms\": %d}\n",
                       u16 ? "VIADDMNMX.U16x2" : "VIADDMNMX.U32", ms, per_clk_sm, per_clk_sm * 32,
                       instr * (u16 ? 2 : 1) / (ms * 1e-3), clk, nsm);
        }
    }
    return 0;
}
