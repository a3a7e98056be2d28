// fp64 pipe characterisation on this GPU (tools only, not product): throughput of dependent
// (x + b)·a − b chains as a function of warps per SM and independent chains per thread (ILP),
// plus the dependent-issue latency (1 warp, ILP 1), and (argument "ops") the rate of add-only,
// multiply-only and 2u − p (DFMA) chains at 16 warps × ILP 8.  Prints one JSON line per configuration.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void probe(double* out, int iters, double a, double b) {
    double x[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dadd_rn(x[i], b);
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dmul_rn(x[i], a);
#pragma unroll
        for (int i = 0; i < ILP; ++i) x[i] = __dsub_rn(x[i], b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += x[i];
    if (s == -1.2345) out[threadIdx.x] = s;
}

template <int ILP>
void run(int sms, int warps_per_sm, double* out) {
    const int threads = 32 * (warps_per_sm < 32 ? warps_per_sm : 32);
    const int blocks_per_sm = (warps_per_sm * 32 + threads - 1) / threads;
    const int blocks = sms * blocks_per_sm;
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<ILP><<<blocks, threads>>>(out, iters / 10, 1.0, 0.5);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        probe<ILP><<<blocks, threads>>>(out, iters, 1.0, 0.5);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double instr = double(blocks) * threads * iters * 3.0 * ILP;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_sm_clk = instr / (best * 1e-3) / sms / (clk * 1e3);
    printf("{\"warps_per_sm\": %d, \"ilp\": %d, \"tops\": %.3f, \"lanes_per_clk_per_sm\": %.2f, \"cycles_per_dep_op_1warp\": %.2f}\n",
           warps_per_sm, ILP, instr / (best * 1e-3) / 1e12, per_sm_clk,
           (warps_per_sm == 1 && sms == 1) ? (best * 1e-3) * clk * 1e3 / (iters * 3.0) : 0.0);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

// OP 1: x + b three times; OP 2: x·a three times; OP 3: fma(2, x, −b) three times
template <int OP>
__global__ void probe_op(double* out, int iters, double a, double b) {
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                x[i] = OP == 1 ? __dadd_rn(x[i], b) : OP == 2 ? __dmul_rn(x[i], a) : __fma_rn(2.0, x[i], -b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i];
    if (s == -1.2345) out[threadIdx.x] = s;
}

template <int OP>
void run_op(int sms, double* out, const char* name) {
    const int threads = 512, blocks = sms, iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe_op<OP><<<blocks, threads>>>(out, iters / 10, 1.0, 0.0);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        probe_op<OP><<<blocks, threads>>>(out, iters, 1.0, 0.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double instr = double(blocks) * threads * iters * 3.0 * 8;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("{\"op\": \"%s\", \"warps_per_sm\": 16, \"ilp\": 8, \"tops\": %.3f, \"lanes_per_clk_per_sm\": %.2f}\n", name,
           instr / (best * 1e-3) / 1e12, instr / (best * 1e-3) / sms / (clk * 1e3));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 1024 * sizeof(double));
    if (argc > 1) {   // "ops": per-instruction-type rates
        run_op<1>(sms, out, "dadd");
        run_op<2>(sms, out, "dmul");
        run_op<3>(sms, out, "dfma_2u_minus_p");
        cudaFree(out);
        return 0;
    }
    run<1>(1, 1, out);   // latency: one warp, one chain
    for (int w : {4, 8, 16, 24, 32, 64}) {
        run<1>(sms, w, out);
        run<2>(sms, w, out);
        run<4>(sms, w, out);
        run<8>(sms, w, out);
    }
    cudaFree(out);
    return 0;
}
