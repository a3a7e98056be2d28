// Probe: does a pending cuStreamWaitValue32 on one stream block kernels of another stream of the
// same context?  (nvcc -gencode arch=compute_100a,code=sm_100a -o wv waitvalue_probe.cu; ./wv 0)
// On the B200 pool (driver 580.159) it does — see DESIGN.md §8.
#include <cuda_runtime.h>
#include <cstdio>
typedef int (*Pfn)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
__global__ void sig(unsigned int* p, unsigned int v) { __threadfence_system(); asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
int main(int argc, char** argv) {
    int variant = argc > 1 ? atoi(argv[1]) : 0;
    void* fp = nullptr; cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuStreamWaitValue32", &fp, cudaEnableDefault, &q);
    printf("entry %d q=%d fp=%p\n", (int)e, (int)q, fp);
    int flush = 0; cudaDeviceGetAttribute(&flush, cudaDevAttrCanFlushRemoteWrites, 0);
    printf("can flush remote writes: %d\n", flush);
    Pfn wait = (Pfn)fp;
    unsigned int* m; cudaMalloc(&m, 256); cudaMemset(m, 0, 256); cudaDeviceSynchronize();
    cudaStream_t s1, s2; cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    unsigned int flags = (variant & 1) ? (1u << 30) : 0u;
    int r = wait(s1, (unsigned long long)m, 0, flags);
    printf("wait(>=0) ret %d\n", r); fflush(stdout);
    e = cudaStreamSynchronize(s1);
    printf("sync after satisfied wait: %s\n", cudaGetErrorString(e)); fflush(stdout);
    r = wait(s1, (unsigned long long)m, 1, flags);
    printf("wait(>=1) ret %d, query %d\n", r, (int)cudaStreamQuery(s1)); fflush(stdout);
    sig<<<1, 1, 0, s2>>>(m, 1);
    e = cudaStreamSynchronize(s2);
    printf("signal done %s\n", cudaGetErrorString(e)); fflush(stdout);
    e = cudaStreamSynchronize(s1);
    printf("sync after signalled wait: %s\n", cudaGetErrorString(e)); fflush(stdout);
    return 0;
}
