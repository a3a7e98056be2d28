// Launch wrappers of the temporally blocked stencil k_step2d_tb.
// One translation unit per precision (TSW_TB_DTYPE = double / float) and variant (TSW_TB_EN = 0:
// plain, 1: with the fused energy of S5), compiled in parallel with the runtime: the kernel's
// instantiations (K = 2..8 × 4- / 8-warp CTAs × peer stores on / off) dominate the build.  The
// runtime calls tb_setup / tb_launch (declared in tsw_kernels.cuh) with the arguments it prepared.
#define TSW_TB_UNIT 1
#include "tsw_kernels.cuh"

#ifndef TSW_TB_DTYPE
#error "compile with -DTSW_TB_DTYPE=double or float"
#endif
#ifndef TSW_TB_EN
#error "compile with -DTSW_TB_EN=0 or 1"
#endif

namespace tsw {

template <typename T, int K, int NC, bool EN>
cudaError_t tb_setup(size_t smem, int* occ) {
    for (auto fn : {k_step2d_tb<T, K, false, NC, EN>, k_step2d_tb<T, K, true, NC, EN>}) {
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, k_step2d_tb<T, K, false, NC, EN>, NC * 32, smem);
}

template <typename T, int K, int NC, bool EN>
cudaError_t tb_launch(bool push, unsigned blocks, size_t smem, cudaStream_t stream, const TbArgs<T>& a, int depth) {
    if (push)
        k_step2d_tb<T, K, true, NC, EN><<<blocks, NC * 32, smem, stream>>>(a, depth);
    else
        k_step2d_tb<T, K, false, NC, EN><<<blocks, NC * 32, smem, stream>>>(a, depth);
    return cudaGetLastError();
}

#define TSW_TB_INST(K, NC)                                                                                   \
    template cudaError_t tb_setup<TSW_TB_DTYPE, K, NC, bool(TSW_TB_EN)>(size_t, int*);                       \
    template cudaError_t tb_launch<TSW_TB_DTYPE, K, NC, bool(TSW_TB_EN)>(bool, unsigned, size_t, cudaStream_t, \
                                                                         const TbArgs<TSW_TB_DTYPE>&, int);
#define TSW_TB_INST_K(K) TSW_TB_INST(K, (tb_wide_nc<TSW_TB_DTYPE, K>())) TSW_TB_INST(K, 4)
TSW_TB_INST_K(2)
TSW_TB_INST_K(3)
TSW_TB_INST_K(4)
TSW_TB_INST_K(5)
TSW_TB_INST_K(6)
TSW_TB_INST_K(7)
TSW_TB_INST_K(8)
TSW_TB_INST_K(9)
TSW_TB_INST_K(10)

}  // namespace tsw
