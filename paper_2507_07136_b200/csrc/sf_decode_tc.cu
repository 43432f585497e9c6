// sf_decode_tc.cu -- tcgen05 3xTF32 codebook GEMM (in progress; SIMT until it lands).
#include "sf_common.cuh"

namespace sf {
int launch_decode(int64_t P, int L, int D, const float* w, int64_t w_stride, const float* cb,
                  float* out, cudaStream_t st) {
    return launch_decode_simt(P, L, D, w, w_stride, cb, out, st);
}
}  // namespace sf
