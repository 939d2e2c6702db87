// gemm_tc.cu -- batched dense Toeplitz product on tcgen05 int8 tensor cores.
// (placeholder: the tcgen05 kernel lands in the next milestone)
#include "qrng_internal.cuh"

namespace qrng {
namespace gemm {

bool supported(uint64_t, uint64_t) { return false; }

qrng_status plan_init(Plan &, uint64_t, uint64_t, const uint8_t *, cudaStream_t) {
    set_error("GEMM path not built yet");
    return QRNG_E_UNSUPPORTED;
}

void plan_free(Plan &pl) {
    if (pl.seed_words) cudaFree(pl.seed_words);
    pl = Plan{};
}

qrng_status extract(const Plan &, const uint8_t *, uint64_t, uint64_t, uint64_t, const OutStream &,
                    cudaStream_t) {
    set_error("GEMM path not built yet");
    return QRNG_E_UNSUPPORTED;
}

}  // namespace gemm
}  // namespace qrng
