// Dense fast path: fused single-pass FP64 tensor-core (DMMA) kernels. (placeholder until landed)
#include "state.h"

namespace nadmm {

bool dmma_supported(const Shard&) { return false; }

void dmma_pass(Shard&, PassMode, const double*, const int32_t*) {
    raise(NADMM_ECONFIG, "dmma path not available for this shard");
}

}  // namespace nadmm
