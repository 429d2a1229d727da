// Launch wrappers for the solver's vector/scalar kernels (kernels_vec.cu).
#pragma once

#include "state.h"

namespace nadmm {

// g = gbase - rho (z - x + y/rho) (or gbase), with <g,g>/<t,t> partials; *nvec = partial count.
void launch_grad_aug(Shard& s, const int32_t* guard, int* nvec);
// f_x, |g|; prologue checks or trace row of the finished Newton iteration.
void launch_value_finish(Shard& s, int nvec, int prologue, const int32_t* guard);
// One full Newton iteration (CG, certificate, fallbacks, batched Armijo, step, new cache/grad).
void launch_newton_iteration(Shard& s, int cg_max, int ls_max);
void launch_set_int(Shard& s, int32_t* dst, int v);
// One Newton iteration of a node group (dmma_group.cuh); timers: cg_max + 1 event pairs or null.
void launch_group_iteration(const std::vector<Shard*>& g, int clusters, int cg_max, HvTimer* timers);
// Picks the CG-tail variant for the shard's d (cluster kernel when it fits); outside stream capture.
void tail_setup(Shard& s);

}  // namespace nadmm
