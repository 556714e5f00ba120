// launch.cuh -- kernel launches with Programmatic Dependent Launch (PDL).
//
// A kernel launched through launch_k may begin (launch, prologue: barrier
// init, TMEM allocation, descriptor prefetch) while the previous kernel on the
// stream is still finishing; it executes pdl_wait() (griddepcontrol.wait)
// before it touches global memory, which returns once the previous grid has
// completed and its writes are visible. Without the attribute pdl_wait is a
// no-op. DC_NO_PDL=1 launches without it.
#pragma once
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>

#include "common.hpp"

namespace dc {

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Acquire-poll a (possibly peer-mapped) flag until (int)(*p - target) >= 0,
// at system scope. A peer that has not arrived after kSpinTimeoutNs is a
// protocol error (a rank skipped a collective call), not a reason to hang the
// GPU: the kernel traps, the launch fails and the next CUDA call reports it.
constexpr unsigned long long kSpinTimeoutNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ void spin_until_geq(const uint32_t *p, uint32_t target) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if ((int)(v - target) >= 0) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > kSpinTimeoutNs) __trap();
    }
}

// Set while a loopback-group plan (capi.cu) launches: its virtual ranks share
// one GPU's SMs, and a kernel launched early that waits on the previous one
// could hold the SMs another virtual rank's halo kernel needs (deadlock).
extern thread_local bool g_no_pdl;
inline bool pdl_enabled() {
    static const bool on = std::getenv("DC_NO_PDL") == nullptr;
    return on && !g_no_pdl;
}
struct NoPdlScope {
    bool prev;
    explicit NoPdlScope(bool on) : prev(g_no_pdl) { g_no_pdl = g_no_pdl || on; }
    ~NoPdlScope() { g_no_pdl = prev; }
};

// Dynamic shared memory floor of every kernel that allocates tensor memory
// (conv_v2, wgrad_v2, conv_gemm, wgrad): more than half of an SM's 228 KB, so
// two such CTAs never share an SM. Their TMEM allocations could otherwise
// exceed the SM's 512 columns; tcgen05.alloc then blocks until the other CTA
// exits, and when both belong to CTA pairs (cluster launches) of two kernels
// running side by side -- stride phases on their own streams, interior and
// boundary tiles, virtual ranks of a loopback group -- each pair waits for its
// partner, which waits for the other pair's TMEM: a deadlock.
constexpr size_t kTmemExclusiveSmem = 116 * 1024;
inline size_t tmem_kernel_smem(size_t need) { return need > kTmemExclusiveSmem ? need : kTmemExclusiveSmem; }

// Set while a plan sizes its workspaces at creation (capi.cu presize): the
// host-side configuration runs and allocates, no kernel is launched.
extern thread_local bool g_dry_run;

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cluster,
              const char *what, Args &&...args) {
    if (g_dry_run) return;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[2];
    int na = 0;
    if (pdl_enabled()) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cluster > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster, at[na].val.clusterDim.y = 1, at[na].val.clusterDim.z = 1;
        ++na;
    }
    cfg.gridDim = grid, cfg.blockDim = block, cfg.dynamicSmemBytes = smem, cfg.stream = st;
    cfg.attrs = at, cfg.numAttrs = na;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    DC_REQUIRE(e == cudaSuccess, DC_ERR_CUDA, "%s launch: %s", what, cudaGetErrorString(e));
    ++g_launches;
}

}  // namespace dc
