// sched.cuh — the tile schedulers of the persistent kernels (forward.cu,
// zonal_band.cu, codec_warp.cu), device side.
//
// Dynamic: lane 0 of each warp claims the next run of tiles from a global
// 64-bit counter (atomicAdd), so the tiles in flight form one compact address
// window.  Each kernel family owns 64 counter slots; the host
// (SchedGuard, abi.cu) hands a launch a slot only once every earlier launch on
// that slot is ordered before it (same stream, or an event wait), so two
// launches never draw from one counter at the same time.  The last warp of a
// launch resets its slot.
// Static: a launch recorded into a CUDA graph gets no slot (ctr == nullptr) —
// replays of one graph may overlap — and warp w takes claims w, w + nw, ...
#pragma once
#include <stdint.h>

namespace dct16a {

constexpr int kSchedSlots = 64;

// Lane-0 state of one warp's claims.
struct Claims {
    unsigned long long* ctr;   // the launch's counter pair, or nullptr (static schedule)
    long long gw, nw, k;       // static: global warp index, warps in the grid, claims made

    __device__ __forceinline__ Claims(unsigned long long* c, long long gw_, long long nw_)
        : ctr(c), gw(gw_), nw(nw_), k(0) {}

    // index of this warp's next claim (claims only grow)
    __device__ __forceinline__ long long next() {
        if (ctr) return static_cast<long long>(atomicAdd(ctr, 1ull));
        return gw + (k++) * nw;
    }
};

// Lane 0 of every warp, after its last claim: the last warp of the launch
// resets the slot for the next launch ordered after this one.
__device__ __forceinline__ void claims_done(unsigned long long* ctr, int total_warps) {
    if (!ctr) return;
    __threadfence();
    if (atomicAdd(ctr + 1, 1ull) == static_cast<unsigned long long>(total_warps) - 1) {
        ctr[0] = 0;
        ctr[1] = 0;
        __threadfence();
    }
}

}  // namespace dct16a
