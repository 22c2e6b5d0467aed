// spa_band_fixed.cu -- band_kernel instantiations with the code length
// compiled in (NFIX) for the BASELINE.json configs' codes, in a translation
// unit of their own so the build compiles them in parallel with spa_band.cu.
// Sizes, shared-memory region bases, band offsets and the row stride become
// immediates: fewer integer instructions per edge-update, identical
// arithmetic.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "band_common.cuh"
#include "ldpc_internal.h"

namespace ldpc {
namespace {
using namespace band;
#include "channel_common.cuh"
#include "band_kernel.cuh"

template <int WR, int WC, int B0, int MODE, int N>
void *et_pair(bool et) {
    return et ? reinterpret_cast<void *>(&band_kernel<WR, WC, B0, true, MODE, N>)
              : reinterpret_cast<void *>(&band_kernel<WR, WC, B0, false, MODE, N>);
}
// few iterations: the no-vote instantiation (fixed-iteration mode; under early
// termination the votes are off anyway)
template <int WR, int WC, int B0, int MODE, int N>
void *et_pair_nv(bool et, bool novote) {
    if (novote && !et) return reinterpret_cast<void *>(&band_kernel<WR, WC, B0, false, MODE, N, false, 0, true>);
    return et_pair<WR, WC, B0, MODE, N>(et);
}
}  // namespace

// (n, wr, wc, rows per thread, mode) as band_plan resolves them in auto mode:
//   C4 16200 (3,6) VM+16-bit; C2 1008 (3,6) check-major; C3 3996 (3,6/12)
//   check-major; Table I 1032 (wc 9/6 VM+16-bit, 3 check-major).  Measured
//   on B200 against NFIX = 0: C2 +2.6, C4 +2.9, C3-R3/4 +0.7, Table I R1/4
//   (100k frames) +1.3 points of the SFU roofline; C3 (3,4) -0.7 (left out).
// Lane-pair kernels (LPR = 2): Table I R1/4 and R1/2 (wc x wr >= 64).  The
// (3,12) codes measured worse with them (C3-R3/4 60 -> 47%, T1-R3/4 at 100k
// frames 53 -> 51%), C1 -3%.
template <int WR, int WC, int MODE, int N>
void *lpr2(bool et, bool novote) {
    if (et) return reinterpret_cast<void *>(&band_kernel<WR, WC, 1, true, MODE, N, false, 0, false, 2>);
    if (novote) return reinterpret_cast<void *>(&band_kernel<WR, WC, 1, false, MODE, N, false, 0, true, 2>);
    return reinterpret_cast<void *>(&band_kernel<WR, WC, 1, false, MODE, N, false, 0, false, 2>);
}

// Rows per thread of a compile-time-n kernel when it differs from band_plan's
// default (0: the default).  C3-R1/4 (999 rows per band): two rows per thread,
// 512 threads, three CTAs per SM (its launch bounds) -- one 1024-thread CTA
// held 64 registers per thread and left two thirds of shared memory idle.
int band_fixed_b0(int n, int wr, int wc, int64_t frames, int sms) {
    if (n == 3996 && wr == 4 && wc == 3) return 2;
    // C3-R1/2: two rows per thread (352 threads, 56 registers) at three CTAs
    // per SM instead of one row per thread (672 threads, 40 registers) at two:
    // 4.47 -> 5.20 Gbit/s, issue 0.61 -> 0.71 (LDPC_C3R12_B0=1: the old plan)
    const char *e = std::getenv("LDPC_C3R12_B0");
    if (n == 3996 && wr == 6 && wc == 3 && frames > sms && !(e && std::atoi(e) == 1)) return 2;
    // C2: two rows per thread (96 threads, 56 registers) at 12 CTAs per SM
    // instead of one (192 threads, 40 registers) at 7: sweep 5.13 -> 5.42
    // Gbit/s, 1.0 dB +8% (14 CTAs at 40 registers spill: 5.09).
    // LDPC_C2_B0=1: the old plan
    const char *e2 = std::getenv("LDPC_C2_B0");
    // (batches only: a lone frame -- stream mode -- keeps one row per thread,
    // twice the warps on its SM: 100 -> 80 us per C2 frame)
    if (n == 1008 && wr == 6 && wc == 3 && frames > sms && !(e2 && std::atoi(e2) == 1)) return 2;
    return 0;
}
// Compile-time-n codes whose auto plan is variable-major E with 16-bit
// offsets (MODE 2) although R fits shared memory: C3 (n = 3996).  Check-major
// E left the variable phase gathering E at random banks (40% of its shared
// wavefronts were conflicts once occupancy made the kernel MIO-bound).
bool band_fixed_vm(int n, int wr, int wc) {
    return n == 3996 && wc == 3 && (wr == 4 || wr == 6 || wr == 12) && !std::getenv("LDPC_NO_VM_FIXED");
}

void *pick_band_kernel_fixed(int n, int wr, int wc, int b0, bool et, int mode, int max_iter, int lpr) {
    const bool novote = band_novote(n, wr, wc, max_iter, et);
    if (lpr == 2) {
        if (b0 != 1) return nullptr;
        if (wr == 12 && n == 1032) {
            if (wc == 9 && mode == 2) return lpr2<12, 9, 2, 1032>(et, novote);
            if (wc == 6 && mode == 2) return lpr2<12, 6, 2, 1032>(et, novote);
        }
        return nullptr;
    }
    if (lpr != 1) return nullptr;
    if (wc == 3 && wr == 6 && n == 16200 && b0 == 3 && mode == 2) {
        // R of RPRE of the 3 band-0 rows prefetched before the check->variable
        // barrier.  Round 1 (scalar psi): 0 rows 65.8%, 1 67.2%, 2 68.2%, 3
        // 66.8% (spills) of the SFU roofline.  Round 2 (packed psi, more
        // register pairs): 0 rows 84.6% (63 registers, no spill), 1 83.9%
        // (8-byte spill), 2 82.9% (28-byte spill) -- 0 is the default;
        // LDPC_RPRE=1/2 for A/B
        const char *e = std::getenv("LDPC_RPRE");
        const int rp = e ? std::atoi(e) : 0;
        if (rp == 1) return et ? reinterpret_cast<void *>(&band_kernel<6, 3, 3, true, 2, 16200, false, 1>)
                               : reinterpret_cast<void *>(&band_kernel<6, 3, 3, false, 2, 16200, false, 1>);
        if (rp == 2) return et ? reinterpret_cast<void *>(&band_kernel<6, 3, 3, true, 2, 16200, false, 2>)
                               : reinterpret_cast<void *>(&band_kernel<6, 3, 3, false, 2, 16200, false, 2>);
        return et_pair<6, 3, 3, 2, 16200>(et);
    }
    if (wc == 3 && wr == 6 && n == 1008 && b0 == 1 && mode == 0) return et_pair<6, 3, 1, 0, 1008>(et);
    if (wc == 3 && wr == 6 && n == 1008 && b0 == 2 && mode == 0) return et_pair<6, 3, 2, 0, 1008>(et);
    if (wc == 3 && wr == 6 && n == 96 && b0 == 1 && mode == 0) {     // C1: band-0 rows on lane pairs
        if (std::getenv("LDPC_NO_B0PAIR")) return et_pair_nv<6, 3, 1, 0, 96>(et, novote);
        if (et) return reinterpret_cast<void *>(&band_kernel<6, 3, 1, true, 0, 96, false, 0, false, 1, 2>);
        if (novote) return reinterpret_cast<void *>(&band_kernel<6, 3, 1, false, 0, 96, false, 0, true, 1, 2>);
        return reinterpret_cast<void *>(&band_kernel<6, 3, 1, false, 0, 96, false, 0, false, 1, 2>);
    }
    if (wc == 3 && wr == 4 && n == 3996 && b0 == 2 && mode == 0) return et_pair<4, 3, 2, 0, 3996>(et);   // C3-R1/4
    if (wc == 3 && n == 3996 && mode == 2) {      // C3, variable-major E + 16-bit offsets
        if (wr == 4 && b0 == 2) return et_pair<4, 3, 2, 2, 3996>(et);
        if (wr == 6 && b0 == 1) return et_pair<6, 3, 1, 2, 3996>(et);
        if (wr == 6 && b0 == 2) return et_pair<6, 3, 2, 2, 3996>(et);
        if (wr == 12 && b0 == 1) return et_pair<12, 3, 1, 2, 3996>(et);
    }
    if (wc == 3 && n == 3996 && b0 == 1 && mode == 0) {
        if (wr == 6) return et_pair<6, 3, 1, 0, 3996>(et);
        if (wr == 12) return et_pair<12, 3, 1, 0, 3996>(et);
    }
    if (wr == 12 && n == 1032 && b0 == 1) {
        if (wc == 9 && mode == 2) return et_pair_nv<12, 9, 1, 2, 1032>(et, novote);
        if (wc == 6 && mode == 2) return et_pair_nv<12, 6, 1, 2, 1032>(et, novote);
        if (wc == 3 && mode == 0) return et_pair_nv<12, 3, 1, 0, 1032>(et, novote);
    }
    return nullptr;
}

}  // namespace ldpc
