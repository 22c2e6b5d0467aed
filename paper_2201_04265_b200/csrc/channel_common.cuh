// channel_common.cuh -- the counter-based generators of the workload recipe
// (DESIGN.md "Inputs"), shared by the harness kernels (codec_kernels.cu) and
// the fused simulate decoder (spa_band_sim.cu) so both draw bit-identical
// frames.  Included inside an anonymous namespace.
#pragma once

// ---------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11): the counter-based generator the
// workload recipe fixes.
struct U4 {
    uint32_t x, y, z, w;
};
__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// BPSK + AWGN noise of Philox block j of frame fr: counter
// (j, fr_lo, fr_hi, 1); Box-Muller in fp64 on (x, y) and (z, w).
__device__ __forceinline__ void channel_normals(uint64_t seed, uint64_t fr, int j, double (&z)[4]) {
    const double two_pi = 6.283185307179586476925286766559;
    const double inv32 = 1.0 / 4294967296.0;
    const U4 r = philox(U4{uint32_t(j), uint32_t(fr), uint32_t(fr >> 32), 1u}, uint32_t(seed), uint32_t(seed >> 32));
    {
        const double rad = sqrt(-2.0 * log((double(r.x) + 1.0) * inv32));
        double sn, cs;
        sincos(two_pi * (double(r.y) * inv32), &sn, &cs);
        z[0] = rad * cs;
        z[1] = rad * sn;
    }
    {
        const double rad = sqrt(-2.0 * log((double(r.z) + 1.0) * inv32));
        double sn, cs;
        sincos(two_pi * (double(r.w) * inv32), &sn, &cs);
        z[2] = rad * cs;
        z[3] = rad * sn;
    }
}
// Channel LLR, Eq. 4 (reading Q1): y = x + sigma z, R = fp32(clamp(2y/sigma^2,
// +-30)), with no FMA contraction so the fp64 roundings are the plain formula's.
__device__ __forceinline__ float channel_llr(bool one, double sigma, double z) {
    const double x = one ? 1.0 : -1.0;
    const double y = __dadd_rn(x, __dmul_rn(sigma, z));
    double l = __ddiv_rn(__dmul_rn(2.0, y), __dmul_rn(sigma, sigma));
    l = fmin(fmax(l, -30.0), 30.0);
    return float(l);
}
