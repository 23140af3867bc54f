// lx_gram.cuh -- explicit weighted Gram M = A diag(D) A^T and its D-VJP.
//
// Reference: weighted_gram_unphased (operator.hpp:371-415), phased_gram
// (operator.hpp:217-248), gram_vjp_weights (gradients.hpp:190-219).
//
//   1. lx_gram_buckets: one warp per row rank r in [0, n]: the columns with
//      r_of_col == r form the contiguous sorted range
//      [lower_bound(B, A_{r-1}), lower_bound(B, A_r)), so the reference's
//      scatter-adds become a deterministic segmented reduction (fixed lane
//      order + xor tree, fp64), no atomics.
//   2. U / V / C scans reuse lx_carry (fp64 anchored scans, anchors 2A; a
//      zero anchor array turns it into a plain cumulative sum for C).
//   3. lx_gram_out: lower triangle in sorted order, mirrored through perm_a
//      (bit-exact symmetry, operator.hpp:410-411).
#pragma once

#include <type_traits>

#include "lx_common.cuh"

namespace lx {
namespace gram {

template <class R>
__device__ __forceinline__ uint32_t lower_bound(const R* v, uint32_t m, R x) {
    uint32_t lo = 0, hi = m;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (v[mid] < x)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// ell[c][r], rho[c][r] (r < n) and mass[c][r] (r <= n) for NCH weight channels
// (phased: cos^2, cos*sin, sin^2 of psi times D).
template <class R, int NCH>
__global__ void lx_gram_buckets(const R* __restrict__ A, uint32_t n, const R* __restrict__ B, uint32_t k,
                                const uint32_t* __restrict__ perm_b, const R* __restrict__ D,
                                const R* __restrict__ cpsi, const R* __restrict__ spsi, R* __restrict__ ell,
                                R* __restrict__ rho, R* __restrict__ mass) {
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r > n) return;
    const uint32_t lo = r == 0 ? 0 : lower_bound(B, k, A[r - 1]);
    const uint32_t hi = r == n ? k : lower_bound(B, k, A[r]);
    double se[NCH], sr[NCH], sm[NCH];
    for (int c = 0; c < NCH; ++c) se[c] = sr[c] = sm[c] = 0.0;
    for (uint32_t s = lo + lane; s < hi; s += 32) {
        const uint32_t u = perm_b[s];
        const R d = D[u];
        R w[NCH];
        if constexpr (NCH == 3) {
            const R cc = cpsi[s], ss = spsi[s];  // sorted-order phases
            w[0] = xmul(xmul(cc, cc), d);
            w[1] = xmul(xmul(cc, ss), d);
            w[2] = xmul(xmul(ss, ss), d);
        } else {
            w[0] = d;
        }
        const R bs = B[s];
        const R e_ell = r < n ? xexp(xmul(R(2), xsub(bs, A[r]))) : R(0);
        const R e_rho = r >= 1 ? xexp(xmul(R(2), xsub(A[r - 1], bs))) : R(0);
        for (int c = 0; c < NCH; ++c) {
            se[c] += (double)w[c] * (double)e_ell;
            sr[c] += (double)w[c] * (double)e_rho;
            sm[c] += (double)w[c];
        }
    }
    for (int off = 16; off > 0; off >>= 1)
        for (int c = 0; c < NCH; ++c) {
            se[c] += __shfl_xor_sync(FULL, se[c], off);
            sr[c] += __shfl_xor_sync(FULL, sr[c], off);
            sm[c] += __shfl_xor_sync(FULL, sm[c], off);
        }
    if (lane == 0) {
        for (int c = 0; c < NCH; ++c) {
            if (r < n) ell[(size_t)c * n + r] = (R)se[c];
            if (r >= 1) rho[(size_t)c * n + r - 1] = (R)sr[c];
            mass[(size_t)c * (n + 1) + r] = (R)sm[c];
        }
    }
}

template <class R>
__global__ void lx_double_anchors(const R* __restrict__ A, uint32_t n, R* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = xmul(R(2), A[i]);
}

// Lower triangle (sorted js <= is), mirrored: M[u_i][u_j] = M[u_j][u_i].
template <class R, int NCH>
__global__ void lx_gram_out(const R* __restrict__ A, uint32_t n, const uint32_t* __restrict__ perm_a,
                            const R* __restrict__ U, const R* __restrict__ V, const R* __restrict__ Cm,
                            const R* __restrict__ cphi, const R* __restrict__ sphi, R* __restrict__ M) {
    const uint32_t is = blockIdx.y * blockDim.y + threadIdx.y;
    const uint32_t js = blockIdx.x * blockDim.x + threadIdx.x;
    if (is >= n || js > is) return;
    const R e = xexp(xsub(A[js], A[is]));
    R g[NCH];
    for (int c = 0; c < NCH; ++c) {
        const R* Uc = U + (size_t)c * n;
        const R* Vc = V + (size_t)c * n;
        const R* Cc = Cm + (size_t)c * (n + 1);
        g[c] = xmul(e, xadd(xadd(Uc[js], xsub(Cc[is], Cc[js])), Vc[is]));
    }
    const uint32_t ui = perm_a[is], uj = perm_a[js];
    R m = g[0];
    if constexpr (NCH == 3) {
        // operator.hpp:240-242 evaluated with (i, j) = (max, min) user index so
        // the mirrored entries are literally the same value
        const uint32_t hs = ui > uj ? is : js, ls = ui > uj ? js : is;  // sorted-order phases
        const R ci = cphi[hs], si = sphi[hs], cj = cphi[ls], sj = sphi[ls];
        m = xadd(xadd(xmul(xmul(ci, cj), g[0]), xmul(xadd(xmul(ci, sj), xmul(si, cj)), g[1])),
                 xmul(xmul(si, sj), g[2]));
    }
    M[(size_t)ui * n + uj] = m;
    M[(size_t)uj * n + ui] = m;
}

// inverse permutation: pos[perm[i]] = i
__global__ void lx_invert_perm(const uint32_t* __restrict__ perm, uint32_t m, uint32_t* __restrict__ pos) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) pos[perm[i]] = i;
}

// D_bar[t] = sum_i exp(-|a_i/t - b_t/t|) * Y[i][t]  (gradients.hpp:211-217), user order
template <class R>
__global__ void lx_gram_vjp_contract(const R* __restrict__ A, const uint32_t* __restrict__ pos_a, uint32_t n,
                                     const R* __restrict__ B, const uint32_t* __restrict__ pos_b, uint32_t k,
                                     const R* __restrict__ Y, R* __restrict__ Dbar) {
    const uint32_t tcol = blockIdx.x * blockDim.x + threadIdx.x;
    if (tcol >= k) return;
    const R bt = B[pos_b[tcol]];
    R acc = R(0);
    for (uint32_t i = 0; i < n; ++i) {
        const R ai = A[pos_a[i]];
        const R d = xsub(ai, bt);
        acc = xfma(xexp(-(d < R(0) ? -d : d)), Y[(size_t)i * k + tcol], acc);
    }
    Dbar[tcol] = acc;
}

// Cotangent checks of gram_vjp_weights (gradients.hpp:196-205) on the device:
// flags[0] = max |G_ij| and flags[1] = max |G_ij - G_ji| over i > j, flags[2]
// != 0 when an entry is not finite.  Non-negative IEEE values order like their
// bit patterns, so the maxima are integer atomicMax on the bits.
template <class R>
__global__ void lx_sym_check(const R* __restrict__ G, uint32_t n, R* __restrict__ flags) {
    using U = typename std::conditional<sizeof(R) == 8, unsigned long long, unsigned int>::type;
    R mabs = R(0), masym = R(0);
    int bad = 0;
    const size_t total = (size_t)n * n;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
        const uint32_t i = (uint32_t)(e / n), j = (uint32_t)(e % n);
        const R v = G[e];
        bad |= !isfinite(v);
        if (j < i) {
            const R d = v - G[(size_t)j * n + i];
            mabs = fmax(mabs, v < R(0) ? -v : v);
            masym = fmax(masym, d < R(0) ? -d : d);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        mabs = fmax(mabs, __shfl_xor_sync(0xffffffffu, mabs, o));
        masym = fmax(masym, __shfl_xor_sync(0xffffffffu, masym, o));
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
    }
    if ((threadIdx.x & 31) == 0) {
        U* f = reinterpret_cast<U*>(flags);
        if (mabs == mabs) atomicMax(&f[0], *reinterpret_cast<const U*>(&mabs));
        if (masym == masym) atomicMax(&f[1], *reinterpret_cast<const U*>(&masym));
        if (bad) f[2] = U(1);
    }
}

}  // namespace gram
}  // namespace lx
