// similarity.cu -- fp64 Pearson similarity as a DMMA SYRK with a fused epilogue.
//
// Replaces simmatrix.py:105-123 pearson_similarity + _kernels.py:17-37 pearson_kernel
// (reference: xc = x - mean(x); inv = 1/||xc|| or 0; out[i,j] = clamp(sum_k
// xc_ik xc_jk * inv_i * inv_j); out[i,i] = 1; mirrored).
//
// B200 design:
//   * prologue kernel centres each row once and writes Xc into a zero-padded
//     workspace (row stride Lp = roundup(L, 16)) plus inv[n];
//   * SYRK kernel: one CTA per upper-triangular 128x128 tile (I <= J), 8 warps,
//     3-stage cp.async pipeline of 128x16 fp64 panels, `mma.sync.m8n8k4.f64`
//     (DMMA; sm_100a has no tcgen05 kind::f64), warp tile 64x32;
//   * epilogue stages the tile in shared memory and writes S[I,J] and the
//     mirrored S[J,I] from the SAME value, so S is exactly symmetric; the
//     diagonal tile only uses its upper triangle; diagonal = 1, zero-norm rows 0,
//     clamp to [-1, 1].
#include "common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>

namespace {

constexpr int PBM = 128;          // tile rows / cols
constexpr int PBK = 16;           // k panel
constexpr int PSTR = PBK + 4;     // smem row stride (doubles): conflict-free fragments
constexpr int PSTAGES = 3;
constexpr int PTHREADS = 256;
constexpr int TSTR = PBM + 1;     // epilogue tile stride (doubles)

__global__ void center_rows_kernel(const double *__restrict__ X, int64_t n, int64_t L, int64_t Lp,
                                   double *__restrict__ Xc, double *__restrict__ inv) {
    int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    int lane = threadIdx.x & 31;
    if (row >= n) return;
    const double *x = X + row * L;
    double s = 0.0;
    for (int64_t k = lane; k < L; k += 32) s += x[k];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    double mean = s / (double)L;
    double q = 0.0;
    double *xc = Xc + row * Lp;
    for (int64_t k = lane; k < Lp; k += 32) {
        double v = k < L ? x[k] - mean : 0.0;
        xc[k] = v;
        q = fma(v, v, q);
    }
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if (lane == 0) {
        double nrm = sqrt(q);
        inv[row] = nrm > 0.0 ? 1.0 / nrm : 0.0;
    }
}

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool valid) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void tile_of(int64_t t, int64_t nb, int64_t &I, int64_t &J) {
    // row-major enumeration of the upper triangle: row I has nb - I tiles
    double a = 2.0 * nb + 1.0;
    int64_t i = (int64_t)floor((a - sqrt(a * a - 8.0 * (double)t)) / 2.0);
    if (i < 0) i = 0;
    if (i > nb - 1) i = nb - 1;
    auto start = [&](int64_t r) { return r * nb - r * (r - 1) / 2; };
    while (i > 0 && start(i) > t) i--;
    while (i + 1 < nb && start(i + 1) <= t) i++;
    I = i;
    J = i + (t - start(i));
}

__global__ void __launch_bounds__(PTHREADS, 1)
syrk_dmma_kernel(const double *__restrict__ Xc, const double *__restrict__ inv, int64_t n, int64_t Lp,
                 double *__restrict__ S) {
    extern __shared__ __align__(16) double psmem[];
    double *As = psmem;                          // [PSTAGES][PBM][PSTR]
    double *Bs = psmem + PSTAGES * PBM * PSTR;   // [PSTAGES][PBM][PSTR]
    const int64_t nb = (n + PBM - 1) / PBM;
    int64_t I, J;
    tile_of(blockIdx.x, nb, I, J);
    const int64_t i0 = I * PBM, j0 = J * PBM;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2;   // 0..1 -> 64-row slab
    const int wn = warp & 3;    // 0..3 -> 32-col slab
    const int nk = (int)(Lp / PBK);

    auto load_stage = [&](int stage, int kt) {
        const int64_t k0 = (int64_t)kt * PBK;
        double *as = As + stage * PBM * PSTR;
        double *bs = Bs + stage * PBM * PSTR;
#pragma unroll
        for (int c = tid; c < PBM * (PBK / 2); c += PTHREADS) {
            int r = c / (PBK / 2), q = c % (PBK / 2);
            int64_t gi = i0 + r, gj = j0 + r;
            cp_async16(as + r * PSTR + 2 * q, Xc + (gi < n ? gi : 0) * Lp + k0 + 2 * q, gi < n);
            cp_async16(bs + r * PSTR + 2 * q, Xc + (gj < n ? gj : 0) * Lp + k0 + 2 * q, gj < n);
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < PSTAGES - 1; s++) {
        if (s < nk) load_stage(s, s);
        cp_async_commit();
    }
    const int fr = lane >> 2, fc = lane & 3;
    for (int kt = 0; kt < nk; kt++) {
        cp_async_wait<PSTAGES - 2>();
        __syncthreads();
        int nxt = kt + PSTAGES - 1;
        if (nxt < nk) load_stage(nxt % PSTAGES, nxt);
        cp_async_commit();
        const double *as = As + (kt % PSTAGES) * PBM * PSTR + (wm * 64) * PSTR;
        const double *bs = Bs + (kt % PSTAGES) * PBM * PSTR + (wn * 32) * PSTR;
#pragma unroll
        for (int kk = 0; kk < PBK; kk += 4) {
            double af[8], bf[4];
#pragma unroll
            for (int a = 0; a < 8; a++) af[a] = as[(a * 8 + fr) * PSTR + kk + fc];
#pragma unroll
            for (int b = 0; b < 4; b++) bf[b] = bs[(b * 8 + fr) * PSTR + kk + fc];
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // ---- epilogue: scale, zero-norm, clamp into the smem tile T[128][129]
    double *T = psmem;
#pragma unroll
    for (int a = 0; a < 8; a++) {
        int r = wm * 64 + a * 8 + fr;
        int64_t gi = i0 + r;
        double ii = gi < n ? inv[gi] : 0.0;
#pragma unroll
        for (int b = 0; b < 4; b++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                int c = wn * 32 + b * 8 + fc * 2 + h;
                int64_t gj = j0 + c;
                double jj = gj < n ? inv[gj] : 0.0;
                double v;
                if (ii == 0.0 || jj == 0.0) {
                    v = 0.0;
                } else {
                    v = acc[a][b][h] * ii * jj;
                    v = v > 1.0 ? 1.0 : (v < -1.0 ? -1.0 : v);
                }
                T[r * TSTR + c] = v;
            }
        }
    }
    __syncthreads();
    const bool diag = (I == J);
    // rows of the I block: S[i0 + r][j0 + c]
    for (int e = tid; e < PBM * PBM; e += PTHREADS) {
        int r = e / PBM, c = e % PBM;
        int64_t gi = i0 + r, gj = j0 + c;
        if (gi >= n || gj >= n) continue;
        double v;
        if (!diag) v = T[r * TSTR + c];
        else v = r < c ? T[r * TSTR + c] : (r == c ? 1.0 : T[c * TSTR + r]);
        S[gi * n + gj] = v;
    }
    if (!diag) {
        // mirrored rows of the J block: S[j0 + c][i0 + r] = T[r][c]
        for (int e = tid; e < PBM * PBM; e += PTHREADS) {
            int c = e / PBM, r = e % PBM;
            int64_t gi = i0 + r, gj = j0 + c;
            if (gi >= n || gj >= n) continue;
            S[gj * n + gi] = T[r * TSTR + c];
        }
    }
}


// ---------------------------------------------------------------- TMA-fed SYRK
// Same tiling and fused epilogue as syrk_dmma_kernel; the operand panels arrive by TMA
// (cp.async.bulk.tensor.2d over a tensor map of Xc, 128 rows x 16 doubles = one 128-byte
// swizzled row per Xc row) into a 4-stage mbarrier ring instead of 4,096 cp.async per
// panel.  The 128-byte swizzle (16-byte chunk c of row r at c ^ (r & 7)) lets a lane read
// its fragment pair for two k-steps with one conflict-free 16-byte load: lane (fr, fc)
// takes k = 4 fc + s in k-step s (A and B alike), so steps 2h and 2h+1 need chunk 2 fc + h.
// Out-of-range rows (n not a multiple of 128) are zero-filled by the TMA unit.
constexpr int TS_STAGES = 4;
constexpr int TS_PANEL = PBM * PBK;   // doubles per operand panel (16 KB)

__device__ __forceinline__ unsigned ts_smem(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(PTHREADS, 1)
syrk_tma_kernel(const __grid_constant__ CUtensorMap tmX, const double *__restrict__ inv, int64_t n, int64_t Lp,
                double *__restrict__ S) {
    extern __shared__ __align__(16) unsigned char ts_raw[];
    __shared__ __align__(8) uint64_t bar[TS_STAGES];
    // the swizzled boxes need 1024-byte aligned destinations
    double *base = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(ts_raw) + 1023) & ~(uintptr_t)1023);
    const int64_t nb = (n + PBM - 1) / PBM;
    int64_t I, J;
    tile_of(blockIdx.x, nb, I, J);
    const int64_t i0 = I * PBM, j0 = J * PBM;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 2, wn = warp & 3;
    const int nk = (int)(Lp / PBK);
    if (tid == 0) {
        for (int s = 0; s < TS_STAGES; s++)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(ts_smem(&bar[s])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // Xc (n x Lp doubles, ~100 MB at n = 50k) stays in L2 while the 8 n^2 bytes of S stream past
    // it: operand panels are loaded evict_last, S is stored evict_first (st.global.cs)
    uint64_t pol = 0;
    if (tid == 0) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
    auto issue = [&](int kt) {   // thread 0: both operand panels of k-tile kt
        const int s = kt % TS_STAGES;
        double *as = base + (size_t)s * 2 * TS_PANEL, *bs = as + TS_PANEL;
        const unsigned b = ts_smem(&bar[s]);
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(2u * TS_PANEL * 8u)
                     : "memory");
        const int k0 = kt * PBK;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
                ts_smem(as)),
            "l"(&tmX), "r"(k0), "r"((int)i0), "r"(b), "l"(pol)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(
                ts_smem(bs)),
            "l"(&tmX), "r"(k0), "r"((int)j0), "r"(b), "l"(pol)
            : "memory");
    };
    if (tid == 0)
        for (int kt = 0; kt < TS_STAGES - 1 && kt < nk; kt++) issue(kt);

    double acc[8][4][2];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    const int fr = lane >> 2, fc = lane & 3;
    for (int kt = 0; kt < nk; kt++) {
        __syncthreads();   // k-tile kt-1 is consumed: its stage may be refilled
        if (tid == 0 && kt + TS_STAGES - 1 < nk) issue(kt + TS_STAGES - 1);
        const int s = kt % TS_STAGES;
        {
            const unsigned b = ts_smem(&bar[s]), par = (unsigned)((kt / TS_STAGES) & 1);
            asm volatile(
                "{\n .reg .pred p;\n TS_W_%=:\n"
                " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
                " @!p bra TS_W_%=;\n}\n" ::"r"(b),
                "r"(par)
                : "memory");
        }
        const double *as = base + (size_t)s * 2 * TS_PANEL + (wm * 64) * PBK;
        const double *bs = base + (size_t)s * 2 * TS_PANEL + TS_PANEL + (wn * 32) * PBK;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int ch = ((2 * fc + h) ^ fr) * 2;   // swizzled 16-byte chunk of rows 8q + fr
            double2 af[8], bf[4];
#pragma unroll
            for (int a = 0; a < 8; a++) af[a] = *reinterpret_cast<const double2 *>(as + (a * 8 + fr) * PBK + ch);
#pragma unroll
            for (int b = 0; b < 4; b++) bf[b] = *reinterpret_cast<const double2 *>(bs + (b * 8 + fr) * PBK + ch);
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a].x, bf[b].x);
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a].y, bf[b].y);
        }
    }
    __syncthreads();   // every panel consumed: the ring becomes the epilogue tile

    // ---- epilogue: scale, zero-norm, clamp into the smem tile T[128][129]
    double *T = base;
#pragma unroll
    for (int a = 0; a < 8; a++) {
        const int r = wm * 64 + a * 8 + fr;
        const int64_t gi = i0 + r;
        const double ii = gi < n ? inv[gi] : 0.0;
#pragma unroll
        for (int b = 0; b < 4; b++) {
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int c = wn * 32 + b * 8 + fc * 2 + h;
                const int64_t gj = j0 + c;
                const double jj = gj < n ? inv[gj] : 0.0;
                double v;
                if (ii == 0.0 || jj == 0.0) {
                    v = 0.0;
                } else {
                    v = acc[a][b][h] * ii * jj;
                    v = v > 1.0 ? 1.0 : (v < -1.0 ? -1.0 : v);
                }
                T[r * TSTR + c] = v;
            }
        }
    }
    __syncthreads();
    const bool diag = (I == J);
    // rows of the I block, two columns per store when the row start is 16-byte aligned
    const bool vec = ((n & 1) == 0);
    for (int e = tid; e < PBM * PBM / 2; e += PTHREADS) {
        const int r = e / (PBM / 2), c = 2 * (e % (PBM / 2));
        const int64_t gi = i0 + r, gj = j0 + c;
        if (gi >= n || gj >= n) continue;
        double v0, v1;
        if (!diag) {
            v0 = T[r * TSTR + c];
            v1 = T[r * TSTR + c + 1];
        } else {
            v0 = r < c ? T[r * TSTR + c] : (r == c ? 1.0 : T[c * TSTR + r]);
            v1 = r < c + 1 ? T[r * TSTR + c + 1] : (r == c + 1 ? 1.0 : T[(c + 1) * TSTR + r]);
        }
        if (vec && gj + 1 < n) {
            __stcs(reinterpret_cast<double2 *>(S + gi * n + gj), make_double2(v0, v1));
        } else {
            S[gi * n + gj] = v0;
            if (gj + 1 < n) S[gi * n + gj + 1] = v1;
        }
    }
    if (!diag) {
        // mirrored rows of the J block: S[j0 + c][i0 + r] = T[r][c], two rows r per store
        for (int e = tid; e < PBM * PBM / 2; e += PTHREADS) {
            const int c = e / (PBM / 2), r = 2 * (e % (PBM / 2));
            const int64_t gi = i0 + r, gj = j0 + c;
            if (gi >= n || gj >= n) continue;
            const double v0 = T[r * TSTR + c], v1 = T[(r + 1) * TSTR + c];
            if (vec && gi + 1 < n) {
                __stcs(reinterpret_cast<double2 *>(S + gj * n + gi), make_double2(v0, v1));
            } else {
                S[gj * n + gi] = v0;
                if (gi + 1 < n) S[gj * n + gi + 1] = v1;
            }
        }
    }
}

// ---------------------------------------------------------------- validation
__global__ void validate_kernel(const double *__restrict__ S, int64_t n, int32_t *flags) {
    __shared__ double A[32][33];
    __shared__ double B[32][33];
    const int64_t nb = (n + 31) / 32;
    int64_t I, J;
    {
        int64_t t = blockIdx.x;
        double a = 2.0 * nb + 1.0;
        int64_t i = (int64_t)floor((a - sqrt(a * a - 8.0 * (double)t)) / 2.0);
        if (i < 0) i = 0;
        if (i > nb - 1) i = nb - 1;
        auto start = [&](int64_t r) { return r * nb - r * (r - 1) / 2; };
        while (i > 0 && start(i) > t) i--;
        while (i + 1 < nb && start(i + 1) <= t) i++;
        I = i;
        J = i + (t - start(i));
    }
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    int f = 0;
    for (int r = ty; r < 32; r += 8) {
        int64_t gi = I * 32 + r, gj = J * 32 + tx;
        double a = (gi < n && gj < n) ? S[gi * n + gj] : 0.0;
        A[r][tx] = a;
        int64_t hi = J * 32 + r, hj = I * 32 + tx;
        double b = (hi < n && hj < n) ? S[hi * n + hj] : 0.0;
        B[r][tx] = b;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        int64_t gi = I * 32 + r, gj = J * 32 + tx;
        if (gi >= n || gj >= n) continue;
        double a = A[r][tx];
        double b = B[tx][r];   // S[gj][gi]
        if (isnan(a) || isnan(b)) f |= TG_BAD_NAN;
        if (!(a == b)) f |= TG_BAD_ASYM;
        if (a < -1.0 || a > 1.0 || b < -1.0 || b > 1.0) f |= TG_BAD_RANGE;
        if (gi == gj && !(a == 1.0)) f |= TG_BAD_DIAG;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    if (tx == 0 && f) atomicOr(flags, f);
}


// ---------------------------------------------------------------- reference-order variant
// _kernels.py:17-37 evaluated in the reference's own arithmetic order: for each
// pair a sequential k loop s += xc_ik * xc_jk (separate rounding of the product
// and the sum, no FMA), r = (s * inv_i) * inv_j, clamp.  Bit-identical to the
// reference's S given the same xc / inv (its numpy prologue).  CTA tile 64 x 64
// pairs (upper triangle), 16 x 16 threads with 4 x 4 pairs each, k staged in
// shared memory 16 at a time; FP64 pipe bound (2 ops per pair per k).
constexpr int RX_T = 64;
constexpr int RX_K = 16;

__global__ void __launch_bounds__(256) pearson_refexact_kernel(const double *__restrict__ xc,
                                                                const double *__restrict__ inv, int64_t n,
                                                                int64_t L, double *__restrict__ S) {
    // upper-triangular tile (I <= J) from the linear block id
    const int64_t nt = (n + RX_T - 1) / RX_T;
    int64_t b = blockIdx.x, I = 0;
    while (b >= nt - I) { b -= nt - I; I++; }
    const int64_t J = I + b;
    __shared__ double As[RX_K][RX_T + 1];
    __shared__ double Bs[RX_K][RX_T + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = I * RX_T, j0 = J * RX_T;
    double acc[4][4];
#pragma unroll
    for (int r = 0; r < 4; r++)
#pragma unroll
        for (int c = 0; c < 4; c++) acc[r][c] = 0.0;
    for (int64_t k0 = 0; k0 < L; k0 += RX_K) {
        for (int e = threadIdx.x; e < RX_T * RX_K; e += 256) {
            const int rr = e / RX_K, kk = e % RX_K;
            const int64_t gi = i0 + rr, gj = j0 + rr, gk = k0 + kk;
            As[kk][rr] = (gi < n && gk < L) ? xc[gi * L + gk] : 0.0;
            Bs[kk][rr] = (gj < n && gk < L) ? xc[gj * L + gk] : 0.0;
        }
        __syncthreads();
        const int kend = (int)(L - k0 < RX_K ? L - k0 : RX_K);
        for (int kk = 0; kk < kend; kk++) {
            double a[4], bv[4];
#pragma unroll
            for (int r = 0; r < 4; r++) a[r] = As[kk][ty * 4 + r];
#pragma unroll
            for (int c = 0; c < 4; c++) bv[c] = Bs[kk][tx * 4 + c];
#pragma unroll
            for (int r = 0; r < 4; r++)
#pragma unroll
                for (int c = 0; c < 4; c++) acc[r][c] = __dadd_rn(acc[r][c], __dmul_rn(a[r], bv[c]));
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; r++) {
        const int64_t i = i0 + ty * 4 + r;
        if (i >= n) continue;
#pragma unroll
        for (int c = 0; c < 4; c++) {
            const int64_t j = j0 + tx * 4 + c;
            if (j >= n || j < i) continue;
            if (j == i) { S[i * n + i] = 1.0; continue; }
            double v;
            if (inv[i] == 0.0 || inv[j] == 0.0) {
                v = 0.0;
            } else {
                v = __dmul_rn(__dmul_rn(acc[r][c], inv[i]), inv[j]);
                if (v > 1.0) v = 1.0;
                else if (v < -1.0) v = -1.0;
            }
            S[i * n + j] = v;
            S[j * n + i] = v;
        }
    }
}

}  // namespace

// Tensor map of the centred, padded series Xc (n rows of Lp doubles): 128 x 16 boxes, 128-byte
// swizzle, zero fill past row n.  cuTensorMapEncodeTiled comes from the driver through the
// runtime's entry-point query (no libcuda link).  Returns 0 on success.
static int tg_tensor_map_xc(CUtensorMap *tm, const double *Xc, int64_t n, int64_t Lp) {
    static PFN_cuTensorMapEncodeTiled encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return 1;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
    }
    const cuuint64_t dims[2] = {(cuuint64_t)Lp, (cuuint64_t)n};
    const cuuint64_t strides[1] = {(cuuint64_t)Lp * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)PBK, (cuuint32_t)PBM};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(Xc), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? 0 : 2;
}

TG_API size_t tg_pearson_workspace_bytes(int64_t n, int64_t L) {
    int64_t Lp = (L + PBK - 1) / PBK * PBK;
    return tg_align_up((size_t)n * Lp * sizeof(double), 256) + tg_align_up((size_t)n * sizeof(double), 256) + 512;
}

TG_API int tg_pearson_f64(const double *X, int64_t n, int64_t L, double *S, void *ws, size_t ws_bytes,
                          void *stream) {
    if (n < 1 || L < 1 || !X || !S) return TG_ERR_ARG;
    if (ws_bytes < tg_pearson_workspace_bytes(n, L)) return TG_ERR_WORKSPACE;
    int64_t Lp = (L + PBK - 1) / PBK * PBK;
    TgArena ar(ws, ws_bytes);
    double *Xc = ar.take<double>((size_t)n * Lp);
    double *inv = ar.take<double>(n);
    cudaStream_t st = tg_stream(stream);
    center_rows_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(X, n, L, Lp, Xc, inv); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    const int64_t nb = (n + PBM - 1) / PBM;
    const int64_t tiles = nb * (nb + 1) / 2;
    size_t smem = (size_t)2 * PSTAGES * PBM * PSTR * sizeof(double);
    size_t smem_epi = (size_t)PBM * TSTR * sizeof(double);
    if (smem_epi > smem) smem = smem_epi;
    static const bool use_cp_async = std::getenv("TG_SYRK_CPASYNC") != nullptr;   // A/B switch (development)
    CUtensorMap tm;
    if (!use_cp_async && n <= INT_MAX && tg_tensor_map_xc(&tm, Xc, n, Lp) == 0) {
        size_t tsm = (size_t)TS_STAGES * 2 * TS_PANEL * sizeof(double);
        if (smem_epi > tsm) tsm = smem_epi;
        tsm += 1024;   // alignment slack for the swizzled boxes
        TG_CUDA_CHECK(cudaFuncSetAttribute(syrk_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm));
        syrk_tma_kernel<<<(unsigned)tiles, PTHREADS, tsm, st>>>(tm, inv, n, Lp, S); tg_count_launch(1);
        TG_LAUNCH_CHECK();
        return TG_OK;
    }
    // per call: the attribute is per device, and a cached flag would skip a second device
    TG_CUDA_CHECK(cudaFuncSetAttribute(syrk_dmma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    syrk_dmma_kernel<<<(unsigned)tiles, PTHREADS, smem, st>>>(Xc, inv, n, Lp, S); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_validate_f64(const double *S, int64_t n, int32_t *flags, void *stream) {
    if (n < 1 || !S || !flags) return TG_ERR_ARG;
    cudaStream_t st = tg_stream(stream);
    TG_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(int32_t), st));
    const int64_t nb = (n + 31) / 32;
    validate_kernel<<<(unsigned)(nb * (nb + 1) / 2), 256, 0, st>>>(S, n, flags); tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}

TG_API int tg_pearson_refexact_f64(const double *xc, const double *inv, int64_t n, int64_t L, double *S, void *stream) {
    if (n < 1 || L < 0 || !xc || !inv || !S) return TG_ERR_ARG;
    const int64_t nt = (n + RX_T - 1) / RX_T;
    const int64_t tiles = nt * (nt + 1) / 2;
    if (tiles > 0x7fffffffLL) return TG_ERR_ARG;
    pearson_refexact_kernel<<<(unsigned)tiles, 256, 0, tg_stream(stream)>>>(xc, inv, n, L, S);
    tg_count_launch(1);
    TG_LAUNCH_CHECK();
    return TG_OK;
}
