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
