/* kernels.c -- O1: the paper's benchmark kernels, unsliced, as plain loops (TEST INFRASTRUCTURE).
 *
 * PAPER.md names the kernels only (tb:description); the definitions below are the
 * readings R17/R18 of SURVEY.md §8(c) O1, restated in DESIGN.md §3.  Each loop is the plain
 * definition of one output element; there is no blocking, tiling or reordering, so slicing
 * (a slice only remaps block indices) must reproduce exactly these values.
 * Floating-point kernels accumulate in fp64 from the fp32/bf16 inputs and round once.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OUT_N(idx, n_idx, n_all) ((idx) ? (n_idx) : (size_t)(n_all))
#define FLAT(idx, o) ((idx) ? (size_t)(idx)[o] : (size_t)(o))

/* PC, pointer chasing ("Traversing an array randomly", 40M accesses, 256x16384 threads).
 * Thread t starts at start(t) = (t * 2654435761 mod 2^32) mod N and follows next[] `hops`
 * times; out_p[t] = final node, out_acc[t] = sum of the visited nodes (mod 2^32). */
void or_pc(const int32_t* next, uint32_t n_nodes, uint32_t hops, uint32_t n_threads,
           const int64_t* idx, size_t n_idx, int32_t* out_p, uint32_t* out_acc) {
    size_t n = OUT_N(idx, n_idx, n_threads);
    for (size_t o = 0; o < n; ++o) {
        uint32_t t = (uint32_t)FLAT(idx, o);
        uint32_t p = (uint32_t)(t * 2654435761u) % n_nodes;
        uint32_t acc = 0;
        for (uint32_t h = 0; h < hops; ++h) {
            p = (uint32_t)next[p];
            acc += p;
        }
        out_p[o] = (int32_t)p;
        out_acc[o] = acc;
    }
}

static int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* SAD (MPEG motion estimation on a 1920x1072 image).  For macroblock m = my*(W/16)+mx and
 * search offset (dx,dy) in [0,32]^2 (displacement dx-16, dy-16), the sum over the 16x16 block of
 * |cur - ref|, reference pixels clamped to the frame edge.  out[m*1089 + dy*33 + dx]. */
void or_sad(const uint8_t* cur, const uint8_t* ref, int width, int height,
            const int64_t* idx, size_t n_idx, uint16_t* out) {
    int mbw = width / 16, mbh = height / 16;
    size_t n_all = (size_t)mbw * mbh * 1089;
    size_t n = OUT_N(idx, n_idx, n_all);
    for (size_t o = 0; o < n; ++o) {
        size_t flat = FLAT(idx, o);
        int m = (int)(flat / 1089), pos = (int)(flat % 1089);
        int dy = pos / 33, dx = pos % 33;
        int mx = m % mbw, my = m / mbw;
        uint32_t sum = 0;
        for (int r = 0; r < 16; ++r)
            for (int c = 0; c < 16; ++c) {
                int cy = my * 16 + r, cx = mx * 16 + c;
                int ry = clampi(cy + dy - 16, 0, height - 1);
                int rx = clampi(cx + dx - 16, 0, width - 1);
                int d = (int)cur[(size_t)cy * width + cx] - (int)ref[(size_t)ry * width + rx];
                sum += (uint32_t)(d < 0 ? -d : d);
            }
        out[o] = (uint16_t)sum;
    }
}

/* SPMV (CUSP CSR): y_i = sum_j a_ij x_j in row order, fp64 accumulate, one rounding.
 * absrow_i = sum_j |a_ij x_j| (scale of the normwise tolerance). */
void or_spmv(const int32_t* rowptr, const int32_t* cols, const float* vals, const float* x,
             int n_rows, const int64_t* idx, size_t n_idx, float* y, double* absrow) {
    size_t n = OUT_N(idx, n_idx, n_rows);
    for (size_t o = 0; o < n; ++o) {
        size_t i = FLAT(idx, o);
        double s = 0.0, a = 0.0;
        for (int j = rowptr[i]; j < rowptr[i + 1]; ++j) {
            double t = (double)vals[j] * (double)x[cols[j]];
            s += t;
            a += fabs(t);
        }
        y[o] = (float)s;
        if (absrow) absrow[o] = a;
    }
}

/* ST, 7-point stencil on a regular 3-D grid (Parboil).  Layout in[z][y][x].
 * Interior: out = c1*(sum of the 6 face neighbours) - c0*in; boundary points: out = in. */
void or_stencil(const float* in, int nx, int ny, int nz, float c0, float c1,
                const int64_t* idx, size_t n_idx, float* out, double* absmag) {
    size_t n_all = (size_t)nx * ny * nz;
    size_t n = OUT_N(idx, n_idx, n_all);
    size_t sy = (size_t)nx, sz = (size_t)nx * ny;
    for (size_t o = 0; o < n; ++o) {
        size_t f = FLAT(idx, o);
        int x = (int)(f % nx), y = (int)((f / nx) % ny), z = (int)(f / sz);
        double v = in[f];
        if (x == 0 || y == 0 || z == 0 || x == nx - 1 || y == ny - 1 || z == nz - 1) {
            out[o] = in[f];
            if (absmag) absmag[o] = fabs(v);
            continue;
        }
        double nb[6] = {in[f - sz], in[f + sz], in[f - sy], in[f + sy], in[f - 1], in[f + 1]};
        double s = 0.0, a = 0.0;
        for (int k = 0; k < 6; ++k) { s += nb[k]; a += fabs(nb[k]); }
        out[o] = (float)((double)c1 * s - (double)c0 * v);
        if (absmag) absmag[o] = (double)c1 * a + (double)c0 * fabs(v);
    }
}

static double bf16_to_double(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* MM: C = A B, A MxK, B KxN given K-major as Bt (N x K); bf16 inputs, fp32 output.
 * C[m][n] = sum_k A[m][k] * Bt[n][k], fp64 accumulate in k order, one rounding. */
void or_mm(const uint16_t* A, const uint16_t* Bt, int M, int N, int K,
           const int64_t* idx, size_t n_idx, float* C, double* absmag) {
    size_t n = OUT_N(idx, n_idx, (size_t)M * N);
    for (size_t o = 0; o < n; ++o) {
        size_t f = FLAT(idx, o);
        size_t m = f / N, nn = f % N;
        double s = 0.0, a = 0.0;
        for (int k = 0; k < K; ++k) {
            double t = bf16_to_double(A[m * K + k]) * bf16_to_double(Bt[nn * K + k]);
            s += t;
            a += fabs(t);
        }
        C[o] = (float)s;
        if (absmag) absmag[o] = a;
    }
}

/* MRIQ (Parboil MRI-Q ComputeQ): for voxel i,
 * Qr_i = sum_k phiMag_k cos(2 pi (kx_k x_i + ky_k y_i + kz_k z_i)), Qi_i likewise with sin. */
void or_mriq(const float* x, const float* y, const float* z, int num_x,
             const float* kx, const float* ky, const float* kz, const float* phimag, int num_k,
             const int64_t* idx, size_t n_idx, float* qr, float* qi, double* absmag) {
    const double two_pi = 6.283185307179586476925286766559;
    size_t n = OUT_N(idx, n_idx, num_x);
    for (size_t o = 0; o < n; ++o) {
        size_t i = FLAT(idx, o);
        double sr = 0.0, si = 0.0, a = 0.0;
        for (int k = 0; k < num_k; ++k) {
            double t = (double)kx[k] * x[i] + (double)ky[k] * y[i] + (double)kz[k] * z[i];
            sr += (double)phimag[k] * cos(two_pi * t);
            si += (double)phimag[k] * sin(two_pi * t);
            a += fabs((double)phimag[k]);
        }
        qr[o] = (float)sr;
        qi[o] = (float)si;
        if (absmag) absmag[o] = a;
    }
}

/* Cumulative normal by Abramowitz & Stegun 26.2.17 (|error| < 7.5e-8), the CUDA SDK
 * BlackScholes polynomial. */
double or_cnd(double d) {
    const double A1 = 0.31938153, A2 = -0.356563782, A3 = 1.781477937, A4 = -1.821255978,
                 A5 = 1.330274429;
    const double RSQRT2PI = 0.39894228040143267793994605993438;
    double K = 1.0 / (1.0 + 0.2316419 * fabs(d));
    double cnd = RSQRT2PI * exp(-0.5 * d * d) * (K * (A1 + K * (A2 + K * (A3 + K * (A4 + K * A5)))));
    if (d > 0) cnd = 1.0 - cnd;
    return cnd;
}

/* BS (SDK Black-Scholes): European call and put, riskless rate R, volatility V.
 * mag = S + X e^{-RT}, the size of the two terms (scale of the normwise tolerance). */
void or_bs(const float* S, const float* X, const float* T, size_t n, double R, double V,
           const int64_t* idx, size_t n_idx, float* call, float* put, double* mag) {
    size_t no = OUT_N(idx, n_idx, n);
    for (size_t o = 0; o < no; ++o) {
        size_t i = FLAT(idx, o);
        double s = S[i], x = X[i], t = T[i];
        double sqrtT = sqrt(t);
        double d1 = (log(s / x) + (R + 0.5 * V * V) * t) / (V * sqrtT);
        double d2 = d1 - V * sqrtT;
        double c1 = or_cnd(d1), c2 = or_cnd(d2);
        double expRT = exp(-R * t);
        call[o] = (float)(s * c1 - x * expRT * c2);
        put[o] = (float)(x * expRT * (1.0 - c2) - s * (1.0 - c1));
        if (mag) mag[o] = s + x * expRT;
    }
}

/* TEA (Wheeler & Needham): 32 cycles, delta 0x9E3779B9, on 64-bit blocks (v0,v1). */
void or_tea(const uint32_t* v, size_t n_pairs, const uint32_t key[4],
            const int64_t* idx, size_t n_idx, uint32_t* out) {
    size_t n = OUT_N(idx, n_idx, n_pairs);
    for (size_t o = 0; o < n; ++o) {
        size_t i = FLAT(idx, o);
        uint32_t v0 = v[2 * i], v1 = v[2 * i + 1], sum = 0;
        for (int c = 0; c < 32; ++c) {
            sum += 0x9E3779B9u;
            v0 += ((v1 << 4) + key[0]) ^ (v1 + sum) ^ ((v1 >> 5) + key[1]);
            v1 += ((v0 << 4) + key[2]) ^ (v0 + sum) ^ ((v0 >> 5) + key[3]);
        }
        out[2 * o] = v0;
        out[2 * o + 1] = v1;
    }
}

void or_tea_decrypt(const uint32_t* v, size_t n_pairs, const uint32_t key[4], uint32_t* out) {
    for (size_t i = 0; i < n_pairs; ++i) {
        uint32_t v0 = v[2 * i], v1 = v[2 * i + 1], sum = 0x9E3779B9u * 32u;
        for (int c = 0; c < 32; ++c) {
            v1 -= ((v0 << 4) + key[2]) ^ (v0 + sum) ^ ((v0 >> 5) + key[3]);
            v0 -= ((v1 << 4) + key[0]) ^ (v1 + sum) ^ ((v1 >> 5) + key[1]);
            sum -= 0x9E3779B9u;
        }
        out[2 * i] = v0;
        out[2 * i + 1] = v1;
    }
}

/* MatrixAdd (Fig. fig:slicing): C = A + B on n x n fp32. */
void or_matadd(const float* A, const float* B, int n, float* C) {
    for (size_t i = 0; i < (size_t)n * n; ++i) C[i] = A[i] + B[i];
}

/* Synthetic streaming kernel (the paper's "testing kernels" P:698-702):
 * y_i = f^fmas(x_i), f(v) = fmaf(v, a, b) (fused multiply-add, one rounding each). */
void or_synth(const float* x, size_t n, int fmas, float a, float b,
              const int64_t* idx, size_t n_idx, float* y) {
    size_t no = OUT_N(idx, n_idx, n);
    for (size_t o = 0; o < no; ++o) {
        float v = x[FLAT(idx, o)];
        for (int c = 0; c < fmas; ++c) v = fmaf(v, a, b);
        y[o] = v;
    }
}
