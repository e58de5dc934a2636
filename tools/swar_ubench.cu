// tools/swar_ubench.cu -- microbenchmark of the K2 inner loop (8x8 register micro-tile per
// thread, operands from shared memory) for several SWAR instruction mixes and launch shapes.
// Reports word-compares per clock per SM (R_int = 32).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o swar_ubench swar_ubench.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("%s -> %s\n", #x, cudaGetErrorString(e));                   \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

// V: 0 = IMAD + IDP4A, 1 = IMAD + IMAD.HI, 2 = LEA.HI, 3 = paper POPC, 4 = IADD3 + IDP4A
template <int V>
__device__ __forceinline__ uint32_t step(uint32_t x, uint32_t y, uint32_t xm, uint32_t ym, uint32_t acc,
                                         uint32_t one, uint32_t sh25) {
    uint32_t u = (x ^ y) | 0x80808080u, p, v, r;
    if (V == 0) {
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(p) : "r"(u), "r"(one), "n"(0xFEFEFEFFu));
        asm("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v) : "r"(p), "r"(xm), "r"(ym));
        asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "n"(0x01010101), "r"(acc));
    } else if (V == 1) {
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(p) : "r"(u), "r"(one), "n"(0xFEFEFEFFu));
        asm("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v) : "r"(p), "r"(xm), "r"(ym));
        asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "r"(sh25), "r"(acc));
    } else if (V == 2) {
        asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(p) : "r"(u), "r"(one), "n"(0xFEFEFEFFu));
        asm("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v) : "r"(p), "r"(xm), "r"(ym));
        r = acc + (v >> 7);
    } else if (V == 3) {
        p = u - 0x01010101u;
        v = ~p & ((x | y) & 0x80808080u);
        r = acc + __popc(v);
    } else {
        p = u - 0x01010101u;
        asm("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v) : "r"(p), "r"(xm), "r"(ym));
        asm("dp4a.u32.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(v), "n"(0x01010101), "r"(acc));
    }
    return r;
}


// Explicitly scheduled 8x8 step: a software pipeline over the 64 pairs in which every ALU op
// (LOP3) is followed by an FMA-pipe op (IADD / IDP4A), kept in order by asm volatile.
__device__ __forceinline__ void step_pipelined(const uint32_t (&x)[8], const uint32_t (&y)[8], const uint32_t (&xm)[8],
                                               const uint32_t (&ym)[8], uint32_t (&acc)[8][8]) {
    uint32_t u[64], p[64], v[64];
#pragma unroll
    for (int q = 0; q < 64 + 3; ++q) {
        if (q < 64) {
            const int i = q >> 3, j = q & 7;
            asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[i]), "r"(y[j]));  // (a^b)|c
        }
        if (q >= 1 && q - 1 < 64) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - 1]) : "r"(u[q - 1]));
        if (q >= 2 && q - 2 < 64) {
            const int i = (q - 2) >> 3, j = (q - 2) & 7;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v[q - 2]) : "r"(p[q - 2]), "r"(xm[i]), "r"(ym[j]));
        }
        if (q >= 3) {
            const int i = (q - 3) >> 3, j = (q - 3) & 7;
            asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;" : "+r"(acc[i][j]) : "r"(v[q - 3]));
        }
    }
}

// MASKS: 0 = compute x & M in registers per k, 1 = load from a second smem plane, 2 = no LDS in the
// loop at all (register-resident operands perturbed per k: the compute ceiling)
template <int V, int MASKS, int NT, int MINB = 1, int UNR = 4, int SYNC = 0>
__global__ void __launch_bounds__(NT, MINB) bench(const uint32_t* __restrict__ g, int reps, uint32_t one,
                                                uint32_t sh25, uint32_t* out, unsigned long long* cycles) {
    __shared__ __align__(16) uint32_t sA[16 * 128], sB[16 * 128], mA[16 * 128], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
        sA[i] = g[i];
        sB[i] = g[i + 32 * 128];
        mA[i] = g[i] & 0x80808080u;
        mB[i] = g[i + 32 * 128] & 0x80808080u;
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    uint32_t x[8], y[8], xm[8], ym[8];
    if (MASKS == 2) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            x[i] = sA[4 * tr + i];
            y[i] = sB[4 * tc + i];
            xm[i] = x[i] & 0x80808080u;
            ym[i] = y[i] & 0x80808080u;
        }
    }
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (SYNC) {  // per-chunk mask transform + barrier, as in k2_tiled
            for (int i = threadIdx.x; i < 16 * 128 / 4; i += NT) {
                uint4 v = reinterpret_cast<const uint4*>(sA)[i];
                v.x &= 0x80808080u; v.y &= 0x80808080u; v.z &= 0x80808080u; v.w &= 0x80808080u;
                reinterpret_cast<uint4*>(mA)[i] = v;
                uint4 w = reinterpret_cast<const uint4*>(sB)[i];
                w.x &= 0x80808080u; w.y &= 0x80808080u; w.z &= 0x80808080u; w.w &= 0x80808080u;
                reinterpret_cast<uint4*>(mB)[i] = w;
            }
            __syncthreads();
        }
#pragma unroll UNR
        for (int k = 0; k < 16; ++k) {
            if (MASKS != 2) {
                const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
                const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
                const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
                const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
                x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
                y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
                if (MASKS == 1) {
                    const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
                    const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
                    const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
                    const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
                    xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
                    ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
                } else {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        xm[i] = x[i] & 0x80808080u;
                        ym[i] = y[i] & 0x80808080u;
                    }
                }
            } else {
                // every (x_i, y_j) pair must change per k, else ptxas hoists the unchanged compares
                // out of the k loop: y_j += one (runtime 1) with an FMA-pipe IMAD, 8 per 256 compute
                // instructions -- the ceiling measured this way is ~3% low
#pragma unroll
                for (int j = 0; j < 8; ++j) asm volatile("mad.lo.u32 %0, %0, 1, %1;" : "+r"(y[j]) : "r"(one));
            }
            if (V == 5) {
                step_pipelined(x, y, xm, ym, acc);
            } else {
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = step<V>(x[i], y[j], xm[i], ym[j], acc[i][j], one, sh25);
            }
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int V, int MASKS, int NT, int MINB = 1, int UNR = 4, int SYNC = 0>
void run(const char* name, const uint32_t* g, int sms, uint32_t* out, unsigned long long* cyc) {
    const int reps = 2000;
    sms *= MINB;  // MINB CTAs per SM
    bench<V, MASKS, NT, MINB, UNR, SYNC><<<sms, NT>>>(g, 10, 1u, 1u << 25, out, cyc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench<V, MASKS, NT, MINB, UNR, SYNC><<<sms, NT>>>(g, reps, 1u, 1u << 25, out, cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    std::vector<unsigned long long> c(sms);
    CK(cudaMemcpy(c.data(), cyc, sms * 8, cudaMemcpyDeviceToHost));
    double mc = 0;
    for (auto v : c) mc += v;
    mc /= sms;
    const double per_block = (double)NT * 64.0 * 16.0 * reps;  // word-compares per block
    printf("{\"variant\": \"%s%s\", \"threads\": %d, \"ctas_per_sm\": %d, \"unroll\": %d, \"cmp_per_clk_per_sm\": %.2f, "
           "\"frac_of_32\": %.3f, \"tcmp_per_s\": %.3f, \"ms\": %.2f, \"eff_mhz\": %.0f}\n",
           name, SYNC ? "+sync" : "", NT, MINB, UNR, MINB * per_block / mc, MINB * per_block / mc / 32.0,
           per_block * sms / (ms * 1e-3) / 1e12, ms, mc / (ms * 1e-3) / 1e6);
}


template <int NT, int MINB, bool LDS>
__global__ void __launch_bounds__(NT, MINB) bench_pf(const uint32_t* __restrict__ g, int reps, uint32_t* out,
                                                      unsigned long long* cycles) {
    __shared__ __align__(16) uint32_t sA[16 * 128], sB[16 * 128], mA[16 * 128], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * 128; i += blockDim.x) {
        sA[i] = g[i];
        sB[i] = g[i + 32 * 128];
        mA[i] = g[i] & 0x80808080u;
        mB[i] = g[i + 32 * 128] & 0x80808080u;
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    auto ld = [&](int k, uint32_t (&x)[8], uint32_t (&y)[8], uint32_t (&xm)[8], uint32_t (&ym)[8]) {
        const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
        const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
        const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
        const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
        const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
        const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
        const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
        const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
        x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
        y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
        xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
        ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
    };
    uint32_t x0[8], y0[8], xm0[8], ym0[8], x1[8], y1[8], xm1[8], ym1[8];
    ld(0, x0, y0, xm0, ym0);
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; k += 2) {
            if (LDS) ld(k + 1, x1, y1, xm1, ym1);
            else {
#pragma unroll
                for (int i = 0; i < 8; ++i) { x1[i] = x0[i] + 1; y1[i] = y0[i]; xm1[i] = xm0[i]; ym1[i] = ym0[i]; }
            }
            step_pipelined(x0, y0, xm0, ym0, acc);
            if (LDS) ld((k + 2) & 15, x0, y0, xm0, ym0);
            else {
#pragma unroll
                for (int i = 0; i < 8; ++i) x0[i] = x1[i] + 1;
            }
            step_pipelined(x1, y1, xm1, ym1, acc);
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int NT, int MINB, bool LDS>
void run_pf(const char* name, const uint32_t* g, int sms, uint32_t* out, unsigned long long* cyc) {
    const int reps = 2000;
    sms *= MINB;
    bench_pf<NT, MINB, LDS><<<sms, NT>>>(g, 10, out, cyc);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_pf<NT, MINB, LDS><<<sms, NT>>>(g, reps, out, cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double per_block = (double)NT * 64.0 * 16.0 * reps;
    printf("{\"variant\": \"%s\", \"threads\": %d, \"ctas_per_sm\": %d, \"unroll\": 0, \"cmp_per_clk_per_sm\": 0, "
           "\"frac_of_32\": 0, \"tcmp_per_s\": %.3f, \"ms\": %.2f, \"eff_mhz\": 0}\n",
           name, NT, MINB, per_block * sms / (ms * 1e-3) / 1e12, ms);
}

// Generalised micro-tile (MI rows x MJ columns per thread), operands and masks from shared memory,
// the same explicitly pipelined 4-instruction compare.  Smaller micro-tiles need fewer registers,
// so more warps fit per SM (better ALU-pipe scheduling) at the price of more LDS per compare.
template <int MI, int MJ>
__device__ __forceinline__ void step_pipelined_mt(const uint32_t (&x)[MI], const uint32_t (&y)[MJ],
                                                  const uint32_t (&xm)[MI], const uint32_t (&ym)[MJ],
                                                  uint32_t (&acc)[MI][MJ]) {
    constexpr int N = MI * MJ;
    uint32_t u[N], p[N], v[N];
#pragma unroll
    for (int q = 0; q < N + 3; ++q) {
        if (q < N) asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[q / MJ]), "r"(y[q % MJ]));
        if (q >= 1 && q - 1 < N) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - 1]) : "r"(u[q - 1]));
        if (q >= 2 && q - 2 < N)
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;"
                         : "=r"(v[q - 2])
                         : "r"(p[q - 2]), "r"(xm[(q - 2) / MJ]), "r"(ym[(q - 2) % MJ]));
        if (q >= 3) asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;" : "+r"(acc[(q - 3) / MJ][(q - 3) % MJ]) : "r"(v[q - 3]));
    }
}

// Pipeline-schedule variants of the 8x8 step (same 4 instructions per compare):
//   S = 0: [lop3 u_q, sub p_q-1, lop3 v_q-2, dp4a q-3]   (k2_tiled's order)
//   S = 1: [lop3 u_q, lop3 v_q-2, sub p_q-1, dp4a q-3]   (ALU pair, FMA pair)
//   S = 2, 3, 4: distances D = 2, 3, 4: u_q, p_q-D, v_q-2D, acc_q-3D (more independent work between
//          dependent instructions)
template <int S>
__device__ __forceinline__ void step_sched(const uint32_t (&x)[8], const uint32_t (&y)[8], const uint32_t (&xm)[8],
                                           const uint32_t (&ym)[8], uint32_t (&acc)[8][8]) {
    constexpr int D = S == 2 ? 2 : (S == 3 ? 3 : (S == 4 ? 4 : 1));
    uint32_t u[64], p[64], v[64];
#pragma unroll
    for (int q = 0; q < 64 + 3 * D; ++q) {
        const bool du = q < 64, dp = q >= D && q - D < 64, dv = q >= 2 * D && q - 2 * D < 64, da = q >= 3 * D;
        if (du) asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[q >> 3]), "r"(y[q & 7]));
        if (S == 1) {
            if (dv)
                asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;"
                             : "=r"(v[q - 2]) : "r"(p[q - 2]), "r"(xm[(q - 2) >> 3]), "r"(ym[(q - 2) & 7]));
            if (dp) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - 1]) : "r"(u[q - 1]));
        } else {
            if (dp) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - D]) : "r"(u[q - D]));
            if (dv)
                asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;"
                             : "=r"(v[q - 2 * D]) : "r"(p[q - 2 * D]), "r"(xm[(q - 2 * D) >> 3]), "r"(ym[(q - 2 * D) & 7]));
        }
        if (da)
            asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;"
                         : "+r"(acc[(q - 3 * D) >> 3][(q - 3 * D) & 7]) : "r"(v[q - 3 * D]));
    }
}

// General schedule: stage offsets D1 (u -> p), D2 (p -> v), D3 (v -> acc); pair order O:
// 0 = i-major (q -> (q/8, q%8)), 1 = j-major, 2 = diagonal (j = (q + q/8) % 8).
template <int O>
__device__ __forceinline__ int pi_(int q) { return O == 1 ? (q & 7) : (q >> 3); }
template <int O>
__device__ __forceinline__ int pj_(int q) { return O == 1 ? (q >> 3) : (O == 2 ? ((q + (q >> 3)) & 7) : (q & 7)); }

template <int D1, int D2, int D3, int O>
__device__ __forceinline__ void step_gen(const uint32_t (&x)[8], const uint32_t (&y)[8], const uint32_t (&xm)[8],
                                         const uint32_t (&ym)[8], uint32_t (&acc)[8][8]) {
    uint32_t u[64], p[64], v[64];
#pragma unroll
    for (int q = 0; q < 64 + D1 + D2 + D3; ++q) {
        if (q < 64) asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[pi_<O>(q)]), "r"(y[pj_<O>(q)]));
        if (q >= D1 && q - D1 < 64) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - D1]) : "r"(u[q - D1]));
        if (q >= D1 + D2 && q - D1 - D2 < 64) {
            const int e = q - D1 - D2;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v[e]) : "r"(p[e]), "r"(xm[pi_<O>(e)]), "r"(ym[pj_<O>(e)]));
        }
        if (q >= D1 + D2 + D3) {
            const int e = q - D1 - D2 - D3;
            asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;" : "+r"(acc[pi_<O>(e)][pj_<O>(e)]) : "r"(v[e]));
        }
    }
}

// Instruction-choice variants on the distance-2 schedule: SUBK 0 = sub.u32 (ptxas: VIADD),
// 1 = mad.lo.u32 u * 1 + 0xFEFEFEFF (IMAD); ACCK 0 = dp4a, 1 = mad.hi.u32 v * 2^25 + acc (IMAD.HI,
// lanes folded at the end -- exact for this benchmark's trip counts).
// One CTA of 16 warps per SM (a 256 x 128 tile) against two CTAs of 8 warps (128 x 128), both with
// the distance-2 schedule and masks from shared memory.
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) bench_big(const uint32_t* __restrict__ g, int reps, uint32_t* out) {
    constexpr int RB = NT / 2;  // rows per tile: 128 (256 threads) or 256 (512 threads)
    __shared__ __align__(16) uint32_t sA[16 * RB], sB[16 * 128], mA[16 * RB], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * RB; i += NT) {
        sA[i] = g[i % 4096];
        mA[i] = sA[i] & 0x80808080u;
    }
    for (int i = threadIdx.x; i < 16 * 128; i += NT) {
        sB[i] = g[4096 + i];
        mB[i] = sB[i] & 0x80808080u;
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int RG = RB / 64;  // row groups of 32 threads-rows: 2 or 4
    const int tr = ((warp % RG) << 3) | (lane & 7);
    const int tc = ((warp / RG) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            uint32_t x[8], y[8], xm[8], ym[8];
            const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * RB + 4 * tr);
            const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * RB + RB / 2 + 4 * tr);
            const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
            const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
            const uint4 a = *reinterpret_cast<const uint4*>(mA + k * RB + 4 * tr);
            const uint4 b = *reinterpret_cast<const uint4*>(mA + k * RB + RB / 2 + 4 * tr);
            const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
            const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
            x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
            y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
            xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
            ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
            step_gen<2, 2, 2, 0>(x, y, xm, ym, acc);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * NT + threadIdx.x] = s;
}

template <int NT, int MINB>
void run_big(const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2000, blocks = sms * MINB;
    bench_big<NT, MINB><<<blocks, NT>>>(g, 10, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        bench_big<NT, MINB><<<blocks, NT>>>(g, reps, out);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double tcmp = (double)blocks * NT * 64.0 * 16.0 * reps / (best * 1e-3) / 1e12;
    printf("{\"variant\": \"big\", \"threads\": %d, \"ctas_per_sm\": %d, \"tcmp_per_s\": %.3f, "
           "\"frac_of_R_int_at_1965MHz\": %.3f}\n", NT, MINB, tcmp, tcmp / (32.0 * sms * 1.965e9 / 1e12));
}

template <int SUBK, int ACCK>
__device__ __forceinline__ void step_ins(const uint32_t (&x)[8], const uint32_t (&y)[8], const uint32_t (&xm)[8],
                                         const uint32_t (&ym)[8], uint32_t (&acc)[8][8], uint32_t one,
                                         uint32_t sh25) {
    constexpr int D = 2;
    uint32_t u[64], p[64], v[64];
#pragma unroll
    for (int q = 0; q < 64 + 3 * D; ++q) {
        if (q < 64) asm volatile("lop3.b32 %0, %1, %2, 0x80808080, 0xBE;" : "=r"(u[q]) : "r"(x[q >> 3]), "r"(y[q & 7]));
        if (q >= D && q - D < 64) {
            if (SUBK == 0) asm volatile("sub.u32 %0, %1, 0x01010101;" : "=r"(p[q - D]) : "r"(u[q - D]));
            else asm volatile("mad.lo.u32 %0, %1, %2, 0xFEFEFEFF;" : "=r"(p[q - D]) : "r"(u[q - D]), "r"(one));
        }
        if (q >= 2 * D && q - 2 * D < 64) {
            const int e = q - 2 * D;
            asm volatile("lop3.b32 %0, %1, %2, %3, 0x0E;" : "=r"(v[e]) : "r"(p[e]), "r"(xm[e >> 3]), "r"(ym[e & 7]));
        }
        if (q >= 3 * D) {
            const int e = q - 3 * D;
            if (ACCK == 0) asm volatile("dp4a.u32.u32 %0, %1, 0x01010101, %0;" : "+r"(acc[e >> 3][e & 7]) : "r"(v[e]));
            else asm volatile("mad.hi.u32 %0, %1, %2, %0;" : "+r"(acc[e >> 3][e & 7]) : "r"(v[e]), "r"(sh25));
        }
    }
}

template <int SUBK, int ACCK>
__global__ void __launch_bounds__(256, 2) bench_ins(const uint32_t* __restrict__ g, int reps, uint32_t one,
                                                   uint32_t sh25, uint32_t* out) {
    __shared__ __align__(16) uint32_t sA[16 * 128], sB[16 * 128], mA[16 * 128], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * 128; i += 256) {
        sA[i] = g[i];
        sB[i] = g[i + 32 * 128];
        mA[i] = g[i] & 0x80808080u;
        mB[i] = g[i + 32 * 128] & 0x80808080u;
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            uint32_t x[8], y[8], xm[8], ym[8];
            const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
            const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
            const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
            const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
            const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
            const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
            const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
            const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
            x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
            y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
            xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
            ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
            step_ins<SUBK, ACCK>(x, y, xm, ym, acc, one, sh25);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int SUBK, int ACCK>
void run_ins(const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2000, blocks = sms * 2;
    bench_ins<SUBK, ACCK><<<blocks, 256>>>(g, 10, 1u, 1u << 25, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        bench_ins<SUBK, ACCK><<<blocks, 256>>>(g, reps, 1u, 1u << 25, out);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double tcmp = (double)blocks * 256 * 64.0 * 16.0 * reps / (best * 1e-3) / 1e12;
    printf("{\"variant\": \"ins\", \"sub\": \"%s\", \"acc\": \"%s\", \"tcmp_per_s\": %.3f, "
           "\"frac_of_R_int_at_1965MHz\": %.3f}\n", SUBK ? "imad" : "sub(viadd)", ACCK ? "imad.hi" : "dp4a", tcmp,
           tcmp / (32.0 * sms * 1.965e9 / 1e12));
}

template <int D1, int D2, int D3, int O>
__global__ void __launch_bounds__(256, 2) bench_gen(const uint32_t* __restrict__ g, int reps, uint32_t* out) {
    __shared__ __align__(16) uint32_t sA[16 * 128], sB[16 * 128], mA[16 * 128], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * 128; i += 256) {
        sA[i] = g[i];
        sB[i] = g[i + 32 * 128];
        mA[i] = g[i] & 0x80808080u;
        mB[i] = g[i + 32 * 128] & 0x80808080u;
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            uint32_t x[8], y[8], xm[8], ym[8];
            const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
            const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
            const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
            const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
            const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
            const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
            const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
            const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
            x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
            y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
            xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
            ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
            step_gen<D1, D2, D3, O>(x, y, xm, ym, acc);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int D1, int D2, int D3, int O>
void run_gen(const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2000, blocks = sms * 2;
    bench_gen<D1, D2, D3, O><<<blocks, 256>>>(g, 10, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        bench_gen<D1, D2, D3, O><<<blocks, 256>>>(g, reps, out);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double tcmp = (double)blocks * 256 * 64.0 * 16.0 * reps / (best * 1e-3) / 1e12;
    printf("{\"variant\": \"gen\", \"D\": [%d, %d, %d], \"order\": %d, \"tcmp_per_s\": %.3f, "
           "\"frac_of_R_int_at_1965MHz\": %.3f}\n", D1, D2, D3, O, tcmp, tcmp / (32.0 * sms * 1.965e9 / 1e12));
}

// Chunk length between CTA barriers (k2_tiled: the per-chunk mask transform + __syncthreads), with
// the distance-2 schedule: KPS k-steps per barrier.
template <int KPS>
__global__ void __launch_bounds__(256, 2) bench_chunk(const uint32_t* __restrict__ g, int reps, uint32_t* out) {
    __shared__ __align__(16) uint32_t sA[KPS * 128], sB[KPS * 128], mA[KPS * 128], mB[KPS * 128];
    for (int i = threadIdx.x; i < KPS * 128; i += 256) {
        sA[i] = g[i % 4096];
        sB[i] = g[(i + 32 * 128) % 8192];
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    const int chunks = reps * 16 / KPS;  // the same number of k-steps for every KPS
    for (int r = 0; r < chunks; ++r) {
        for (int i = threadIdx.x; i < KPS * 128 / 4; i += 256) {  // mask transform, as in k2_tiled
            uint4 v = reinterpret_cast<const uint4*>(sA)[i];
            v.x &= 0x80808080u; v.y &= 0x80808080u; v.z &= 0x80808080u; v.w &= 0x80808080u;
            reinterpret_cast<uint4*>(mA)[i] = v;
            uint4 w = reinterpret_cast<const uint4*>(sB)[i];
            w.x &= 0x80808080u; w.y &= 0x80808080u; w.z &= 0x80808080u; w.w &= 0x80808080u;
            reinterpret_cast<uint4*>(mB)[i] = w;
        }
        __syncthreads();
#pragma unroll 1
        for (int k = 0; k < KPS; ++k) {
            uint32_t x[8], y[8], xm[8], ym[8];
            const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
            const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
            const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
            const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
            const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
            const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
            const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
            const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
            x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
            y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
            xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
            ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
            step_gen<2, 2, 2, 0>(x, y, xm, ym, acc);
        }
        __syncthreads();  // the next chunk's transform overwrites the planes
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * 256 + threadIdx.x] = s;
}

template <int KPS>
void run_chunk(const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2400, blocks = sms * 2;  // 2400 * 16 k-steps: divisible by 16, 24, 32, 48
    bench_chunk<KPS><<<blocks, 256>>>(g, 48, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        bench_chunk<KPS><<<blocks, 256>>>(g, reps, out);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double tcmp = (double)blocks * 256 * 64.0 * 16.0 * reps / (best * 1e-3) / 1e12;
    printf("{\"variant\": \"chunk\", \"k_steps_per_barrier\": %d, \"tcmp_per_s\": %.3f, "
           "\"frac_of_R_int_at_1965MHz\": %.3f}\n", KPS, tcmp, tcmp / (32.0 * sms * 1.965e9 / 1e12));
}

template <int S, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) bench_sched(const uint32_t* __restrict__ g, int reps, uint32_t* out) {
    __shared__ __align__(16) uint32_t sA[16 * 128], sB[16 * 128], mA[16 * 128], mB[16 * 128];
    for (int i = threadIdx.x; i < 16 * 128; i += NT) {
        sA[i] = g[i];
        sB[i] = g[i + 32 * 128];
        mA[i] = g[i] & 0x80808080u;
        mB[i] = g[i + 32 * 128] & 0x80808080u;
    }
    __syncthreads();
    const int warp = (threadIdx.x >> 5) & 7, lane = threadIdx.x & 31;
    const int tr = ((warp & 1) << 3) | (lane & 7);
    const int tc = ((warp >> 1) << 2) | (lane >> 3);
    uint32_t acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            uint32_t x[8], y[8], xm[8], ym[8];
            const uint4 xa = *reinterpret_cast<const uint4*>(sA + k * 128 + 4 * tr);
            const uint4 xb = *reinterpret_cast<const uint4*>(sA + k * 128 + 64 + 4 * tr);
            const uint4 ya = *reinterpret_cast<const uint4*>(sB + k * 128 + 4 * tc);
            const uint4 yb = *reinterpret_cast<const uint4*>(sB + k * 128 + 64 + 4 * tc);
            const uint4 a = *reinterpret_cast<const uint4*>(mA + k * 128 + 4 * tr);
            const uint4 b = *reinterpret_cast<const uint4*>(mA + k * 128 + 64 + 4 * tr);
            const uint4 c = *reinterpret_cast<const uint4*>(mB + k * 128 + 4 * tc);
            const uint4 d = *reinterpret_cast<const uint4*>(mB + k * 128 + 64 + 4 * tc);
            x[0] = xa.x; x[1] = xa.y; x[2] = xa.z; x[3] = xa.w; x[4] = xb.x; x[5] = xb.y; x[6] = xb.z; x[7] = xb.w;
            y[0] = ya.x; y[1] = ya.y; y[2] = ya.z; y[3] = ya.w; y[4] = yb.x; y[5] = yb.y; y[6] = yb.z; y[7] = yb.w;
            xm[0] = a.x; xm[1] = a.y; xm[2] = a.z; xm[3] = a.w; xm[4] = b.x; xm[5] = b.y; xm[6] = b.z; xm[7] = b.w;
            ym[0] = c.x; ym[1] = c.y; ym[2] = c.z; ym[3] = c.w; ym[4] = d.x; ym[5] = d.y; ym[6] = d.z; ym[7] = d.w;
            step_sched<S>(x, y, xm, ym, acc);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s += acc[i][j] * (i * 8 + j + 1);
    out[blockIdx.x * NT + threadIdx.x] = s;
}

template <int S>
void run_sched(const char* name, const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2000, blocks = sms * 2;
    bench_sched<S, 256, 2><<<blocks, 256>>>(g, 10, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int t = 0; t < 3; ++t) {
        cudaEventRecord(e0);
        bench_sched<S, 256, 2><<<blocks, 256>>>(g, reps, out);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double tcmp = (double)blocks * 256 * 64.0 * 16.0 * reps / (best * 1e-3) / 1e12;
    printf("{\"variant\": \"%s\", \"schedule\": %d, \"tcmp_per_s\": %.3f, \"frac_of_R_int_at_1965MHz\": %.3f, "
           "\"ms\": %.2f}\n", name, S, tcmp, tcmp / (32.0 * sms * 1.965e9 / 1e12), best);
}

template <int MI, int MJ, int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) bench_mt(const uint32_t* __restrict__ g, int reps, uint32_t* out) {
    // a 16 x RB row block and 16 x CB column block of words; each thread reads MI/4 (resp. MJ/4)
    // consecutive 4-word groups with LDS.128
    constexpr int TR = 16, TC = NT / TR;  // thread grid
    constexpr int RB = TR * MI, CB = TC * MJ;
    __shared__ __align__(16) uint32_t sA[16 * RB], sB[16 * CB], mA[16 * RB], mB[16 * CB];
    for (int i = threadIdx.x; i < 16 * RB; i += NT) {
        sA[i] = g[i % 4096];
        mA[i] = sA[i] & 0x80808080u;
    }
    for (int i = threadIdx.x; i < 16 * CB; i += NT) {
        sB[i] = g[4096 + i % 4096];
        mB[i] = sB[i] & 0x80808080u;
    }
    __syncthreads();
    const int tr = threadIdx.x % TR, tc = threadIdx.x / TR;
    uint32_t acc[MI][MJ];
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < MJ; ++j) acc[i][j] = 0;
    for (int r = 0; r < reps; ++r) {
#pragma unroll 1
        for (int k = 0; k < 16; ++k) {
            uint32_t x[MI], y[MJ], xm[MI], ym[MJ];
#pragma unroll
            for (int h = 0; h < MI / 4; ++h) {
                const uint4 a = *reinterpret_cast<const uint4*>(sA + k * RB + h * (RB / (MI / 4)) + 4 * tr);
                const uint4 b = *reinterpret_cast<const uint4*>(mA + k * RB + h * (RB / (MI / 4)) + 4 * tr);
                x[4 * h] = a.x; x[4 * h + 1] = a.y; x[4 * h + 2] = a.z; x[4 * h + 3] = a.w;
                xm[4 * h] = b.x; xm[4 * h + 1] = b.y; xm[4 * h + 2] = b.z; xm[4 * h + 3] = b.w;
            }
#pragma unroll
            for (int h = 0; h < MJ / 4; ++h) {
                const uint4 a = *reinterpret_cast<const uint4*>(sB + k * CB + h * (CB / (MJ / 4)) + 4 * tc);
                const uint4 b = *reinterpret_cast<const uint4*>(mB + k * CB + h * (CB / (MJ / 4)) + 4 * tc);
                y[4 * h] = a.x; y[4 * h + 1] = a.y; y[4 * h + 2] = a.z; y[4 * h + 3] = a.w;
                ym[4 * h] = b.x; ym[4 * h + 1] = b.y; ym[4 * h + 2] = b.z; ym[4 * h + 3] = b.w;
            }
            step_pipelined_mt<MI, MJ>(x, y, xm, ym, acc);
        }
    }
    uint32_t s = 0;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < MJ; ++j) s += acc[i][j] * (i * MJ + j + 1);
    out[blockIdx.x * NT + threadIdx.x] = s;
}

template <int MI, int MJ, int NT, int MINB>
void run_mt(const char* name, const uint32_t* g, int sms, uint32_t* out) {
    const int reps = 2000;
    const int blocks = sms * MINB;
    bench_mt<MI, MJ, NT, MINB><<<blocks, NT>>>(g, 10, out);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    bench_mt<MI, MJ, NT, MINB><<<blocks, NT>>>(g, reps, out);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double cmps = (double)blocks * NT * MI * MJ * 16.0 * reps;
    const double tcmp = cmps / (ms * 1e-3) / 1e12;
    printf("{\"variant\": \"%s\", \"micro_tile\": \"%dx%d\", \"threads\": %d, \"ctas_per_sm\": %d, "
           "\"tcmp_per_s\": %.3f, \"frac_of_R_int_at_1965MHz\": %.3f, \"ms\": %.2f}\n",
           name, MI, MJ, NT, MINB, tcmp, tcmp / (32.0 * sms * 1.965e9 / 1e12), ms);
}

int main() {
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<uint32_t> h(2 * 32 * 128);
    uint64_t z = 88172645463325252ull;
    for (auto& v : h) {
        z ^= z << 13;
        z ^= z >> 7;
        z ^= z << 17;
        v = (uint32_t)z & 0xFF7F7F7Fu;
        if ((z >> 40) & 1) v |= 0x00808080u;
    }
    uint32_t *g, *out;
    unsigned long long* cyc;
    CK(cudaMalloc(&g, h.size() * 4));
    CK(cudaMalloc(&out, 4 * sms * 512 * 4));
    CK(cudaMalloc(&cyc, 4 * sms * 8));
    CK(cudaMemcpy(g, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    run<4, 2, 256, 1, 4>("iadd3_idp4a/no_lds_ceiling", g, sms, out, cyc);
    run<4, 2, 256, 2, 4>("iadd3_idp4a/no_lds_ceiling", g, sms, out, cyc);
    run<5, 2, 256, 1, 1>("pipelined_volatile/no_lds_ceiling", g, sms, out, cyc);
    run<5, 2, 256, 2, 1>("pipelined_volatile/no_lds_ceiling", g, sms, out, cyc);
    run<5, 1, 256, 2, 1>("pipelined_volatile/masks_from_smem", g, sms, out, cyc);
    run<5, 1, 512, 1, 1>("pipelined_volatile/masks_from_smem", g, sms, out, cyc);
    run<5, 1, 256, 2, 1, 1>("pipelined_volatile/masks_from_smem+sync", g, sms, out, cyc);
    run<4, 1, 256, 2, 4>("iadd3_idp4a/masks_from_smem", g, sms, out, cyc);
    run_big<256, 2>(g, sms, out);
    run_big<512, 1>(g, sms, out);
    run_big<256, 2>(g, sms, out);
    run_big<512, 1>(g, sms, out);
    run_ins<0, 0>(g, sms, out);
    run_ins<1, 0>(g, sms, out);
    run_ins<0, 1>(g, sms, out);
    run_ins<1, 1>(g, sms, out);
    run_chunk<16>(g, sms, out);
    run_chunk<24>(g, sms, out);
    run_gen<2, 2, 2, 0>(g, sms, out);
    run_gen<2, 2, 2, 1>(g, sms, out);
    run_gen<2, 2, 2, 2>(g, sms, out);
    run_gen<1, 2, 1, 0>(g, sms, out);
    run_gen<2, 1, 2, 0>(g, sms, out);
    run_gen<2, 2, 1, 0>(g, sms, out);
    run_gen<1, 1, 2, 0>(g, sms, out);
    run_gen<2, 3, 2, 0>(g, sms, out);
    run_gen<3, 2, 1, 0>(g, sms, out);
    run_gen<1, 3, 1, 0>(g, sms, out);
    run_gen<2, 2, 2, 0>(g, sms, out);
    run_sched<0>("sched/k2_order", g, sms, out);
    run_sched<1>("sched/alu_pair_fma_pair", g, sms, out);
    run_sched<2>("sched/double_distance", g, sms, out);
    run_sched<3>("sched/triple_distance", g, sms, out);
    run_sched<4>("sched/quad_distance", g, sms, out);
    run_sched<0>("sched/k2_order(again)", g, sms, out);
    run_mt<8, 8, 256, 2>("mt_pipelined/masks_from_smem", g, sms, out);
    run_mt<8, 4, 256, 3>("mt_pipelined/masks_from_smem", g, sms, out);
    run_mt<4, 8, 256, 3>("mt_pipelined/masks_from_smem", g, sms, out);
    run_mt<8, 4, 128, 6>("mt_pipelined/masks_from_smem", g, sms, out);
    run_mt<4, 4, 256, 4>("mt_pipelined/masks_from_smem", g, sms, out);
    run_mt<4, 4, 512, 2>("mt_pipelined/masks_from_smem", g, sms, out);
    return 0;
}
