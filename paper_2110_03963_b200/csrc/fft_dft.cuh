// fft_dft.cuh -- fp64 complex helpers and the register DFT butterflies (radix 2..16) shared by
// the FFT translation units (kernels_fft.cu: shared-memory Stockham engine; kernels_fft_fs.cu:
// fused-stage engine).  Included INSIDE an anonymous namespace of namespace qva, so every
// translation unit gets its own copies (c_roots / s_roots included).
#pragma once

// roots of unity exp(-2 pi i j / r) for r = 2..16, offset r*(r-1)/2 - 1 (kernels copy them to
// shared memory, s_roots)
__constant__ double2 c_roots[160];
__shared__ double2 s_roots[160];
__device__ __forceinline__ void load_roots() {
    for (int i = threadIdx.x; i < 160; i += blockDim.x) s_roots[i] = c_roots[i];
    __syncthreads();
}

__host__ __device__ constexpr int root_off(int r) { return r * (r - 1) / 2 - 1; }

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 conj_if(double2 a, bool inv) { return inv ? make_double2(a.x, -a.y) : a; }
// multiply by -i (forward) or +i (inverse)
__device__ __forceinline__ double2 mul_mi(double2 a, bool inv) {
    return inv ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

// 16-byte global -> shared copies that bypass the registers (LDGSTS): a thread issues all of its
// block's copies back to back, so a whole column / row block is in flight at once and the
// twiddle-table set-up below overlaps it (the register-staged loads kept at most kLoadU per
// thread in flight and waited a memory latency per batch)
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ bool fft_async_loads() {
#ifdef QVA_FFT_SYNC_LOADS
    return false;
#else
    return true;
#endif
}

// cos / sin (2 pi j / N) for the two-level radix-16 and radix-9 butterflies (compile-time
// constants: indices are unrolled, so they fold into immediates)
__host__ __device__ constexpr double tw_cos(int N, int j) {
    constexpr double c7[7] = {1.0, 0.6234898018587336, -0.22252093395631434, -0.900968867902419, -0.9009688679024191, -0.2225209339563146, 0.6234898018587334};
    constexpr double c9[9] = {1.0, 0.766044443118978, 0.17364817766693041, -0.4999999999999998, -0.9396926207859083, -0.9396926207859084, -0.5000000000000004, 0.17364817766692997, 0.7660444431189778};
    constexpr double c11[11] = {1.0, 0.8412535328311812, 0.41541501300188644, -0.142314838273285, -0.654860733945285, -0.9594929736144974, -0.9594929736144975, -0.6548607339452852, -0.14231483827328523, 0.41541501300188605, 0.8412535328311812};
    constexpr double c13[13] = {1.0, 0.8854560256532099, 0.5680647467311559, 0.120536680255323, -0.35460488704253545, -0.7485107481711012, -0.970941817426052, -0.9709418174260521, -0.7485107481711013, -0.3546048870425359, 0.1205366802553232, 0.5680647467311548, 0.88545602565321};
    constexpr double c16[16] = {1.0, 0.9238795325112867, 0.7071067811865476, 0.38268343236508984, 6.123233995736766e-17, -0.3826834323650897, -0.7071067811865475, -0.9238795325112867, -1.0, -0.9238795325112868, -0.7071067811865477, -0.38268343236509034, -1.8369701987210297e-16, 0.38268343236509, 0.7071067811865474, 0.9238795325112865};
    constexpr double c10[10] = {1.0, 0.8090169943749475, 0.30901699437494745, -0.30901699437494745, -0.8090169943749475, -1.0, -0.8090169943749475, -0.30901699437494745, 0.30901699437494745, 0.8090169943749475};
    constexpr double c6[6] = {1.0, 0.5, -0.5, -1.0, -0.5, 0.5};
    constexpr double c15[15] = {1.0, 0.9135454576426009, 0.6691306063588582, 0.30901699437494745, -0.10452846326765347, -0.5, -0.8090169943749475, -0.9781476007338057, -0.9781476007338057, -0.8090169943749475, -0.5, -0.10452846326765347, 0.30901699437494745, 0.6691306063588582, 0.9135454576426009};
    return N == 16 ? c16[j] : N == 15 ? c15[j] : N == 13 ? c13[j] : N == 11 ? c11[j] : N == 10 ? c10[j] : N == 9 ? c9[j] : N == 6 ? c6[j] : c7[j];
}
__host__ __device__ constexpr double tw_sin(int N, int j) {
    constexpr double s7[7] = {0.0, 0.7818314824680298, 0.9749279121818236, 0.43388373911755823, -0.433883739117558, -0.9749279121818236, -0.7818314824680299};
    constexpr double s9[9] = {0.0, 0.6427876096865393, 0.984807753012208, 0.8660254037844387, 0.3420201433256689, -0.34202014332566866, -0.8660254037844384, -0.9848077530122081, -0.6427876096865396};
    constexpr double s11[11] = {0.0, 0.5406408174555976, 0.9096319953545183, 0.9898214418809328, 0.7557495743542583, 0.28173255684142967, -0.2817325568414294, -0.7557495743542582, -0.9898214418809327, -0.9096319953545186, -0.5406408174555974};
    constexpr double s13[13] = {0.0, 0.4647231720437685, 0.8229838658936564, 0.992708874098054, 0.9350162426854148, 0.6631226582407952, 0.23931566428755768, -0.23931566428755743, -0.663122658240795, -0.9350162426854147, -0.992708874098054, -0.822983865893657, -0.4647231720437684};
    constexpr double s16[16] = {0.0, 0.3826834323650898, 0.7071067811865475, 0.9238795325112867, 1.0, 0.9238795325112867, 0.7071067811865476, 0.3826834323650899, 1.2246467991473532e-16, -0.38268343236508967, -0.7071067811865475, -0.9238795325112865, -1.0, -0.9238795325112866, -0.7071067811865477, -0.3826834323650904};
    constexpr double s10[10] = {0.0, 0.5877852522924731, 0.9510565162951535, 0.9510565162951535, 0.5877852522924731, 0.0, -0.5877852522924731, -0.9510565162951535, -0.9510565162951535, -0.5877852522924731};
    constexpr double s6[6] = {0.0, 0.8660254037844386, 0.8660254037844386, 0.0, -0.8660254037844386, -0.8660254037844386};
    constexpr double s15[15] = {0.0, 0.4067366430758002, 0.7431448254773942, 0.9510565162951535, 0.9945218953682733, 0.8660254037844386, 0.5877852522924731, 0.20791169081775934, -0.20791169081775934, -0.5877852522924731, -0.8660254037844386, -0.9945218953682733, -0.9510565162951535, -0.7431448254773942, -0.4067366430758002};
    return N == 16 ? s16[j] : N == 15 ? s15[j] : N == 13 ? s13[j] : N == 11 ? s11[j] : N == 10 ? s10[j] : N == 9 ? s9[j] : N == 6 ? s6[j] : s7[j];
}

template <int R>
__device__ __forceinline__ void dft(double2 (&a)[R], bool inv);

// length P*Q DFT as P-point DFTs over n1 (n = Q n1 + n2), twiddles w_PQ^{n2 k1}, Q-point DFTs over
// n2; output index k = k1 + P k2
template <int P, int Q>
__device__ __forceinline__ void dft_pq(double2 (&a)[P * Q], bool inv) {
    double2 y[Q][P];
#pragma unroll
    for (int n2 = 0; n2 < Q; ++n2) {
        double2 t[P];
#pragma unroll
        for (int n1 = 0; n1 < P; ++n1) t[n1] = a[Q * n1 + n2];
        dft<P>(t, inv);
#pragma unroll
        for (int k1 = 0; k1 < P; ++k1) y[n2][k1] = t[k1];
    }
#pragma unroll
    for (int n2 = 1; n2 < Q; ++n2)
#pragma unroll
        for (int k1 = 1; k1 < P; ++k1) {
            const int j = n2 * k1;
            const double wc = tw_cos(P * Q, j), ws = tw_sin(P * Q, j);
            y[n2][k1] = cmul(y[n2][k1], make_double2(wc, inv ? ws : -ws));
        }
#pragma unroll
    for (int k1 = 0; k1 < P; ++k1) {
        double2 t[Q];
#pragma unroll
        for (int n2 = 0; n2 < Q; ++n2) t[n2] = y[n2][k1];
        dft<Q>(t, inv);
#pragma unroll
        for (int k2 = 0; k2 < Q; ++k2) a[k1 + P * k2] = t[k2];
    }
}

template <int R>
__device__ __forceinline__ void dft(double2 (&a)[R], bool inv) {
    if constexpr (R == 2) {
        double2 t = a[0];
        a[0] = cadd(t, a[1]);
        a[1] = csub(t, a[1]);
    } else if constexpr (R == 4) {
        double2 s02 = cadd(a[0], a[2]), d02 = csub(a[0], a[2]);
        double2 s13 = cadd(a[1], a[3]), d13 = csub(a[1], a[3]);
        double2 wd = mul_mi(d13, inv);
        a[0] = cadd(s02, s13);
        a[2] = csub(s02, s13);
        a[1] = cadd(d02, wd);
        a[3] = csub(d02, wd);
    } else if constexpr (R == 3) {
        // X1,2 = a0 - (a1+a2)/2 -/+ i (sqrt3/2)(a1 - a2)   (signs flip for the inverse)
        const double h = 0.86602540378443864676;
        double2 t1 = cadd(a[1], a[2]);
        double2 t2 = make_double2(fma(-0.5, t1.x, a[0].x), fma(-0.5, t1.y, a[0].y));
        double2 d = csub(a[1], a[2]);
        double2 t3 = mul_mi(make_double2(h * d.x, h * d.y), inv);
        a[0] = cadd(a[0], t1);
        a[1] = cadd(t2, t3);
        a[2] = csub(t2, t3);
    } else if constexpr (R == 5) {
        const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
        const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
        double2 t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
        double2 t3 = csub(a[1], a[4]), t4 = csub(a[2], a[3]);
        double2 b1 = make_double2(fma(c1, t1.x, fma(c2, t2.x, a[0].x)), fma(c1, t1.y, fma(c2, t2.y, a[0].y)));
        double2 b2 = make_double2(fma(c2, t1.x, fma(c1, t2.x, a[0].x)), fma(c2, t1.y, fma(c1, t2.y, a[0].y)));
        double2 d1 = mul_mi(make_double2(fma(s1, t3.x, s2 * t4.x), fma(s1, t3.y, s2 * t4.y)), inv);
        double2 d2 = mul_mi(make_double2(fma(s2, t3.x, -s1 * t4.x), fma(s2, t3.y, -s1 * t4.y)), inv);
        a[0] = cadd(a[0], cadd(t1, t2));
        a[1] = cadd(b1, d1);
        a[4] = csub(b1, d1);
        a[2] = cadd(b2, d2);
        a[3] = csub(b2, d2);
    } else if constexpr (R == 7 || R == 11 || R == 13) {
        // odd prime: pairs (u, R-u) give y_t = a0 + sum_u c_tu (a_u + a_{R-u}) -/+ i sum_u s_tu
        // (a_u - a_{R-u}) for (t, R-t): (R-1) real-coefficient FMAs per output instead of 2(R-1)
        constexpr int H = (R - 1) / 2;
        double2 sp[H], sm[H];
#pragma unroll
        for (int u = 1; u <= H; ++u) {
            sp[u - 1] = cadd(a[u], a[R - u]);
            sm[u - 1] = csub(a[u], a[R - u]);
        }
        double2 y0 = a[0];
#pragma unroll
        for (int u = 0; u < H; ++u) y0 = cadd(y0, sp[u]);
#pragma unroll
        for (int t = 1; t <= H; ++t) {
            double2 re = a[0], im = make_double2(0.0, 0.0);
#pragma unroll
            for (int u = 1; u <= H; ++u) {
                const double c = tw_cos(R, (t * u) % R), sn = tw_sin(R, (t * u) % R);
                re = make_double2(fma(c, sp[u - 1].x, re.x), fma(c, sp[u - 1].y, re.y));
                im = make_double2(fma(sn, sm[u - 1].x, im.x), fma(sn, sm[u - 1].y, im.y));
            }
            const double2 mi = mul_mi(im, inv);  // -i im (forward), +i im (inverse)
            a[t] = cadd(re, mi);
            a[R - t] = csub(re, mi);
        }
        a[0] = y0;
    } else if constexpr (R == 16) {
        dft_pq<4, 4>(a, inv);
    } else if constexpr (R == 9) {
        dft_pq<3, 3>(a, inv);
    } else if constexpr (R == 10) {
        dft_pq<2, 5>(a, inv);
    } else if constexpr (R == 6) {
        dft_pq<2, 3>(a, inv);
    } else if constexpr (R == 15) {
        dft_pq<3, 5>(a, inv);
    } else if constexpr (R == 8) {
        // radix-2 split into two length-4 DFTs: X_k = E_k + w8^k O_k, X_{k+4} = E_k - w8^k O_k
        double2 e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
        dft<4>(e, inv);
        dft<4>(o, inv);
        const double h = 0.70710678118654752440;
        double2 w1 = inv ? make_double2(h, h) : make_double2(h, -h);
        double2 w3 = inv ? make_double2(-h, h) : make_double2(-h, -h);
        double2 t0 = o[0], t1 = cmul(o[1], w1), t2 = mul_mi(o[2], inv), t3 = cmul(o[3], w3);
        a[0] = cadd(e[0], t0);
        a[4] = csub(e[0], t0);
        a[1] = cadd(e[1], t1);
        a[5] = csub(e[1], t1);
        a[2] = cadd(e[2], t2);
        a[6] = csub(e[2], t2);
        a[3] = cadd(e[3], t3);
        a[7] = csub(e[3], t3);
    } else {
        double2 y[R];
#pragma unroll
        for (int t = 0; t < R; ++t) {
            double2 acc = a[0];
#pragma unroll
            for (int u = 1; u < R; ++u) {
                double2 w = conj_if(s_roots[root_off(R) + (t * u) % R], inv);
                acc = cadd(acc, cmul(a[u], w));
            }
            y[t] = acc;
        }
#pragma unroll
        for (int t = 0; t < R; ++t) a[t] = y[t];
    }
}
