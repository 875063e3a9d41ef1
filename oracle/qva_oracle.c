/*
 * qva_oracle.c -- plain, slow, obviously-correct CPU oracle for the QVA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant generator with the CUDA path (paper_2110_03963_b200/csrc).
 *
 * What it computes (arXiv 2110.03963, "QuOp_MPI", /root/reference/PAPER.md):
 *   |psi> = prod_{k=1..p} U_M(beta_k) U_Q(gamma_k) |psi0>,   f = <psi|Q|psi>
 *   Eq. 1/2, QAOA Eq. qaoa, QWOA Eq. qwoa.
 * Readings of garbled/ambiguous passages are listed in DESIGN.md ("Readings"), R1..R22.
 *
 * Arithmetic: IEEE fp64, round-to-nearest, no -ffast-math.  State vectors are
 * interleaved (re, im) double pairs, index x = sum_j bit_j(x) 2^j, vertex/qubit j <-> bit j
 * (R8).  OpenMP (if enabled) only splits loops over independent
 * elements/pairs; every reduction is sequential in index order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_API __attribute__((visibility("default")))

OR_API int or_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
/* thread count of the OpenMP loops (timing only: SURVEY 8(d) reports 1 thread and all cores) */
OR_API void or_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* Max-cut qualities.  PAPER.md:721-726 (Eq. maxcut-cost) counts UNCUT edges,
 * C = sum_E 1/2 (1 + Z_i Z_j); the configs (BASELINE.json) fix q_x = -cut_w(x)
 * (R10).  cut_w(x) = sum over edges (u,v) of w_uv [bit_u(x) != bit_v(x)].
 * w == NULL means unit weights. */
OR_API void or_maxcut_q(int n, int m, const int32_t *u, const int32_t *v,
                        const double *w, double *q) {
    uint64_t N = (uint64_t)1 << n;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)N; ++x) {
        double cut = 0.0;
        for (int e = 0; e < m; ++e) {
            int bu = (int)((x >> u[e]) & 1);
            int bv = (int)((x >> v[e]) & 1);
            if (bu != bv) cut += (w ? w[e] : 1.0);
        }
        q[x] = -cut;
    }
}

/* Initial state |+> = N^{-1/2} sum_x |x> (PAPER.md:174-178 Eq. qaoa_initial_state, with the
 * garbled 1/sqrt(n) read as 1/sqrt(N), R2); QWOA uniform over S'. */
OR_API void or_init_uniform(uint64_t N, double *psi) {
    double a = 1.0 / sqrt((double)N);
    for (uint64_t x = 0; x < N; ++x) {
        psi[2 * x] = a;
        psi[2 * x + 1] = 0.0;
    }
}

/* Phase shift U_Q(gamma) = exp(-i gamma Q) (PAPER.md:152-155 Eq. phase_shift_qaoa;
 * diagonal action PAPER.md:307-313):  psi_x <- (cos(gamma q_x) - i sin(gamma q_x)) psi_x,
 * the angle being fl(gamma * q_x). */
OR_API void or_phase(uint64_t N, double *psi, const double *q, double gamma) {
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)N; ++x) {
        double ang = gamma * q[x];
        double c = cos(ang), s = sin(ang);
        double re = psi[2 * x], im = psi[2 * x + 1];
        /* (c - i s)(re + i im) = (c re + s im) + i (c im - s re) */
        psi[2 * x] = c * re + s * im;
        psi[2 * x + 1] = c * im - s * re;
    }
}

/* Transverse-field mixer U_M(beta) = exp(-i beta sum_j X_j) = prod_j exp(-i beta X_j)
 * (PAPER.md:159-171 Eq. mixing_qaoa + Fig. hypercube, read as sum_j X_j, R1).
 * exp(-i beta X) = cos(beta) I - i sin(beta) X, so for every qubit j and every pair
 * (x, x|2^j) with bit j of x clear:  a' = c a - i s b,  b' = -i s a + c b. */
OR_API void or_mixer_x(int n, double *psi, double beta) {
    uint64_t N = (uint64_t)1 << n;
    double c = cos(beta), s = sin(beta);
    for (int j = 0; j < n; ++j) {
        uint64_t bit = (uint64_t)1 << j;
#pragma omp parallel for schedule(static)
        for (int64_t x = 0; x < (int64_t)N; ++x) {
            if ((uint64_t)x & bit) continue;
            uint64_t y = (uint64_t)x | bit;
            double ar = psi[2 * x], ai = psi[2 * x + 1];
            double br = psi[2 * y], bi = psi[2 * y + 1];
            /* -i s b = s bi - i s br */
            psi[2 * x] = c * ar + s * bi;
            psi[2 * x + 1] = c * ai - s * br;
            psi[2 * y] = c * br + s * ai;
            psi[2 * y + 1] = c * bi - s * ar;
        }
    }
}

/* QAOAz parity mixer (Eqs. parity_terms / qaoaz_mixers; R19):
 *   U_parity(t) = exp(-i t B_last) exp(-i t B_even) exp(-i t B_odd)
 * over the ordered qubit subsequence s[0..K): B_odd pairs (s0,s1), (s2,s3), ...; B_even pairs
 * (s1,s2), (s3,s4), ... (no wrap); B_last = the wrap pair (s_{K-1}, s0) iff K is odd (K >= 3).
 * Pairs inside one B act on disjoint qubits, so exp(-i t B) is the product of the pair
 * exponentials.  X_aX_b + Y_aY_b maps |01> <-> |10> with weight 2 and kills |00>, |11>, so
 * exp(-i t (XX+YY)) on the pair (a, b): for x with bit a = 1, bit b = 0 and y = x with the two
 * bits swapped:  u' = cos(2t) u - i sin(2t) v,  v' = -i sin(2t) u + cos(2t) v  (u = psi_x, v = psi_y). */
static void or_pair_xy(int n, double *psi, int a, int b, double t) {
    uint64_t N = (uint64_t)1 << n, ba = (uint64_t)1 << a, bb = (uint64_t)1 << b;
    double c = cos(2.0 * t), s = sin(2.0 * t);
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)N; ++x) {
        if (!((uint64_t)x & ba) || ((uint64_t)x & bb)) continue;
        uint64_t y = ((uint64_t)x ^ ba) | bb;
        double ur = psi[2 * x], ui = psi[2 * x + 1];
        double vr = psi[2 * y], vi = psi[2 * y + 1];
        psi[2 * x] = c * ur + s * vi;
        psi[2 * x + 1] = c * ui - s * vr;
        psi[2 * y] = c * vr + s * ui;
        psi[2 * y + 1] = c * vi - s * ur;
    }
}

OR_API void or_mixer_parity(int n, double *psi, const int *sq, int K, double t) {
    for (int m = 0; m + 1 < K; m += 2) or_pair_xy(n, psi, sq[m], sq[m + 1], t);      /* B_odd  */
    for (int m = 1; m + 1 < K; m += 2) or_pair_xy(n, psi, sq[m], sq[m + 1], t);      /* B_even */
    if (K >= 3 && (K & 1)) or_pair_xy(n, psi, sq[K - 1], sq[0], t);                  /* B_last */
}

/* QAOAz evolution (PAPER.md Eq. qaoaz): for k = 1..p: phase(gamma_k) then U_parity(t_k). */
OR_API void or_evolve_parity(int n, double *psi, const double *q, const int *sq, int K, const double *theta,
                             int p) {
    uint64_t N = (uint64_t)1 << n;
    for (int k = 0; k < p; ++k) {
        or_phase(N, psi, q, theta[2 * k]);
        or_mixer_parity(n, psi, sq, K, theta[2 * k + 1]);
    }
}

/* Circulant mixer, definition written out (Sec. 3, sign read as
 * exp(-i beta lambda_j), R3; lambda indexed by forward-DFT bin j, R4):
 *   U = F^{-1} diag(exp(-i beta lambda)) F,  F_{jx} = exp(-2 pi i j x / N), F^{-1} = F^H / N.
 * U is circulant: U_{xy} = c[(x - y) mod N] with
 *   c[d] = (1/N) sum_j exp(-i beta lambda_j) exp(+2 pi i j d / N).
 * O(N^2); the DFT angle uses the exact integer residue (j*d mod N). */
OR_API void or_mixer_circulant_dense(uint64_t N, double *psi, const double *lambda, double beta) {
    double *cre = (double *)malloc(sizeof(double) * N);
    double *cim = (double *)malloc(sizeof(double) * N);
    double *out = (double *)malloc(sizeof(double) * 2 * N);
    const double two_pi = 6.283185307179586476925286766559;
#pragma omp parallel for schedule(static)
    for (int64_t d = 0; d < (int64_t)N; ++d) {
        double sr = 0.0, si = 0.0;
        for (uint64_t j = 0; j < N; ++j) {
            double el = -beta * lambda[j];
            double er = cos(el), ei = sin(el);
            uint64_t r = (uint64_t)(((unsigned __int128)j * (uint64_t)d) % N);
            double ang = two_pi * (double)r / (double)N;
            double wr = cos(ang), wi = sin(ang);
            sr += er * wr - ei * wi;
            si += er * wi + ei * wr;
        }
        cre[d] = sr / (double)N;
        cim[d] = si / (double)N;
    }
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)N; ++x) {
        double sr = 0.0, si = 0.0;
        for (uint64_t y = 0; y < N; ++y) {
            uint64_t d = ((uint64_t)x + N - y) % N;
            double ur = cre[d], ui = cim[d];
            double pr = psi[2 * y], pi = psi[2 * y + 1];
            sr += ur * pr - ui * pi;
            si += ur * pi + ui * pr;
        }
        out[2 * x] = sr;
        out[2 * x + 1] = si;
    }
    memcpy(psi, out, sizeof(double) * 2 * N);
    free(cre);
    free(cim);
    free(out);
}

/* Circulant mixer for the spectrum lambda = (lam0, c, c, ..., c) -- the complete-graph
 * family (cfg3 uses the K_N Laplacian lam0 = 0, c = N, R5).
 * The j = 0 Fourier mode is the uniform vector, so with P0 = (1/N) 1 1^T:
 *   U = exp(-i beta c) (I - P0) + exp(-i beta lam0) P0
 *   psi' = exp(-i beta c) psi + (exp(-i beta lam0) - exp(-i beta c)) mean(psi) 1.
 * Exact closed form, O(N); mean(psi) is summed sequentially in long double. */
OR_API void or_mixer_complete(uint64_t N, double *psi, double beta, double lam0, double c) {
    long double mr = 0.0L, mi = 0.0L;
    for (uint64_t x = 0; x < N; ++x) {
        mr += (long double)psi[2 * x];
        mi += (long double)psi[2 * x + 1];
    }
    double meanr = (double)(mr / (long double)N), meani = (double)(mi / (long double)N);
    double ecr = cos(-beta * c), eci = sin(-beta * c);
    double e0r = cos(-beta * lam0), e0i = sin(-beta * lam0);
    double dr = e0r - ecr, di = e0i - eci;
    double kr = dr * meanr - di * meani, ki = dr * meani + di * meanr;
#pragma omp parallel for schedule(static)
    for (int64_t x = 0; x < (int64_t)N; ++x) {
        double pr = psi[2 * x], pi = psi[2 * x + 1];
        psi[2 * x] = ecr * pr - eci * pi + kr;
        psi[2 * x + 1] = ecr * pi + eci * pr + ki;
    }
}

/* Objective f = <psi|Q|psi> = sum_x |psi_x|^2 q_x (Eq. 2).  Sequential
 * index-order Neumaier sum in long double. */
OR_API double or_expectation(uint64_t N, const double *psi, const double *q) {
    long double s = 0.0L, comp = 0.0L;
    for (uint64_t x = 0; x < N; ++x) {
        long double re = psi[2 * x], im = psi[2 * x + 1];
        long double t = (re * re + im * im) * (long double)q[x];
        long double y = s + t;
        if (fabsl(s) >= fabsl(t)) comp += (s - y) + t; else comp += (t - y) + s;
        s = y;
    }
    return (double)(s + comp);
}

/* sum_x |psi_x|^2 (norm squared; PAPER.md:1086-1088/1103 report its deviation from 1). */
OR_API double or_norm2(uint64_t N, const double *psi) {
    long double s = 0.0L;
    for (uint64_t x = 0; x < N; ++x) {
        long double re = psi[2 * x], im = psi[2 * x + 1];
        s += re * re + im * im;
    }
    return (double)s;
}

/* Probabilities p_x = |psi_x|^2 (Table 3 get_probabilities). */
OR_API void or_probabilities(uint64_t N, const double *psi, double *prob) {
    for (uint64_t x = 0; x < N; ++x)
        prob[x] = psi[2 * x] * psi[2 * x] + psi[2 * x + 1] * psi[2 * x + 1];
}

/* Full QAOA evolution (PAPER.md:185 Eq. qaoa): psi starts as given (caller initialises,
 * normally with or_init_uniform), then for k = 1..p: phase(gamma_k) then mixer(beta_k);
 * theta = [g1, b1, g2, b2, ...] (R7); layer 1 acts first (R6). */
OR_API void or_evolve_x(int n, double *psi, const double *q, const double *theta, int p) {
    uint64_t N = (uint64_t)1 << n;
    for (int k = 0; k < p; ++k) {
        or_phase(N, psi, q, theta[2 * k]);
        or_mixer_x(n, psi, theta[2 * k + 1]);
    }
}

/* QWOA evolution (PAPER.md:298 Eq. qwoa) with the complete-graph-family spectrum.
 * U_# is the identity in subspace simulation (R20). */
OR_API void or_evolve_complete(uint64_t N, double *psi, const double *q, const double *theta,
                               int p, double lam0, double c) {
    for (int k = 0; k < p; ++k) {
        or_phase(N, psi, q, theta[2 * k]);
        or_mixer_complete(N, psi, theta[2 * k + 1], lam0, c);
    }
}

/* QWOA evolution with an arbitrary spectrum via the O(N^2) circulant definition. */
OR_API void or_evolve_circulant_dense(uint64_t N, double *psi, const double *q, const double *lambda,
                                      const double *theta, int p) {
    for (int k = 0; k < p; ++k) {
        or_phase(N, psi, q, theta[2 * k]);
        or_mixer_circulant_dense(N, psi, lambda, theta[2 * k + 1]);
    }
}

/* Light-cone max-cut expectation (exact reduction).
 * <Q> = sum_e (w_e/2) (<Z_u Z_v> - 1) for q = -cut_w.  In the Heisenberg picture the
 * p-layer QAOA conjugate of Z_u Z_v acts only on vertices within graph distance p of
 * {u, v}; edges with both ends at distance exactly p commute with it.  So <Z_u Z_v> is
 * obtained by simulating QAOA (the same or_evolve_x) on the induced subgraph of that
 * ball, starting from |+>.  Each subgraph simulation is an ordinary full-state oracle run.
 * Returns NAN if a ball exceeds max_qubits.  cone_sizes (optional, length m) receives the
 * number of qubits of each edge's ball. */
OR_API double or_lightcone_maxcut(int n, int m, const int32_t *u, const int32_t *v,
                                  const double *w, const double *theta, int p,
                                  int max_qubits, int32_t *cone_sizes) {
    int *dist = (int *)malloc(sizeof(int) * n);
    int *queue = (int *)malloc(sizeof(int) * n);
    int *local = (int *)malloc(sizeof(int) * n);
    int32_t *su = (int32_t *)malloc(sizeof(int32_t) * (m > 0 ? m : 1));
    int32_t *sv = (int32_t *)malloc(sizeof(int32_t) * (m > 0 ? m : 1));
    double *sw = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    long double total = 0.0L;
    int ok = 1;
    for (int e = 0; e < m && ok; ++e) {
        /* BFS from {u_e, v_e} up to distance p */
        for (int i = 0; i < n; ++i) dist[i] = -1;
        int head = 0, tail = 0;
        dist[u[e]] = 0; queue[tail++] = u[e];
        if (dist[v[e]] < 0) { dist[v[e]] = 0; queue[tail++] = v[e]; }
        while (head < tail) {
            int a = queue[head++];
            if (dist[a] >= p) continue;
            for (int f = 0; f < m; ++f) {
                int b = -1;
                if (u[f] == a) b = v[f]; else if (v[f] == a) b = u[f];
                if (b >= 0 && dist[b] < 0) { dist[b] = dist[a] + 1; queue[tail++] = b; }
            }
        }
        int k = 0;
        for (int i = 0; i < n; ++i) local[i] = (dist[i] >= 0) ? k++ : -1;
        if (cone_sizes) cone_sizes[e] = k;
        if (k > max_qubits) { ok = 0; break; }
        int ms = 0;
        for (int f = 0; f < m; ++f) {
            if (local[u[f]] >= 0 && local[v[f]] >= 0) {
                su[ms] = local[u[f]]; sv[ms] = local[v[f]]; sw[ms] = w ? w[f] : 1.0; ++ms;
            }
        }
        uint64_t NS = (uint64_t)1 << k;
        double *psi = (double *)malloc(sizeof(double) * 2 * NS);
        double *q = (double *)malloc(sizeof(double) * NS);
        or_maxcut_q(k, ms, su, sv, sw, q);
        or_init_uniform(NS, psi);
        or_evolve_x(k, psi, q, theta, p);
        int la = local[u[e]], lb = local[v[e]];
        long double zz = 0.0L;
        for (uint64_t x = 0; x < NS; ++x) {
            long double pr = (long double)psi[2 * x] * psi[2 * x] + (long double)psi[2 * x + 1] * psi[2 * x + 1];
            int par = (int)(((x >> la) ^ (x >> lb)) & 1);
            zz += par ? -pr : pr;
        }
        total += (long double)(w ? w[e] : 1.0) * 0.5L * (zz - 1.0L);
        free(psi);
        free(q);
    }
    free(dist); free(queue); free(local); free(su); free(sv); free(sw);
    return ok ? (double)total : NAN;
}
