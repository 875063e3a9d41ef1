// kernels_tile.cu -- the X-mixer tile pass: one HBM round trip over the state that applies, to
// every tile of 2^12 amplitudes, any subset of the single-qubit rotations exp(-i beta X_j)
// whose qubits are tile bits (Eq. mixing_qaoa, reading R1), optionally the
// phase exp(-i gamma q_x) between two rotation sets (Eq. phase_shift_qaoa, PAPER.md:152-155;
// diagonal action, Sec. 3) and optionally the partial sums of
// <psi|Q|psi> = sum |psi_x|^2 q_x and of the norm (Eq. 2).
//
// sm_100a design:
//  * persistent grid, one CTA per SM, 256 threads = two consumer warpgroups that take alternate
//    tiles; there is no producer warp: the warpgroup that frees a stage refills it (one elected
//    thread claims the next tile from a per-pass atomic counter and issues its TMA load);
//  * a STAGES-deep ring of 64 KiB shared-memory tiles filled by cp.async.bulk.tensor (one 5-D
//    box per tile: the tile bits are box dimensions, the other index bits are coordinates, so
//    strided high-qubit tiles cost one instruction) with SWIZZLE_128B, completion on mbarriers;
//  * the qualities (fp64 or compact integer codes, or per-tile records of generated max-cut q)
//    arrive in the same stage by a 1-D bulk copy from a copy pre-permuted into consumer order
//    (conflict-free 16-byte smem reads);
//  * each consumer thread holds 32 amplitudes; rotations (and the QAOAz pair terms) run on
//    register groups of 5 tile bits; a group change is one in-place swizzled smem transpose
//    (conflict-free LDS.128/STS.128);
//  * the finished tile is written back to its stage in the load layout and leaves with one TMA
//    tensor store (cp.async.bulk.tensor ... bulk_group), or, for the fused multi-GPU exchange,
//    with register stores into the peers' IPC-mapped buffers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>
#include <utility>

#include "qva_internal.h"

namespace qva {

namespace {

constexpr int kTile = 1 << kTileBits;      // 4096 amplitudes
constexpr int kWG = 2;                      // consumer warpgroups (alternate tiles)
constexpr int kCT = 128;                    // consumer threads per warpgroup
constexpr int kCW = kWG * kCT / 32;         // consumer warps per CTA
constexpr int kAPT = kTile / kCT;           // 32 amplitudes per consumer thread
constexpr int kThreads = kWG * kCT;         // no producer warp: each warpgroup refills what it frees
constexpr int kTabRep = 8;                  // smem phase-table replicas (one per 16-B bank group)
constexpr int kTabSmemMax = 64;             // entries held in smem (int8 codes, batch == 1)
constexpr int kGfMembers = 24;              // weighted generated q: factorised phase for batches <= 24

static_assert(kAPT == 1 << kGroupBits, "group width");
static_assert(kCT == 1 << kCT_BITS, "warpgroup width");

template <typename F, int... K>
__device__ __forceinline__ void static_for_impl(F &f, std::integer_sequence<int, K...>) {
    (f(std::integral_constant<int, K>()), ...);
}
template <int N, typename F>
__device__ __forceinline__ void static_for(F &&f) {
    static_for_impl(f, std::make_integer_sequence<int, N>());
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap *map, uint32_t bar, const int (&c)[5]) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap *map, uint32_t src, const int (&c)[5]) {
    asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]), "r"(c[4]), "r"(src)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void wg_sync(int wg) { asm volatile("bar.sync %0, %1;" ::"r"(1 + wg), "n"(kCT) : "memory"); }

// Rotation exp(-i beta X) on the pair (a, b) (a: bit clear, b: bit set) in factored form:
// a' = a - i t b, b' = b - i t a with t = tan beta (4 DFMA); the dropped scalar cos beta is applied
// once per pass (PassAngles::scale).  Intermediates of k factored rotations are bounded by
// (|cos|+|sin|)^k <= 2^(k/2) times the final magnitude, so the factoring costs at most ~k/2
// bits of relative accuracy.  t = 0 is an exact identity, which is how a register bit that is
// not rotated in a step is skipped without a branch.  |cos beta| < 2^-10 is handled on the
// host by applying two half-angle steps.
__device__ __forceinline__ void fbutterfly(double2 &a, double2 &b, double t) {
    const double ar = a.x, ai = a.y, br = b.x, bi = b.y;
    a = make_double2(fma(t, bi, ar), fma(-t, br, ai));
    b = make_double2(fma(t, ai, br), fma(-t, ar, bi));
}

template <int J>
__device__ __forceinline__ void rot_bit(double2 (&v)[kAPT], double t) {
#pragma unroll
    for (int e = 0; e < kAPT; ++e)
        if (!(e & (1 << J))) fbutterfly(v[e], v[e | (1 << J)], t);
}

// register bits a group can rotate: X all 5, Y its first 4 (its 5th bit, tile bit 3, belongs to
// X), W its first 3 (tile bits 0..2)
template <int G>
__device__ __forceinline__ void rotate_group(double2 (&v)[kAPT], int mask, double t) {
    rot_bit<0>(v, (mask & 1) ? t : 0.0);
    rot_bit<1>(v, (mask & 2) ? t : 0.0);
    rot_bit<2>(v, (mask & 4) ? t : 0.0);
    if (G != 2) rot_bit<3>(v, (mask & 8) ? t : 0.0);
    if (G == 0) rot_bit<4>(v, (mask & 16) ? t : 0.0);
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// Shared-memory address of register element e of consumer thread c in register group G (the
// compile-time twin of api.cu kGroups) under SWIZZLE_128B (16-byte slot = i ^ ((i >> 3) & 7)):
//   X: ebit {3,4,5,6,7}   tbit {0,1,2,8,9,10,11}  slot = (l ^ e[0:3]) | e << 3 | h << 8
//   Y: ebit {8,9,10,11,3} tbit {0,1,2,4,5,6,7}    slot = (l ^ (e4 | h[0:2] << 1)) | e4 << 3 | h << 4 | e[0:4] << 8
//   W: ebit {0,1,2,6,7}   tbit {3,4,5,8,9,10,11}  slot = (e[0:3] ^ l) | l << 3 | e[3:5] << 6 | h << 8
// (l = c & 7, h = c >> 3).  In bytes every address is (A ^ x(e)) + k(e) with a per-thread base A,
// x(e) < 128 and k(e) a multiple of 128, so each access is one LOP3 + LDS/STS with an immediate.
// A is laundered through a register move per item so ptxas cannot hoist the 8 XOR variants of
// every stage out of the loop (they would not fit the register budget).
// Groups 3 (V) and 4 (Z), added for the QAOAz parity pair terms, use the general form of the same
// addressing: with T(c) / E(e) the tile indices of the thread bits / register bits (disjoint),
// the swizzled 16-B slot is linear over GF(2): slot(T | E) = slot(T) ^ slot(E), slot(i) = i ^ ((i >> 3)
// & 7), so addr = (A ^ x(e)) + k(e) with A = buf + 16 slot(T(c)), x(e) = 16 slot(E(e)) mod 1024 and
// k(e) = the rest (bits >= 10 of A and of 16 slot(E(e)) are disjoint, and buf is 1024-B aligned).
//   V: ebit {6,7,8,9,10}  tbit {0,1,2,3,4,5,11}
//   Z: ebit {1,2,3,10,11} tbit {0,4,5,6,7,8,9}
// (the first three thread bits of each group hit distinct bank-group bits, i0^i3, i1^i4, i2^i5).
__host__ __device__ constexpr int dev_ebit(int G, int j) {
    constexpr int V[5] = {6, 7, 8, 9, 10}, Z[5] = {1, 2, 3, 10, 11};
    return G == 3 ? V[j] : Z[j];
}
__host__ __device__ constexpr int dev_tbit(int G, int j) {
    constexpr int V[7] = {0, 1, 2, 3, 4, 5, 11}, Z[7] = {0, 4, 5, 6, 7, 8, 9};
    return G == 3 ? V[j] : Z[j];
}
__host__ __device__ constexpr uint32_t swz_slot(uint32_t i) { return i ^ ((i >> 3) & 7); }
template <int G>
__device__ __forceinline__ constexpr uint32_t gen_e_index(int e) {
    uint32_t i = 0;
    for (int j = 0; j < kGroupBits; ++j)
        if ((e >> j) & 1) i |= 1u << dev_ebit(G, j);
    return i;
}
template <int G>
__device__ __forceinline__ uint32_t group_base(uint32_t buf, int c) {
    const uint32_t l = c & 7, h = c >> 3;
    uint32_t a;
    if (G == 0) a = buf + (l << 4) + (h << 12);
    else if (G == 1) a = buf + ((l ^ ((h & 3) << 1)) << 4) + (h << 8);
    else if (G == 2) a = buf + (l << 4) + (l << 7) + (h << 12);
    else {
        uint32_t T = 0;
#pragma unroll
        for (int j = 0; j < kCT_BITS; ++j) T |= (uint32_t)((c >> j) & 1) << dev_tbit(G, j);
        a = buf + (swz_slot(T) << 4);
    }
    asm volatile("mov.b32 %0, %0;" : "+r"(a));
    return a;
}
template <int G>
__device__ __forceinline__ uint32_t group_addr(uint32_t A, int e) {
    if (G == 0) return (A ^ ((e & 7) << 4)) + (e << 7);
    if (G == 1) return (A ^ ((e >> 4) << 4)) + ((e >> 4) << 7) + ((e & 15) << 12);
    if (G == 2) return (A ^ ((e & 7) << 4)) + ((e >> 3) << 10);
    const uint32_t k = swz_slot(gen_e_index<G>(e)) << 4;
    return (A ^ (k & 1023u)) + (k & ~1023u);
}

// QAOAz pair term exp(-i t (X_a X_b + Y_a Y_b)) on register bits (JA, JB): the Givens rotation by
// 2t on the {01, 10} pairs (R19), u' = c u - i s v, v' = c v - i s u with c = cos 2t, s = sin 2t;
// the {00, 11} elements are unchanged.  Same arithmetic as the oracle's or_pair_xy.
template <int JA, int JB>
__device__ __forceinline__ void givens_pair(double2 (&v)[kAPT], double c, double s) {
#pragma unroll
    for (int e = 0; e < kAPT; ++e)
        if (((e >> JA) & 1) && !((e >> JB) & 1)) {
            const int f = e ^ (1 << JA) ^ (1 << JB);
            const double2 u = v[e], w = v[f];
            v[e] = make_double2(fma(c, u.x, s * w.y), fma(c, u.y, -s * w.x));
            v[f] = make_double2(fma(c, w.x, s * u.y), fma(c, w.y, -s * u.x));
        }
}
__device__ __forceinline__ void apply_pairs(double2 (&v)[kAPT], const PassStep &st, double c, double s) {
    for (int k = 0; k < st.npair; ++k) {
        switch (st.pair[k]) {
            case 0 * 8 + 1: givens_pair<0, 1>(v, c, s); break;
            case 0 * 8 + 2: givens_pair<0, 2>(v, c, s); break;
            case 0 * 8 + 3: givens_pair<0, 3>(v, c, s); break;
            case 0 * 8 + 4: givens_pair<0, 4>(v, c, s); break;
            case 1 * 8 + 2: givens_pair<1, 2>(v, c, s); break;
            case 1 * 8 + 3: givens_pair<1, 3>(v, c, s); break;
            case 1 * 8 + 4: givens_pair<1, 4>(v, c, s); break;
            case 2 * 8 + 3: givens_pair<2, 3>(v, c, s); break;
            case 2 * 8 + 4: givens_pair<2, 4>(v, c, s); break;
            case 3 * 8 + 4: givens_pair<3, 4>(v, c, s); break;
            default: break;
        }
    }
}
__device__ __forceinline__ double2 lds128(uint32_t a) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, double2 v) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

template <int G>
__device__ __forceinline__ void smem_read_g(double2 (&v)[kAPT], uint32_t buf, int c) {
    const uint32_t A = group_base<G>(buf, c);
#pragma unroll
    for (int e = 0; e < kAPT; ++e) v[e] = lds128(group_addr<G>(A, e));
}
template <int G>
__device__ __forceinline__ void smem_write_g(const double2 (&v)[kAPT], uint32_t buf, int c) {
    const uint32_t A = group_base<G>(buf, c);
#pragma unroll
    for (int e = 0; e < kAPT; ++e) sts128(group_addr<G>(A, e), v[e]);
}
// The q stage holds the tile's q in consumer order (qt_gather_kernel): fp64 values, or integer
// codes stored as j = code - qmin (uint8 / uint16).  Chunk c of 16 bytes of thread t sits at
// 16-byte index c * kCT + t (conflict-free LDS.128).
template <int QB>
__device__ __forceinline__ void apply_phase_group(double2 (&v)[kAPT], const unsigned char *qs, int c, int lane,
                                                  double gamma, const double2 *tab_s, const double2 *tab_g) {
    if (QB == 8) {
        const double2 *q2 = reinterpret_cast<const double2 *>(qs);
#pragma unroll
        for (int k = 0; k < kAPT / 2; ++k) {
            const double2 qq = q2[k * kCT + c];
            double sn, cs;
            sincos(gamma * qq.x, &sn, &cs);
            v[2 * k] = cmul(v[2 * k], make_double2(cs, -sn));
            sincos(gamma * qq.y, &sn, &cs);
            v[2 * k + 1] = cmul(v[2 * k + 1], make_double2(cs, -sn));
        }
    } else {
        constexpr int PER = 16 / (QB > 0 ? QB : 1);  // codes per 16-byte chunk
        const uint4 *q4 = reinterpret_cast<const uint4 *>(qs);
        const double2 *tab_l = tab_s + (lane & (kTabRep - 1));
#pragma unroll
        for (int k = 0; k < kAPT / PER; ++k) {
            const uint4 w = q4[k * kCT + c];
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int m = 0; m < PER; ++m) {
                int j;
                if (QB == 1) j = (int)((ww[m >> 2] >> (8 * (m & 3))) & 0xff);
                else j = (int)((ww[m >> 1] >> (16 * (m & 1))) & 0xffff);
                const double2 f = tab_s ? tab_l[j * kTabRep] : __ldg(tab_g + j);
                v[k * PER + m] = cmul(v[k * PER + m], f);
            }
        }
    }
}

template <int QB>
__device__ __forceinline__ void accumulate_expect(const double2 (&v)[kAPT], const unsigned char *qs, int c, int qmin,
                                                  double &acc, double &nrm) {
    if (QB == 8) {
        const double2 *q2 = reinterpret_cast<const double2 *>(qs);
#pragma unroll
        for (int k = 0; k < kAPT / 2; ++k) {
            const double2 qq = q2[k * kCT + c];
            const double p0 = v[2 * k].x * v[2 * k].x + v[2 * k].y * v[2 * k].y;
            const double p1 = v[2 * k + 1].x * v[2 * k + 1].x + v[2 * k + 1].y * v[2 * k + 1].y;
            acc = fma(p0, qq.x, acc);
            acc = fma(p1, qq.y, acc);
            nrm += p0 + p1;
        }
    } else {
        constexpr int PER = 16 / (QB > 0 ? QB : 1);
        const uint4 *q4 = reinterpret_cast<const uint4 *>(qs);
#pragma unroll
        for (int k = 0; k < kAPT / PER; ++k) {
            const uint4 w = q4[k * kCT + c];
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int m = 0; m < PER; ++m) {
                int j;
                if (QB == 1) j = (int)((ww[m >> 2] >> (8 * (m & 3))) & 0xff);
                else j = (int)((ww[m >> 1] >> (16 * (m & 1))) & 0xffff);
                const double2 a = v[k * PER + m];
                const double pr = a.x * a.x + a.y * a.y;
                acc = fma(pr, (double)(j + qmin), acc);
                nrm += pr;
            }
        }
    }
}

// ---- generated MaxCut qualities (QB = kQGenInt / kQGenF64) --
// q_x = -cut_w(x) is assembled per element from a per-tile record (the q stage holds it instead
// of 4096 stored values) and per-pass constants: with the tile's coordinate qubits T, the
// consumer thread's 7 thread-bit qubits H and its 5 register-bit qubits E,
//   cut(x) = [TT + K_H + K_E](t) + sum_{a in H, x_a = 1} kappa_a(t) + C(c)
//            + sum_j e_j (kappa_{E_j}(t) + beta_j(c)) + G(e)
// (kappa_a = sum over a's T-neighbours of w (1 - 2 x_b); C, beta: edges inside the tile touching
// H; G: edges among the E qubits).  Exact in integers for unit weights (phase by table), fp64
// sums otherwise.  Record: int {int32 T, int8 kappa[12]} (16 B) / fp64 {T, kappa[12]} (112 B).
template <int QB>
struct QGenT {
    using V = typename std::conditional<QB == kQGenInt, int, double>::type;
};
template <int QB>
constexpr uint32_t q_stage_bytes() {
    return QB == kQGenInt ? 16u : (QB == kQGenF64 ? 112u : (uint32_t)kTile * QB);
}
template <int QB>
__device__ __forceinline__ void gen_coeffs(const unsigned char *rec, const TileGroup &g, int c,
                                           const typename QGenT<QB>::V (&cst)[6], typename QGenT<QB>::V &S,
                                           typename QGenT<QB>::V (&al)[5]) {
    if constexpr (QB == kQGenInt) {
        const int8_t *k8 = reinterpret_cast<const int8_t *>(rec + 4);
        S = *reinterpret_cast<const int *>(rec) + cst[0];
#pragma unroll
        for (int j = 0; j < kCT_BITS; ++j)
            if ((c >> j) & 1) S += k8[g.tbit[j]];
#pragma unroll
        for (int j = 0; j < kGroupBits; ++j) al[j] = k8[g.ebit[j]] + cst[1 + j];
    } else {
        const double *kd = reinterpret_cast<const double *>(rec + 8);
        S = *reinterpret_cast<const double *>(rec) + cst[0];
#pragma unroll
        for (int j = 0; j < kCT_BITS; ++j)
            if ((c >> j) & 1) S += kd[g.tbit[j]];
#pragma unroll
        for (int j = 0; j < kGroupBits; ++j) al[j] = kd[g.ebit[j]] + cst[1 + j];
    }
}
template <int QB, int E>
__device__ __forceinline__ typename QGenT<QB>::V gen_cut(typename QGenT<QB>::V S,
                                                         const typename QGenT<QB>::V (&al)[5],
                                                         const typename QGenT<QB>::V *G_s) {
    typename QGenT<QB>::V x = S + G_s[E];
    if (E & 1) x += al[0];
    if (E & 2) x += al[1];
    if (E & 4) x += al[2];
    if (E & 8) x += al[3];
    if (E & 16) x += al[4];
    return x;
}
// fp64 weights, one member: exp(i gamma cut) factorised as e^{i gamma S} prod_j (e^{i gamma al_j})^{e_j}
// e^{i gamma G(e)}: 6 sincos per thread and tile instead of one per element, the 32 products
// walked in Gray-code order (one complex multiply per element; |z| = 1 so a removed factor is
// its conjugate), G factors from a per-pass smem table gf_s[32]
template <int E>
__device__ __forceinline__ constexpr int gray_flip() {
    return E == 0 ? -1 : __builtin_ctz((unsigned)E);
}
__device__ __forceinline__ void apply_phase_gen_f64_fact(double2 (&v)[kAPT], double S, const double (&al)[5],
                                                         const double2 *gf_s, double gamma) {
    double sn, cs;
    sincos(gamma * S, &sn, &cs);
    double2 run = make_double2(cs, sn);
    double2 z[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        sincos(gamma * al[j], &sn, &cs);
        z[j] = make_double2(cs, sn);
    }
    // four independent Gray-code chains over the low 3 register bits (one per value of bits 3, 4):
    // the same 31 products as one chain, a quarter of its dependency depth
    double2 r4[4];
    r4[0] = run;
    r4[1] = cmul(run, z[3]);
    r4[2] = cmul(run, z[4]);
    r4[3] = cmul(r4[1], z[4]);
    static_for<8>([&](auto gc) {
        constexpr int Gk = decltype(gc)::value;
        constexpr int El = Gk ^ (Gk >> 1);
        if constexpr (Gk > 0) {
            constexpr int J = gray_flip<Gk>();
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if constexpr ((El >> J) & 1) r4[h] = cmul(r4[h], z[J]);
                else r4[h] = cmul(r4[h], make_double2(z[J].x, -z[J].y));
            }
        }
#pragma unroll
        for (int h = 0; h < 4; ++h) v[El | (h << 3)] = cmul(v[El | (h << 3)], cmul(r4[h], gf_s[El | (h << 3)]));
    });
}

template <int QB>
__device__ __forceinline__ void apply_phase_gen(double2 (&v)[kAPT], const unsigned char *rec, const TileGroup &g,
                                                int c, int lane, const typename QGenT<QB>::V (&cst)[6],
                                                const typename QGenT<QB>::V *G_s, int m_edges, double gamma,
                                                const double2 *tab_s, const double2 *tab_g,
                                                const double2 *gf_s = nullptr) {
    using V = typename QGenT<QB>::V;
    V S, al[5];
    gen_coeffs<QB>(rec, g, c, cst, S, al);
    if constexpr (QB == kQGenF64) {
        if (gf_s) {
            apply_phase_gen_f64_fact(v, S, al, gf_s, gamma);
            return;
        }
    }
    const double2 *tab_l = tab_s + (lane & (kTabRep - 1));
    static_for<kAPT>([&](auto ec) {
        constexpr int E = decltype(ec)::value;
        const V cut = gen_cut<QB, E>(S, al, G_s);
        if constexpr (QB == kQGenInt) {
            const int j = m_edges - cut;  // q - qmin with q = -cut, qmin = -m
            const double2 f = tab_s ? tab_l[j * kTabRep] : __ldg(tab_g + j);
            v[E] = cmul(v[E], f);
        } else {
            double sn, cs;
            sincos(gamma * (-cut), &sn, &cs);
            v[E] = cmul(v[E], make_double2(cs, -sn));
        }
    });
}
template <int QB>
__device__ __forceinline__ void accumulate_gen(const double2 (&v)[kAPT], const unsigned char *rec, const TileGroup &g,
                                               int c, const typename QGenT<QB>::V (&cst)[6],
                                               const typename QGenT<QB>::V *G_s, double &acc, double &nrm) {
    using V = typename QGenT<QB>::V;
    V S, al[5];
    gen_coeffs<QB>(rec, g, c, cst, S, al);
    static_for<kAPT>([&](auto ec) {
        constexpr int E = decltype(ec)::value;
        const V cut = gen_cut<QB, E>(S, al, G_s);
        const double pr = v[E].x * v[E].x + v[E].y * v[E].y;
        acc = fma(pr, -(double)cut, acc);
        nrm += pr;
    });
}

template <int QB>
constexpr bool q_table() { return QB == 1 || QB == kQGenInt; }
template <int QB>
constexpr bool q_gen() { return QB == kQGenInt || QB == kQGenF64; }
template <int STAGES, int QB>
constexpr size_t tile_smem_bytes() {
    return (size_t)STAGES * (kTile * sizeof(double2) + (size_t)q_stage_bytes<QB>()) +
           (q_table<QB>() ? (size_t)kTabSmemMax * kTabRep * sizeof(double2) : 0) +
           (q_gen<QB>() ? 32 * sizeof(double) : 0) + (QB == kQGenF64 ? kGfMembers * 32 * sizeof(double2) : 0) +
           4 * STAGES * sizeof(uint64_t) +  // barriers + claimed items
           (size_t)kMaxBatchSmem * sizeof(PassAngles);
}

__device__ __forceinline__ void tma_coords(const TilePassParams &P, uint64_t member, uint64_t t, int (&c)[5]) {
#pragma unroll
    for (int d = 0; d < 5; ++d) {
        const int w = P.dim_w[d];
        int x = (int)((t >> P.dim_src[d]) & ((1ull << w) - 1));
        if (d == P.member_dim) x += (int)(member << w);
        c[d] = x;
    }
}

__device__ __forceinline__ void flush_partial(const TilePassParams &P, int64_t member, int warp, int lane, double &acc,
                                              double &nrm) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        nrm += __shfl_xor_sync(0xffffffffu, nrm, o);
    }
    if (lane == 0) {
        double2 *slot =
            reinterpret_cast<double2 *>(P.partials) + ((uint64_t)member * gridDim.x + blockIdx.x) * kCW + warp;
        const double2 old = *slot;
        *slot = make_double2(old.x + acc, old.y + nrm);
    }
    acc = nrm = 0.0;
}

// Pass programs: the group sequence, phase position and expectation of the common pass shapes
// fixed at compile time (straight-line code, no register reshuffling at control-flow joins);
// masks and angle slots stay runtime (PassStep).  Program 0 interprets P.steps at run time.
// kTileProgs in qva_internal.h lists the same shapes for the host-side matcher.
template <int PROG>
__device__ __forceinline__ constexpr TileProg prog_def() {
    return kTileProgs[PROG];
}
template <int PROG>
__device__ __forceinline__ constexpr int prog_release() {
    constexpr TileProg D = prog_def<PROG>();
    if (D.expect) return D.n;
    int r = 0;
    for (int k = 1; k < D.n; ++k)
        if (D.g[k] != D.g[k - 1]) r = k;
    if (D.phase_k > r) r = D.phase_k;
    return r;
}


template <int STAGES, int QB, int PROG>
__global__ void __launch_bounds__(kThreads, 1)
tile_pass_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_out,
                 const __grid_constant__ TilePassParams P) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];  // SWIZZLE_128B needs 1024-B alignment
    unsigned char *sm = smem_raw;
    constexpr uint32_t QSB = q_stage_bytes<QB>();
    using GV = typename QGenT<QB>::V;
    double2 *psi_s = reinterpret_cast<double2 *>(sm);
    unsigned char *q_s = sm + (size_t)STAGES * kTile * sizeof(double2);
    double2 *tab_s = reinterpret_cast<double2 *>(q_s + (size_t)STAGES * QSB);
    GV *G_s = reinterpret_cast<GV *>(reinterpret_cast<unsigned char *>(tab_s) +
                                     (q_table<QB>() ? kTabSmemMax * kTabRep * sizeof(double2) : 0));
    double2 *gf_s = reinterpret_cast<double2 *>(reinterpret_cast<unsigned char *>(G_s) +
                                                (q_gen<QB>() ? 32 * sizeof(double) : 0));
    uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<unsigned char *>(gf_s) +
                                                  (QB == kQGenF64 ? kGfMembers * 32 * sizeof(double2) : 0));
    uint64_t *items_s = bars + 2 * STAGES;  // item claimed for each barrier slot
    PassAngles *ang_s = reinterpret_cast<PassAngles *>(items_s + 2 * STAGES);  // [batch]
    // full[round & 1][stage]: item `it` is round it / STAGES of stage it % STAGES.  Rounds r and
    // r - 2 of a stage belong to the same warpgroup, so each barrier is waited by one warpgroup
    // at most one phase ahead (no parity aliasing).
    const uint32_t full0 = smem_u32(bars);
    auto slot_of = [&](uint32_t it) { return ((it / STAGES) & 1) * STAGES + it % STAGES; };
    auto full_bar = [&](uint32_t it) { return full0 + 8 * slot_of(it); };

    constexpr TileProg D = prog_def<PROG>();
    constexpr bool kPhase = PROG == 0 ? QB > 0 : D.phase_k >= 0;
    constexpr bool kExpect = PROG == 0 ? QB > 0 : D.expect;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const uint64_t n_items = P.n_tiles * (uint64_t)P.batch;
    // item order: claimed dynamically from P.work_ctr when set (CTA iteration j takes the next
    // free tile, so the in-flight tiles of the grid stay neighbours and SMs that stream faster
    // take more: static shares left some SMs idle for up to 20 % of a window pass); else
    // interleaved over CTAs (CTA b takes b, b + grid, ...)
    const bool dyn = P.work_ctr != nullptr;
    const uint32_t n_it = (uint32_t)((n_items > blockIdx.x) ? (n_items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
    auto item_of = [&](uint32_t j) -> uint64_t { return blockIdx.x + (uint64_t)j * gridDim.x; };
    const bool load_psi = (P.init != 1);
    const bool tstore = P.tma_store != 0;  // output through a TMA store of the final smem tile
    const bool load_q = (QB > 0) && (P.gq >= 0);
    const bool use_tab_s = q_table<QB>() && kPhase && P.batch == 1 && P.ntab <= kTabSmemMax && P.tab != nullptr;
    const uint32_t qbytes = load_q ? QSB : 0u;
    const uint32_t bytes = (load_psi ? kTile * (uint32_t)sizeof(double2) : 0u) + qbytes;
    const unsigned char *qt = reinterpret_cast<const unsigned char *>(P.qt);

    // TMA traffic for CTA iteration j (item blockIdx.x + j * gridDim.x)
    // A claimed item past the end is a sentinel: the barrier completes with no data and the
    // consumer stops.  Per warpgroup (iteration parity) the claims happen in iteration order, so
    // once a warpgroup meets a sentinel every later iteration of it is one too.
    auto issue = [&](uint32_t j, uint64_t claim = ~0ull) {
        const uint64_t item = dyn ? (claim != ~0ull ? claim : atomicAdd(P.work_ctr, 1ull)) : item_of(j);
        const uint64_t member = item >> P.log2_tiles, t = item & (P.n_tiles - 1);
        const int s = j % STAGES;
        const uint32_t bar = full_bar(j);
        if (dyn) {
            items_s[slot_of(j)] = item;
            if (item >= n_items) {
                mbar_expect_tx(bar, 0);
                return;
            }
        }
        mbar_expect_tx(bar, bytes);
        if (load_psi) {
            int cc[5];
            tma_coords(P, member, t, cc);
            tma_load_5d(smem_u32(psi_s + (size_t)s * kTile), &tmap, bar, cc);
        }
        if (qbytes) bulk_load(smem_u32(q_s + (size_t)s * QSB), qt + t * (uint64_t)qbytes, qbytes, bar);
    };

    if (tid == 0) {
        if (smem_u32(smem_raw) & 1023) __trap();
        for (int k = 0; k < 2 * STAGES; ++k) mbar_init(full0 + 8 * k, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (use_tab_s)
        for (int k = tid; k < P.ntab * kTabRep; k += kThreads) tab_s[k] = P.tab[k / kTabRep];
    for (int k = tid; k < P.batch; k += kThreads) ang_s[k] = P.angles[k];
    // generated qualities: per-pass G(e) table and this consumer thread's constants {C, beta[5]}
    GV gcst[6] = {};
    if constexpr (q_gen<QB>()) {
        if (load_q) {
            const GV *Gg = reinterpret_cast<const GV *>(P.gen_G);
            for (int k = tid; k < 32; k += kThreads) G_s[k] = Gg[k];
            if constexpr (QB == kQGenF64) {  // G factors e^{i gamma_b G(e)} per member b
                if (P.batch <= kGfMembers)
                    for (int k = tid; k < 32 * P.batch; k += kThreads) {
                        double sn, cs;
                        sincos(P.angles[k >> 5].gamma * (double)Gg[k & 31], &sn, &cs);
                        gf_s[k] = P.fold_scale_gf ? cmul(make_double2(cs, sn), P.angles[k >> 5].scale)
                                                  : make_double2(cs, sn);
                    }
            }
            const GV *cg = reinterpret_cast<const GV *>(P.gen_thr) + (size_t)(tid % kCT) * 8;
#pragma unroll
            for (int k = 0; k < 6; ++k) gcst[k] = cg[k];
        }
    }
    __syncthreads();
    if (tid == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        for (uint32_t j = 0; j < (uint32_t)STAGES && (dyn || j < n_it); ++j) issue(j);
    }

    // ---------------- warpgroup wg takes CTA iterations wg, wg + 2, ... ----------------
    const int wg = tid / kCT;
    const int c = tid % kCT;
    // store addressing of the final group (host-computed): phys = member*stride + base(t)
    //   + sum_j c_j << st_tphys[j] + sum_j e_j st_estr[j]
    uint64_t tbase = 0;
#pragma unroll
    for (int j = 0; j < kCT_BITS; ++j) tbase |= (uint64_t)((c >> j) & 1) << P.st_tphys[j];

    double acc = 0.0, nrm = 0.0;
    int64_t acc_member = -1;

    const bool preclaim = dyn && (P.tail_mode & 1), defer = (P.tail_mode & 2) != 0;
    uint32_t pending = ~0u;
    uint64_t pending_claim = ~0ull;
    auto flush_pending = [&]() {
        if (c == 0 && pending != ~0u) {
            bulk_wait_read_all();
            issue(pending, pending_claim);
            pending = ~0u;
        }
    };
    for (uint32_t it = wg; dyn || it < n_it; it += kWG) {
        const int s = it % STAGES;
        uint64_t item;
        flush_pending();
        if (dyn) {
            mbar_wait(full_bar(it), ((it / STAGES) >> 1) & 1);
            item = items_s[slot_of(it)];
            if (item >= n_items) {  // keep the claim chain going for the other warpgroup, then stop
                if (c == 0) issue(it + STAGES);
                break;
            }
        } else {
            item = item_of(it);
        }
        const uint64_t member = item >> P.log2_tiles;
        const uint64_t t = item & (P.n_tiles - 1);
        const PassAngles *ang = ang_s + member;
        const double2 *tab_g = P.tab ? P.tab + member * P.ntab : nullptr;
        if (QB > 0 && kExpect && P.expect && (int64_t)member != acc_member) {
            if (acc_member >= 0) flush_partial(P, acc_member, warp, lane, acc, nrm);
            acc_member = (int64_t)member;
        }

        const uint32_t buf = smem_u32(psi_s + (size_t)s * kTile);
        const unsigned char *qs = q_s + (size_t)s * QSB;
        if (!dyn) mbar_wait(full_bar(it), ((it / STAGES) >> 1) & 1);
        uint64_t pre_claim = ~0ull;
        if (preclaim && c == 0) pre_claim = atomicAdd(P.work_ctr, 1ull);

        // hand stage s back: the whole warpgroup is done with it, so one thread refills it with
        // iteration it + STAGES (the async-proxy write must follow our generic-proxy accesses)
        auto release = [&]() {
            fence_proxy_async();
            wg_sync(wg);
            if (c == 0 && (dyn || it + STAGES < n_it)) issue(it + STAGES, pre_claim);
        };
        double2 v[kAPT];
        if (!load_psi) {
#pragma unroll
            for (int e = 0; e < kAPT; ++e) v[e] = make_double2(P.amp0, 0.0);
        }
        if constexpr (PROG == 0) {
            if (P.release_step < 0 && !tstore) release();
            // every step is straight-line code for a compile-time group: read the tile in that
            // group's layout if the previous step used another one, rotate, apply the phase, and
            // write the tile back if the next step switches
            int prev = load_psi ? -1 : P.steps[0].group;
            for (int k = 0; k < P.n_steps; ++k) {
                const PassStep st = P.steps[k];
                const int next = (k + 1 < P.n_steps) ? P.steps[k + 1].group : st.group;
                const double tt = st.mask ? (st.angle ? ang->t2 : ang->t1) : 0.0;
                auto body = [&](auto gc) {
                    constexpr int G = decltype(gc)::value;
                    if (prev != G) {
                        if (prev >= 0) {
                            flush_pending();
                            wg_sync(wg);
                        }
                        smem_read_g<G>(v, buf, c);
                    }
                    if constexpr (G <= 2) {
                        if (st.mask) rotate_group<G>(v, st.mask, tt);
                    }
                    if (QB > 0 && st.phase) {
                        if constexpr (q_gen<QB>())
                            apply_phase_gen<QB>(v, qs, P.groups[P.gq], c, lane, gcst, G_s, P.gen_m, ang->gamma,
                                                use_tab_s ? tab_s : nullptr, tab_g,
                                                P.batch <= kGfMembers ? gf_s + 32 * member : nullptr);
                        else
                            apply_phase_group<QB>(v, qs, c, lane, ang->gamma, use_tab_s ? tab_s : nullptr, tab_g);
                    }
                    if (st.npair) apply_pairs(v, st, ang->t1, ang->t2);  // QAOAz: after the step's phase
                    if (next != G) smem_write_g<G>(v, buf, c);
                };
                switch (st.group) {
                    case 0: body(std::integral_constant<int, 0>()); break;
                    case 1: body(std::integral_constant<int, 1>()); break;
                    case 2: body(std::integral_constant<int, 2>()); break;
                    case 3: body(std::integral_constant<int, 3>()); break;
                    default: body(std::integral_constant<int, 4>()); break;
                }
                prev = st.group;
                if (k == P.release_step && !tstore) release();
            }
        } else {
            constexpr int REL = prog_release<PROG>();
            static_for<D.n>([&](auto kc) {
                constexpr int K = decltype(kc)::value;
                constexpr int G = prog_def<PROG>().g[K];
                if constexpr (K == 0) {
                    if (load_psi) smem_read_g<G>(v, buf, c);
                } else if constexpr (prog_def<PROG>().g[K - 1] != G) {
                    flush_pending();
                    wg_sync(wg);
                    smem_read_g<G>(v, buf, c);
                }
                if constexpr (prog_def<PROG>().rot[K]) {
                    const PassStep st = P.steps[K];
                    rotate_group<G>(v, st.mask, st.angle ? ang->t2 : ang->t1);
                }
                if constexpr (QB > 0 && K == prog_def<PROG>().phase_k) {
                    if constexpr (q_gen<QB>())
                        apply_phase_gen<QB>(v, qs, P.groups[P.gq], c, lane, gcst, G_s, P.gen_m, ang->gamma,
                                            use_tab_s ? tab_s : nullptr, tab_g,
                                                P.batch <= kGfMembers ? gf_s + 32 * member : nullptr);
                    else
                        apply_phase_group<QB>(v, qs, c, lane, ang->gamma, use_tab_s ? tab_s : nullptr, tab_g);
                }
                if constexpr (PROG >= kFirstParityProg) apply_pairs(v, P.steps[K], ang->t1, ang->t2);  // QAOAz programs
                if constexpr (K == REL) {
                    if (!tstore) release();
                }
                if constexpr (K + 1 < prog_def<PROG>().n && prog_def<PROG>().g[K + 1] != G) smem_write_g<G>(v, buf, c);
            });
        }
        if (P.apply_scale) {
            const double2 sc = ang->scale;
#pragma unroll
            for (int e = 0; e < kAPT; ++e) v[e] = cmul(v[e], sc);
        }
        if constexpr (QB > 0 && kExpect) {
            if (P.expect) {
                if constexpr (q_gen<QB>()) accumulate_gen<QB>(v, qs, P.groups[P.gq], c, gcst, G_s, acc, nrm);
                else accumulate_expect<QB>(v, qs, c, P.qmin, acc, nrm);
            }
        }
        if (tstore) {
            // the tile goes back through shared memory in the load layout and out with one TMA
            // store; the stage is refilled once the store engine has read it
            if constexpr (PROG == 0) {
                switch (P.steps[P.n_steps - 1].group) {
                    case 0: smem_write_g<0>(v, buf, c); break;
                    case 1: smem_write_g<1>(v, buf, c); break;
                    case 2: smem_write_g<2>(v, buf, c); break;
                    case 3: smem_write_g<3>(v, buf, c); break;
                    default: smem_write_g<4>(v, buf, c); break;
                }
            } else {
                smem_write_g<prog_def<PROG>().g[prog_def<PROG>().n - 1]>(v, buf, c);
            }
            flush_pending();
            fence_proxy_async();
            wg_sync(wg);
            if (c == 0) {
                int cc[5];
                tma_coords(P, member, t, cc);
                tma_store_5d(&tmap_out, buf, cc);
                if (defer) {
                    if (dyn || it + STAGES < n_it) {
                        pending = it + STAGES;
                        pending_claim = pre_claim;
                    }
                } else {
                    bulk_wait_read_all();
                    if (dyn || it + STAGES < n_it) issue(it + STAGES, pre_claim);
                }
            }
            continue;
        }
        if constexpr (PROG == 0) {
            if (P.release_step >= P.n_steps) release();
        } else if constexpr (prog_release<PROG>() >= prog_def<PROG>().n) {
            release();
        }

        uint64_t base = member * P.member_stride;
#pragma unroll
        for (int r = 0; r < kMaxRuns; ++r) base |= ((t >> P.run_src[r]) & P.run_mask[r]) << P.run_dst[r];
        double2 *out = P.psi_out;
        if (P.xg) {  // fused exchange: the tile's chunk (never a tile bit) names the receiving rank
            const uint64_t m = (uint64_t)(P.xg - 1) << P.xshift;
            uint64_t src = (uint64_t)P.xrank;
            if (P.xvirt) {
                const int hs = P.xshift + __ffs(P.xg) - 1;  // = L: the virtual shard bits
                src = (base >> hs) & (uint64_t)(P.xg - 1);
                base &= (1ull << hs) - 1;
            }
            out = P.xpeer[(base & m) >> P.xshift];
            base = (base & ~m) | (src << P.xshift);
        }
        double2 *dst = out + base + tbase;
#pragma unroll
        for (int e = 0; e < kAPT; ++e) {
            uint64_t o = 0;
#pragma unroll
            for (int j = 0; j < kGroupBits; ++j)
                if (e & (1 << j)) o += P.st_estr[j];
            __stcs(dst + o, v[e]);
        }
    }
    flush_pending();
    if (tstore && c == 0) bulk_wait_all();
    if (P.xg) __threadfence_system();  // peer stores visible before the host-side barrier
    if (QB > 0 && kExpect && P.expect && acc_member >= 0) flush_partial(P, acc_member, warp, lane, acc, nrm);
}

// Consumer-order uint8 codes j = m - cut(x) of generated unit-weight MaxCut qualities (q = -cut,
// qmin = -m), written once per (q, pass shape, register group) from the same per-tile records and
// per-thread constants the in-pass generator uses: the passes then read 1 B per amplitude through
// the stored-code path (QB = 1) instead of assembling cut(x) per element (A/B on one B200, cfg4:
// the two phase passes 6.35 -> 5.80 ms each).  Layout as qt_gather_kernel: thread c's codes 16 per
// 16-byte chunk at chunk index (e / 16) * kCT + c.
__global__ void gen_codes_kernel(uint8_t *codes, const unsigned char *rec, uint64_t n_tiles, const int *thr,
                                 const int *Gv, TileGroup g, int m) {
    const uint64_t total = n_tiles * kCT;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = k / kCT;
        const int c = (int)(k % kCT);
        int cst[6];
#pragma unroll
        for (int i = 0; i < 6; ++i) cst[i] = thr[c * 8 + i];
        int S, al[5];
        gen_coeffs<kQGenInt>(rec + t * 16, g, c, cst, S, al);
        uint4 out[2];
        uint32_t *w = reinterpret_cast<uint32_t *>(out);
        static_for<kAPT>([&](auto ec) {
            constexpr int E = decltype(ec)::value;
            const int cut = gen_cut<kQGenInt, E>(S, al, Gv);
            const uint32_t j = (uint32_t)(m - cut) & 0xffu;
            if constexpr ((E & 3) == 0) w[E >> 2] = j;
            else w[E >> 2] |= j << (8 * (E & 3));
        });
        uint4 *dst = reinterpret_cast<uint4 *>(codes + t * (uint64_t)kTile);
        dst[c] = out[0];
        dst[kCT + c] = out[1];
    }
}

// logical index of physical index x under a layout given as bit runs (LayoutRuns)
__device__ __forceinline__ uint64_t layout_map(const LayoutRuns &R, uint64_t x) {
    uint64_t y = 0;
    for (int r = 0; r < R.n; ++r) y |= ((x >> R.src[r]) & ((1ull << R.w[r]) - 1)) << R.dst[r];
    return y;
}

// q (fp64 or integer codes) permuted into the consumer order of register group G of tile set S:
// dst[t][pos(tid, e)] = src[logical(phys(t, i(tid, e)))], pos as read by apply_phase_group /
// accumulate_expect; `lay` maps the pass's physical layout to the logical index of q.
// One thread per (tile t, consumer thread c) writes c's 32 values as whole 16-byte chunks.  Both
// maps are bit maps (tile bit b -> physical bit tile_bits[b] -> logical bit), so the logical index
// is the OR of the images of the set bits: the tile's coordinate part once per thread, the
// thread's part once, and one OR per register element from five precomputed bit images (the
// per-element bit loops this replaces made the 1-byte gathers compute-bound: ~10 ms per GiB).
template <typename T>
__global__ void qt_gather_kernel(T *dst, const T *src, const __grid_constant__ TilePassParams P, TileGroup G,
                                 uint64_t n_tiles, int qmin, const __grid_constant__ LayoutRuns lay) {
    constexpr int PER = 16 / (int)sizeof(T);  // values per 16-byte chunk
    const uint64_t total = n_tiles * (uint64_t)kCT;
    uint64_t eimg[kGroupBits];
#pragma unroll
    for (int j = 0; j < kGroupBits; ++j) eimg[j] = layout_map(lay, 1ull << P.tile_bits[G.ebit[j]]);
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < total;
         k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = k / kCT;
        const int c = (int)(k % kCT);
        uint64_t phys = 0;
        for (int r = 0; r < P.n_runs; ++r) phys |= ((t >> P.run_src[r]) & ((1ull << P.run_w[r]) - 1)) << P.run_dst[r];
        for (int j = 0; j < kCT_BITS; ++j) phys |= (uint64_t)((c >> j) & 1) << P.tile_bits[G.tbit[j]];
        const uint64_t base = layout_map(lay, phys);
        T *out = dst + t * (uint64_t)kTile;
#pragma unroll
        for (int ch = 0; ch < kAPT / PER; ++ch) {
            union {
                uint4 u;
                T v[PER];
            } w;
#pragma unroll
            for (int r = 0; r < PER; ++r) {
                const int e = ch * PER + r;
                uint64_t x = base;
#pragma unroll
                for (int j = 0; j < kGroupBits; ++j)
                    if ((e >> j) & 1) x |= eimg[j];
                if (sizeof(T) == 8) w.v[r] = src[x];
                else w.v[r] = (T)((int)src[x] - qmin);  // integer codes stored as j = code - qmin
            }
            reinterpret_cast<uint4 *>(out)[ch * kCT + c] = w.u;
        }
    }
}

// out[logical(x)] = in[x] for every physical index x: returns a permuted state to the natural
// layout (reads are coalesced; writes land in 128-B rows because bits 0..2 never move)
__global__ void permute_copy_kernel(double2 *__restrict__ out, const double2 *__restrict__ in, uint64_t n,
                                    const __grid_constant__ LayoutRuns lay) {
    for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x)
        out[layout_map(lay, x)] = in[x];
}

// Per-tile records of the generated MaxCut qualities (see QGenT): for tile t, with x the logical
// index pattern of its coordinate (and constant) qubits,
//   T(t)     = sum_{TT edges} w [x_u != x_v] + sum_{TB edges (a, b)} w x_b
//   kappa_a  = sum_{TB edges (a, b)} w (1 - 2 x_b)        (a = tile-local bit)
template <typename V>
__global__ void gen_records_kernel(unsigned char *rec, uint64_t n_tiles, uint32_t rec_bytes,
                                   const __grid_constant__ GenPrep g) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
         t += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t x = g.const_val;
        for (int r = 0; r < g.tmap.n; ++r)
            x |= ((t >> g.tmap.src[r]) & ((1ull << g.tmap.w[r]) - 1)) << g.tmap.dst[r];
        V T = 0, kap[kTileBits];
#pragma unroll
        for (int a = 0; a < kTileBits; ++a) kap[a] = 0;
        for (int e = 0; e < g.n_tt; ++e) {
            const int2 uv = g.tt_uv[e];
            const V w = g.w_unit ? (V)1 : (V)g.tt_w[e];
            if (((x >> uv.x) ^ (x >> uv.y)) & 1) T += w;
        }
        for (int e = 0; e < g.n_tb; ++e) {
            const int2 ab = g.tb_ab[e];  // (tile-local bit, logical qubit)
            const V w = g.w_unit ? (V)1 : (V)g.tb_w[e];
            const bool xb = (x >> ab.y) & 1;
            if (xb) T += w;
#pragma unroll
            for (int a = 0; a < kTileBits; ++a)
                if (a == ab.x) kap[a] += xb ? -w : w;
        }
        unsigned char *r = rec + t * rec_bytes;
        if constexpr (std::is_same<V, int>::value) {
            *reinterpret_cast<int *>(r) = T;
            for (int a = 0; a < kTileBits; ++a) reinterpret_cast<int8_t *>(r + 4)[a] = (int8_t)kap[a];
        } else {
            reinterpret_cast<double *>(r)[0] = T;
            for (int a = 0; a < kTileBits; ++a) reinterpret_cast<double *>(r + 8)[a] = kap[a];
        }
    }
}

template <int STAGES, int QB, int PROG>
cudaError_t launch_one(const CUtensorMap &map, const CUtensorMap &map_out, const TilePassParams &p, int grid,
                       cudaStream_t s) {
    static DeviceOnce configured;
    constexpr size_t smem = tile_smem_bytes<STAGES, QB>();
    static_assert(smem <= 232448, "shared memory budget");
    cudaError_t e = once_per_device(configured, [] {
        return cudaFuncSetAttribute(tile_pass_kernel<STAGES, QB, PROG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem);
    });
    if (e != cudaSuccess) return e;
    tile_pass_kernel<STAGES, QB, PROG><<<grid, kThreads, smem, s>>>(map, map_out, p);
    return cudaGetLastError();
}

template <int STAGES, int QB>
cudaError_t launch_prog(const CUtensorMap &map, const CUtensorMap &mo, const TilePassParams &p, int prog, int grid,
                        cudaStream_t s) {
    switch (prog) {
        case 1: return launch_one<STAGES, QB, 1>(map, mo, p, grid, s);
        case 2: return launch_one<STAGES, QB, 2>(map, mo, p, grid, s);
        case 3: return launch_one<STAGES, QB, 3>(map, mo, p, grid, s);
        case 4: return launch_one<STAGES, QB, 4>(map, mo, p, grid, s);
        case 5: return launch_one<STAGES, QB, 5>(map, mo, p, grid, s);
        case 6: return launch_one<STAGES, QB, 6>(map, mo, p, grid, s);
        case 7: return launch_one<STAGES, QB, 7>(map, mo, p, grid, s);
        case 8: return launch_one<STAGES, QB, 8>(map, mo, p, grid, s);
        case 9: return launch_one<STAGES, QB, 9>(map, mo, p, grid, s);
        case 10: return launch_one<STAGES, QB, 10>(map, mo, p, grid, s);
        case 11: return launch_one<STAGES, QB, 11>(map, mo, p, grid, s);
        case 12: return launch_one<STAGES, QB, 12>(map, mo, p, grid, s);
        case 13: return launch_one<STAGES, QB, 13>(map, mo, p, grid, s);
        case 14: return launch_one<STAGES, QB, 14>(map, mo, p, grid, s);
        case 15: return launch_one<STAGES, QB, 15>(map, mo, p, grid, s);
        case 16: return launch_one<STAGES, QB, 16>(map, mo, p, grid, s);
        case 17: return launch_one<STAGES, QB, 17>(map, mo, p, grid, s);
        case 18: return launch_one<STAGES, QB, 18>(map, mo, p, grid, s);
        default: return launch_one<STAGES, QB, 0>(map, mo, p, grid, s);
    }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

}  // namespace

int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;  // B200
    }
    return sms;
}

int tile_pass_grid(uint64_t items) {
    const int sms = num_sms();
    uint64_t g = std::min<uint64_t>(items, (uint64_t)sms);
    return (int)std::max<uint64_t>(g, 1);
}

// TMA dims of a tile pass: maximal runs of input-physical bits that agree in tile membership and
// map to consecutive output bits under obit; tile runs split into <= 8-bit box dims (bits 0-2 =
// 16 doubles = one 128-B swizzle row).
struct TmaDim {
    int lo, w;
    bool tile;
};
static std::vector<TmaDim> tile_dims(const int *tile_bits, int L, const int *obit) {
    uint64_t tmask = 0;
    for (int k = 0; k < kTileBits; ++k) tmask |= 1ull << tile_bits[k];
    auto ob = [&](int b) { return obit ? obit[b] : b; };
    std::vector<TmaDim> dims;
    int b = 0;
    while (b < L) {
        const bool tile = (tmask >> b) & 1;
        const int st = b;
        ++b;
        while (b < L && (((tmask >> b) & 1) != 0) == tile && ob(b) == ob(b - 1) + 1) ++b;
        if (tile) {
            int x = st;
            while (x < b) {
                int w = (x == 0) ? std::min(3, b - x) : std::min(8, b - x);
                dims.push_back({x, w, true});
                x += w;
            }
        } else {
            dims.push_back({st, b - st, false});
        }
    }
    return dims;
}

int tile_tma_dims(const int *tile_bits, int L, const int *obit) { return (int)tile_dims(tile_bits, L, obit).size(); }

// Tensor maps of one member array (or `batch` consecutive members of member_stride = 2^L
// elements) seen through tile set P.tile_bits: dims in ascending input-physical order, each
// maximal run of tile bits split into <= 8-bit box dims (bits 0-2 = 16 doubles = one 128-B
// swizzle row), each run of non-tile bits one dim with box 1 (its coordinate comes from the
// tile number), the member index folded into the topmost non-tile dim.  Fills P.dim_* fields.
//
// The load map reads the input layout; the store map writes the same box to psi_out through
// the bit permutation obit (input physical bit b -> output physical bit obit[b]; nullptr =
// identity, i.e. an in-place style store).  Runs are additionally split wherever obit is not
// consecutive, so every dim of the shared box maps to one contiguous output run: a permuted
// store is still one TMA instruction per tile, with its own strides.
qva_status make_tile_tensor_maps(const double2 *psi_in, double2 *psi_out, int L, int batch, TilePassParams &P,
                                 const int *obit, CUtensorMap *map_in, CUtensorMap *map_out) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled entry point unavailable");
        return QVA_ERR_CUDA;
    }
    auto ob = [&](int b) { return obit ? obit[b] : b; };
    std::vector<TmaDim> dims = tile_dims(P.tile_bits, L, obit);
    if (dims.empty() || !dims[0].tile || dims[0].lo != 0 || dims[0].w != 3 || ob(0) != 0 || ob(1) != 1 ||
        ob(2) != 2) {
        set_error("tile set must contain physical bits 0,1,2 (kept in place by the store map)");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    int member_dim = -1;
    uint64_t member_extra = 1;
    if (batch > 1) {
        if (!dims.back().tile) {
            member_dim = (int)dims.size() - 1;
        } else {
            dims.push_back({L, 0, false});
            member_dim = (int)dims.size() - 1;
        }
        member_extra = (uint64_t)batch;
        // the member index is folded into the top dim: its output run must stay at the top
        const TmaDim &m = dims[member_dim];
        if (m.w > 0 && ob(m.lo) + m.w != L) {
            set_error("batched tile pass: permuted store must keep the top run in place");
            return QVA_ERR_UNSUPPORTED;
        }
    }
    if (dims.size() > 5) {
        set_error("tile set needs more than 5 TMA dimensions");
        return QVA_ERR_UNSUPPORTED;
    }
    cuuint64_t gdim[5], gstride[4], gstride_o[4];
    cuuint32_t box[5], estr[5];
    int src = 0;
    for (int d = 0; d < 5; ++d) {
        estr[d] = 1;
        if (d < (int)dims.size()) {
            const TmaDim &x = dims[d];
            uint64_t sz = 1ull << x.w;
            if (d == member_dim) sz *= member_extra;
            gdim[d] = (d == 0) ? 2 * sz : sz;  // dim 0 counts doubles (re, im)
            box[d] = x.tile ? (cuuint32_t)((d == 0) ? 2 * sz : sz) : 1;
            if (d > 0) {
                gstride[d - 1] = (cuuint64_t)(1ull << x.lo) * sizeof(double2);
                gstride_o[d - 1] = (cuuint64_t)(1ull << (x.lo < L ? ob(x.lo) : L)) * sizeof(double2);
            }
            if (x.tile) {
                P.dim_src[d] = 0;
                P.dim_w[d] = 0;
            } else {
                P.dim_src[d] = src;
                P.dim_w[d] = x.w;
                src += x.w;
            }
        } else {
            gdim[d] = 1;
            box[d] = 1;
            gstride[d - 1] = 16;  // size-1 padding dim: any legal stride
            gstride_o[d - 1] = 16;
            P.dim_src[d] = 0;
            P.dim_w[d] = 0;
        }
    }
    P.member_dim = member_dim;
    // L2 fill granule: 256 B only when every box row run is >= 256 B contiguous (tile bits 0..3)
    static const int promo_env = [] {
        const char *e = getenv("QVA_L2PROMO");
        return e ? atoi(e) : -1;
    }();
    auto promo_for = [&](bool wide) {
        CUtensorMapL2promotion promo = wide ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
        if (promo_env >= 0 && !wide) promo = (CUtensorMapL2promotion)promo_env;
        return promo;
    };
    const bool wide_in = dims.size() > 1 && dims[1].tile && dims[1].lo == 3;
    const bool wide_out = dims.size() > 1 && dims[1].tile && ob(dims[1].lo) == 3;
    CUresult r = enc(map_in, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, const_cast<double2 *>(psi_in), gdim, gstride, box,
                     estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo_for(wide_in),
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS && map_out)
        r = enc(map_out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, psi_out, gdim, gstride_o, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo_for(wide_out),
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
        return QVA_ERR_CUDA;
    }
    return QVA_OK;
}

cudaError_t launch_tile_pass(const CUtensorMap &map, const CUtensorMap &map_out, const TilePassParams &p, int qbytes,
                             int prog, int grid, cudaStream_t s) {
    // programs without phase/expectation never take q; those with it always do
    const bool qprog = prog == 0 || kTileProgs[prog].phase_k >= 0 || kTileProgs[prog].expect;
    switch (qbytes) {
        case 0: return qprog && prog != 0 ? cudaErrorInvalidValue : launch_prog<3, 0>(map, map_out, p, prog, grid, s);
        case 1: return qprog ? launch_prog<3, 1>(map, map_out, p, prog, grid, s) : cudaErrorInvalidValue;
        case 2: return qprog ? launch_prog<3, 2>(map, map_out, p, prog, grid, s) : cudaErrorInvalidValue;
        case 8: return qprog ? launch_prog<2, 8>(map, map_out, p, prog, grid, s) : cudaErrorInvalidValue;
        case kQGenInt: return qprog ? launch_prog<3, kQGenInt>(map, map_out, p, prog, grid, s) : cudaErrorInvalidValue;
        case kQGenF64: return qprog ? launch_prog<3, kQGenF64>(map, map_out, p, prog, grid, s) : cudaErrorInvalidValue;
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_qt_gather(void *dst, const void *src, int qbytes, const TilePassParams &p, const TileGroup &g,
                             uint64_t n_tiles, int qmin, const LayoutRuns &lay, cudaStream_t s) {
    const uint64_t total = n_tiles * (uint64_t)kCT;
    int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 16);
    if (qbytes == 8)
        qt_gather_kernel<double><<<blocks, 256, 0, s>>>((double *)dst, (const double *)src, p, g, n_tiles, 0, lay);
    else if (qbytes == 2)
        qt_gather_kernel<int16_t>
            <<<blocks, 256, 0, s>>>((int16_t *)dst, (const int16_t *)src, p, g, n_tiles, qmin, lay);
    else qt_gather_kernel<int8_t><<<blocks, 256, 0, s>>>((int8_t *)dst, (const int8_t *)src, p, g, n_tiles, qmin, lay);
    return cudaGetLastError();
}

cudaError_t launch_gen_codes(void *codes, const void *rec, uint64_t n_tiles, const void *thr, const void *G,
                             const TileGroup &g, int m, cudaStream_t s) {
    const uint64_t total = n_tiles * kCT;
    int blocks = (int)std::min<uint64_t>((total + 255) / 256, (uint64_t)num_sms() * 16);
    gen_codes_kernel<<<blocks, 256, 0, s>>>((uint8_t *)codes, (const unsigned char *)rec, n_tiles, (const int *)thr,
                                            (const int *)G, g, m);
    return cudaGetLastError();
}

cudaError_t launch_gen_records(void *rec, uint64_t n_tiles, int fp64, const GenPrep &g, cudaStream_t s) {
    int blocks = (int)std::min<uint64_t>((n_tiles + 255) / 256, (uint64_t)num_sms() * 8);
    if (fp64) gen_records_kernel<double><<<blocks, 256, 0, s>>>((unsigned char *)rec, n_tiles, 112, g);
    else gen_records_kernel<int><<<blocks, 256, 0, s>>>((unsigned char *)rec, n_tiles, 16, g);
    return cudaGetLastError();
}

cudaError_t launch_permute_copy(double2 *out, const double2 *in, uint64_t n, const LayoutRuns &lay, cudaStream_t s) {
    int blocks = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)num_sms() * 16);
    permute_copy_kernel<<<blocks, 256, 0, s>>>(out, in, n, lay);
    return cudaGetLastError();
}

int tile_consumer_warps() { return kCW; }

}  // namespace qva
