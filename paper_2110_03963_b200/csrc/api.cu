// api.cu -- the C ABI (include/qva.h): plan lifecycle, layer scheduler, global-qubit exchange,
// batch sharding and NCCL plumbing.  All arithmetic of the method runs in the kernels of
// kernels_x.cu / kernels_fft.cu / kernels_sparse.cu; this file only plans and launches.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <functional>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "qva_internal.h"

namespace qva {

// NVTX range over one C-ABI call (visible in Nsight Systems / ncu --nvtx; a no-op without a tool attached)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange &) = delete;
    NvtxRange &operator=(const NvtxRange &) = delete;
};

static thread_local std::string g_last_error;
void set_error(const std::string &msg) { g_last_error = msg; }
// QVA_TRACE=1: per-launch device times of profiled plans on stderr; 2: also each pass's program
static int g_tstore = [] {
    const char *e = getenv("QVA_TSTORE");
    return e ? atoi(e) : -1;
}();
static int g_trace = [] {
    const char *e = getenv("QVA_TRACE");
    return e ? atoi(e) : 0;
}();

// ---------------------------------------------------------------------------------------------
// X-mixer schedule
//
// The mixer U_M(beta) = prod_j exp(-i beta X_j) is a product of commuting single-qubit
// rotations, and the phase is diagonal, so one HBM pass over a tile of 2^12 amplitudes can
// apply any rotations whose qubits are tile bits, and the phase may sit between two rotation
// sets (tail of layer k, phase gamma_{k+1}, head of layer k+1).  The evolution is a token
// stream PHASE(k) ROT(all,k) PHASE(k+1) ROT(all,k+1) ... (sharded: EXCHANGE / ROT(H,k)
// between epochs) and passes are cut greedily from it.
// ---------------------------------------------------------------------------------------------
struct Token {
    enum Kind { PHASE, ROT, EXCHANGE } kind;
    uint64_t bits;  // ROT: physical bits to rotate
    int layer;      // PHASE: gamma index; ROT: beta index
};

struct PassPlan {
    bool exchange = false;   // this entry is an exchange, not a tile pass
    int set = -1;            // in-place passes: index into the plan's tile sets
    uint32_t r1 = 0, r2 = 0; // tile-local masks
    int a1 = -1, a2 = -1;    // layer index of beta for R1 / R2
    int phase = -1;          // layer index of gamma
    bool expect = false;
    // permuted out-of-place passes (perm_passes): physical tile bits of the input layout, the
    // layout before the pass (physical bit -> logical qubit) and the store permutation
    // (input physical bit -> output physical bit)
    bool permuted = false;
    std::vector<int> tbits, lay_in, obit;
    // QAOAz parity window pass (parity_tile_passes): in place over tile bits `tbits`, the step list
    // (register groups + pair terms) planned on the host, pair angle of layer `play`
    bool parity = false;
    int play = -1;
    std::vector<PassStep> psteps;
};

struct ParityWinPlan {
    std::vector<int> bits;            // window bits (ascending, physical = logical here)
    std::vector<int> ta, tb, cls;     // its pair terms in application order; cls 0 odd, 1 even, 2 last
};
struct ParityItem {              // sharded QAOAz schedule: a window of local bits or one global term
    bool global = false;
    ParityWinPlan win;
    int a = -1, b = -1;
};

static std::vector<std::vector<int>> make_tile_sets(int L) {
    std::vector<std::vector<int>> sets;
    std::vector<int> s0;
    for (int b = 0; b < kTileBits; ++b) s0.push_back(b);
    sets.push_back(s0);
    int next = kTileBits;
    while (next < L) {
        std::vector<int> s = {0, 1, 2};
        while ((int)s.size() < kTileBits && next < L) s.push_back(next++);
        for (int b = 3; (int)s.size() < kTileBits; ++b) s.push_back(b);  // pad with low bits
        std::sort(s.begin(), s.end());
        sets.push_back(s);
    }
    return sets;
}

static uint64_t set_mask(const std::vector<int> &s) {
    uint64_t m = 0;
    for (int b : s) m |= 1ull << b;
    return m;
}

static uint32_t to_local(const std::vector<int> &s, uint64_t phys) {
    uint32_t m = 0;
    for (int k = 0; k < (int)s.size(); ++k)
        if ((phys >> s[k]) & 1) m |= 1u << k;
    return m;
}

static std::vector<PassPlan> cut_passes(const std::vector<Token> &toks, const std::vector<std::vector<int>> &sets,
                                        bool expect_at_end) {
    std::vector<PassPlan> out;
    size_t pos = 0;
    uint64_t pending = 0;
    int cur_layer = -1;
    // Each qubit is rotated by the set that owns it: set 0 owns its 12 bits, set i > 0 owns the
    // bits it adds (its copies of bits 0..2 and padding bits only carry 128-B contiguity).
    std::vector<uint64_t> own(sets.size());
    uint64_t seen = 0;
    for (size_t i = 0; i < sets.size(); ++i) {
        own[i] = set_mask(sets[i]) & ~seen;
        seen |= set_mask(sets[i]);
    }
    auto best_set = [&](uint64_t want) {
        int best = 0, bc = -1;
        for (int i = 0; i < (int)sets.size(); ++i) {
            int c = __builtin_popcountll(want & own[i]);
            if (c > bc) { bc = c; best = i; }
        }
        return best;
    };
    while (true) {
        if (!pending) {
            if (pos >= toks.size()) break;
            const Token &t = toks[pos];
            if (t.kind == Token::ROT) { pending = t.bits; cur_layer = t.layer; ++pos; continue; }
            if (t.kind == Token::EXCHANGE) { PassPlan e; e.exchange = true; out.push_back(e); ++pos; continue; }
        }
        PassPlan pp;
        // choose the tile set
        uint64_t want = pending;
        if (!want && pos < toks.size() && toks[pos].kind == Token::PHASE && pos + 1 < toks.size() &&
            toks[pos + 1].kind == Token::ROT)
            want = toks[pos + 1].bits;
        pp.set = best_set(want);
        uint64_t sm = own[pp.set];
        uint64_t r1 = pending & sm;
        pending &= ~r1;
        pp.r1 = to_local(sets[pp.set], r1);
        pp.a1 = r1 ? cur_layer : -1;
        if (!pending && pos < toks.size() && toks[pos].kind == Token::PHASE) {
            pp.phase = toks[pos].layer;
            ++pos;
            if (pos < toks.size() && toks[pos].kind == Token::ROT) {
                uint64_t r2 = toks[pos].bits & sm;
                pending = toks[pos].bits & ~r2;
                cur_layer = toks[pos].layer;
                pp.r2 = to_local(sets[pp.set], r2);
                pp.a2 = r2 ? cur_layer : -1;
                ++pos;
            }
        }
        out.push_back(pp);
    }
    if (expect_at_end && !out.empty() && !out.back().exchange) out.back().expect = true;
    return out;
}

// ---------------------------------------------------------------------------------------------
// Permuted-layout schedule (single shard).
//
// An in-place pass over a strided tile set reads AND writes 128-B rows scattered over the whole
// state (measured 7.1-8.6 ms per 16-GiB pass vs 5.35 ms for the contiguous set).  Here every pass
// instead writes its tile out of place as one contiguous 64-KiB block (tile bits -> physical bits
// 0..11, in order) and reorders the non-tile bit runs so that the qubits the next pass rotates
// sit in the window 12..20 (128-B rows at a 64-KiB stride: the cheapest strided read).  The
// state therefore lives in a permuted layout (physical bit -> logical qubit) that the plan
// records; bits 0..2 never move.  Passes are cut greedily from the same token stream as
// cut_passes: each pass rotates every pending qubit its tile holds, applies the next phase as soon
// as the current layer is complete and then starts the next layer on the same tile.
// ---------------------------------------------------------------------------------------------
static std::vector<int> window_bits(int w) {
    std::vector<int> t = {0, 1, 2};
    for (int b = w; b < w + 9; ++b) t.push_back(b);
    if (w == 3) t.resize(kTileBits);
    return t;
}

static std::vector<PassPlan> perm_passes(int L, int p, std::vector<int> *final_layout) {
    std::vector<PassPlan> out;
    std::vector<int> lay(L);
    for (int b = 0; b < L; ++b) lay[b] = b;
    const uint64_t all = (1ull << L) - 1;
    uint64_t pending = 0;
    int cur_layer = -1, next_phase = 0;
    std::vector<int> T(kTileBits);
    for (int k = 0; k < kTileBits; ++k) T[k] = k;
    auto logical_mask = [&](const std::vector<int> &ly, const std::vector<int> &bits) {
        uint64_t m = 0;
        for (int b : bits) m |= 1ull << ly[b];
        return m;
    };
    auto local_mask = [&](uint64_t lm) {
        uint32_t m = 0;
        for (int k = 0; k < kTileBits; ++k)
            if ((lm >> lay[T[k]]) & 1) m |= 1u << k;
        return m;
    };
    for (int guard = 0; guard < 64 * (p + 1); ++guard) {
        PassPlan pp;
        pp.permuted = true;
        pp.tbits = T;
        pp.lay_in = lay;
        const uint64_t tl = logical_mask(lay, T);
        const uint64_t r1 = pending & tl;
        pending &= ~r1;
        pp.r1 = local_mask(r1);
        pp.a1 = r1 ? cur_layer : -1;
        if (!pending && next_phase < p) {
            pp.phase = next_phase;
            cur_layer = next_phase++;
            uint64_t r2 = all & tl;
            // a phase pass leaves the three row bits (always tile bits) to the next pass of the
            // layer: layer boundaries keep the compiled X Y | P | Y X shape, and the first pass
            // (write-only, compute-bound) drops its W group (P | X Y)
            if (all & ~tl) r2 &= ~7ull;
            pending = all & ~r2;
            pp.r2 = local_mask(r2);
            pp.a2 = r2 ? cur_layer : -1;
        }
        const bool last = !pending && next_phase >= p;
        pp.expect = last;
        // store map: tile bits (ascending) -> 0..11; non-tile runs, split into <= 9-bit pieces,
        // placed from bit 12 upward in the order that puts the most pending qubits in 12..20
        std::vector<int> obit(L, -1);
        for (int k = 0; k < kTileBits; ++k) obit[T[k]] = k;
        std::vector<std::pair<int, int>> pieces;  // (lo, w)
        {
            int b = 0;
            while (b < L) {
                if (obit[b] >= 0) { ++b; continue; }
                int st = b;
                while (b < L && obit[b] < 0 && b - st < 9) ++b;
                pieces.push_back({st, b - st});
            }
        }
        std::vector<int> order(pieces.size());
        for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
        std::vector<int> best_obit, best_lay;
        int best_score = -1;
        const bool enumerate = pieces.size() <= 6;
        do {
            std::vector<int> ob = obit;
            int pos = kTileBits;
            for (int i : order)
                for (int j = 0; j < pieces[i].second; ++j) ob[pieces[i].first + j] = pos++;
            if (tile_tma_dims(T.data(), L, ob.data()) > 5) continue;
            std::vector<int> nl(L);
            for (int b = 0; b < L; ++b) nl[ob[b]] = lay[b];
            int score = 0;
            for (int b = kTileBits; b < std::min(L, kTileBits + 9); ++b) score += (pending >> nl[b]) & 1;
            if (score > best_score) {
                best_score = score;
                best_obit = ob;
                best_lay = nl;
            }
        } while (enumerate && std::next_permutation(order.begin(), order.end()));
        if (best_score < 0) {  // no order fits 5 TMA dims: keep the runs in place
            best_obit = obit;
            int pos = kTileBits;
            for (auto &pc : pieces)
                for (int j = 0; j < pc.second; ++j) best_obit[pc.first + j] = pos++;
            best_lay.assign(L, 0);
            for (int b = 0; b < L; ++b) best_lay[best_obit[b]] = lay[b];
        }
        pp.obit = best_obit;
        out.push_back(pp);
        lay = best_lay;
        if (last) break;
        // next tile: the 9-bit window (or the contiguous set) holding the most pending qubits
        int best_w = 12, bc = -1;
        for (int w = 3; w + 9 <= L; ++w) {
            if (w > 3 && w < 12) continue;  // windows must not overlap the tile just written
            int c = 0;
            for (int b : window_bits(w)) c += (pending >> lay[b]) & 1;
            if (c > bc || (c == bc && w == 12)) { bc = c; best_w = w; }
        }
        T = window_bits(best_w);
    }
    if (final_layout) *final_layout = lay;
    return out;
}

// tokens of a full evolution over the local bits [0, L) with G shards (g = log2 G global bits)
static std::vector<Token> evolve_tokens(int L, int g, int p) {
    std::vector<Token> t;
    uint64_t all = (L >= 64) ? ~0ull : ((1ull << L) - 1);
    uint64_t H = 0;
    for (int b = L - g; b < L; ++b) H |= 1ull << b;
    for (int k = 0; k < p; ++k) {
        if (g > 0 && k > 0) t.push_back({Token::ROT, H, k - 1});
        t.push_back({Token::PHASE, 0, k});
        t.push_back({Token::ROT, all, k});
        if (g > 0) t.push_back({Token::EXCHANGE, 0, -1});
    }
    if (g > 0 && p > 0) t.push_back({Token::ROT, H, p - 1});
    return t;
}

static std::vector<Token> mixer_tokens(int L, int g) {
    std::vector<Token> t;
    uint64_t all = (1ull << L) - 1;
    t.push_back({Token::ROT, all, 0});
    if (g > 0) {
        uint64_t H = 0;
        for (int b = L - g; b < L; ++b) H |= 1ull << b;
        t.push_back({Token::EXCHANGE, 0, -1});
        t.push_back({Token::ROT, H, 0});
    }
    return t;
}

// Register groups (tile-local bits).  Every rotated tile bit belongs to
// exactly one group: 3..7 -> X, 8..11 -> Y, 0..2 -> W.  Lanes 0-2 of X and Y address tile bits
// 0..2 (128-B contiguous global stores); W's lanes 0-2 address bits 3..5.  Under SWIZZLE_128B
// both choices make every 8-lane phase of a 16-byte smem access conflict-free.
static const TileGroup kGroups[kMaxGroups] = {
    {{3, 4, 5, 6, 7}, {0, 1, 2, 8, 9, 10, 11}},   // X
    {{8, 9, 10, 11, 3}, {0, 1, 2, 4, 5, 6, 7}},   // Y
    {{0, 1, 2, 6, 7}, {3, 4, 5, 8, 9, 10, 11}},   // W
    {{6, 7, 8, 9, 10}, {0, 1, 2, 3, 4, 5, 11}},   // V (parity pair terms; kernels_tile.cu dev_ebit)
    {{1, 2, 3, 10, 11}, {0, 4, 5, 6, 7, 8, 9}},   // Z
};
static int group_of_bit(int b) { return b >= 8 ? 1 : (b >= 3 ? 0 : 2); }
static int ebit_index(int g, int b) {
    for (int j = 0; j < kGroupBits; ++j)
        if (kGroups[g].ebit[j] == b) return j;
    return -1;
}

// Step list of one pass: R1 (angle slot 0), optional phase, R2 (slot 1), optional expectation,
// over the fewest group changes.  pref_gq: preferred q group (reuse of an existing q copy).
static void build_steps(const PassPlan &pp, TilePassParams &tp, int pref_gq, bool half1, bool half2) {
    int m1[kMaxGroups] = {0, 0, 0}, m2[kMaxGroups] = {0, 0, 0};
    for (int b = 0; b < kTileBits; ++b) {
        int g = group_of_bit(b), j = ebit_index(g, b);
        if ((pp.r1 >> b) & 1) m1[g] |= 1 << j;
        if ((pp.r2 >> b) & 1) m2[g] |= 1 << j;
    }
    std::vector<int> G1, G2;
    for (int g = 0; g < kMaxGroups; ++g) {
        if (m1[g]) G1.push_back(g);
        if (m2[g]) G2.push_back(g);
    }
    const bool phase = pp.phase >= 0, expect = pp.expect;
    std::vector<PassStep> best;
    int best_gq = -1;
    double best_cost = 1e30;
    std::vector<int> o1 = G1;
    std::sort(o1.begin(), o1.end());
    do {
        std::vector<int> o2 = G2;
        std::sort(o2.begin(), o2.end());
        do {
            for (int gp_choice = 0; gp_choice < 3; ++gp_choice) {  // X-mixer passes use groups X, Y, W
                std::vector<PassStep> st;
                for (int g : o1) {
                    st.push_back({(int8_t)g, (int8_t)m1[g], 0, 0});
                    if (half1) st.push_back({(int8_t)g, (int8_t)m1[g], 0, 0});  // two half-angle steps
                }
                int gp = -1;
                if (phase) {
                    if (!st.empty()) gp = st.back().group;
                    else if (!o2.empty()) gp = o2.front();
                    else gp = gp_choice;
                    if (!st.empty()) st.back().phase = 1;
                    else st.push_back({(int8_t)gp, 0, 0, 1});
                } else if (gp_choice) {
                    continue;
                }
                for (int g : o2) {
                    st.push_back({(int8_t)g, (int8_t)m2[g], 1, 0});
                    if (half2) st.push_back({(int8_t)g, (int8_t)m2[g], 1, 0});
                }
                if (st.empty()) st.push_back({(int8_t)(expect && pref_gq >= 0 ? pref_gq : 0), 0, 0, 0});
                int gq = phase ? gp : (expect ? st.back().group : -1);
                if (expect && phase && st.back().group != gp) st.push_back({(int8_t)gp, 0, 0, 0});
                double cost = 0.0;
                for (size_t i = 1; i < st.size(); ++i) cost += st[i].group != st[i - 1].group;
                if (st.back().group == 2) cost += 0.25;      // W: 16-B (not 128-B) store runs per lane group
                if (gq >= 0 && pref_gq >= 0 && gq != pref_gq) cost += 0.5;  // would need another q copy
                if (cost < best_cost) {
                    best_cost = cost;
                    best = st;
                    best_gq = gq;
                }
            }
        } while (std::next_permutation(o2.begin(), o2.end()));
    } while (std::next_permutation(o1.begin(), o1.end()));
    tp.n_groups = kMaxGroups;
    for (int g = 0; g < kMaxGroups; ++g) tp.groups[g] = kGroups[g];
    tp.n_steps = (int)best.size();
    for (int i = 0; i < tp.n_steps; ++i) tp.steps[i] = best[i];
    tp.gq = best_gq;
    const TileGroup &gf = kGroups[best.back().group];
    for (int j = 0; j < kGroupBits; ++j) tp.st_estr[j] = 1ull << tp.tile_bits[gf.ebit[j]];
    for (int j = 0; j < kCT_BITS; ++j) tp.st_tphys[j] = tp.tile_bits[gf.tbit[j]];
}

// Step list of a parity window pass: the host-planned steps; q is consumed in the group of the
// phase step (first step) or, for the expectation, the last step (build_parity_plan makes them one)
static void build_parity_steps(const PassPlan &pp, TilePassParams &tp) {
    tp.n_groups = kMaxGroups;
    for (int g = 0; g < kMaxGroups; ++g) tp.groups[g] = kGroups[g];
    tp.n_steps = (int)pp.psteps.size();
    for (int i = 0; i < tp.n_steps; ++i) tp.steps[i] = pp.psteps[i];
    tp.gq = -1;
    for (int i = 0; i < tp.n_steps; ++i)
        if (tp.steps[i].phase) tp.gq = tp.steps[i].group;
    if (pp.expect) tp.gq = tp.steps[tp.n_steps - 1].group;
    const TileGroup &gf = kGroups[tp.steps[tp.n_steps - 1].group];
    for (int j = 0; j < kGroupBits; ++j) tp.st_estr[j] = 1ull << tp.tile_bits[gf.ebit[j]];
    for (int j = 0; j < kCT_BITS; ++j) tp.st_tphys[j] = tp.tile_bits[gf.tbit[j]];
}

// the compile-time program (kTileProgs) whose shape equals this pass, or 0 (generic)
static int match_prog(const TilePassParams &tp) {
    for (int q = 1; q < kNumTileProgs; ++q) {
        const TileProg &D = kTileProgs[q];
        if (D.n != tp.n_steps || D.expect != (tp.expect != 0)) continue;
        // programs 5, 6 start from |+> without a load; the QAOAz programs take either
        if (q < kFirstParityProg && (q == 5 || q == 6) != (tp.init == 1)) continue;
        // only the QAOAz programs apply pair terms, and they take no rotations
        bool pairs = false;
        for (int k = 0; k < tp.n_steps; ++k) pairs |= tp.steps[k].npair != 0;
        if (pairs != (q >= kFirstParityProg)) continue;
        bool ok = true;
        for (int k = 0; k < D.n && ok; ++k) {
            const PassStep &st = tp.steps[k];
            ok = st.group == D.g[k] && (st.phase != 0) == (k == D.phase_k) && (D.rot[k] || st.mask == 0);
        }
        if (ok) return q;
    }
    return 0;
}

}  // namespace qva

using namespace qva;

// ---------------------------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------------------------
struct KernelStat {
    double ms = 0.0;
    int64_t launches = 0;
    double bytes = 0.0;
};
struct PendingEvent {
    cudaEvent_t a, b;
    int cls;
    double bytes;
};

struct qva_plan {
    qva_plan_desc d{};
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    uint64_t N = 0;
    int mixer = 0;
    int world = 1, rank = 0, vshards = 1, G = 1, gbits = 0;
    bool replicated = false;
    uint64_t local_n = 0, offset = 0;   // partition of this rank (global indices)
    int n = -1, L = -1;                 // qubits; local bits per shard
    uint64_t arr_n = 0;                 // elements held by this process
    double2 *psi = nullptr, *psi_alt = nullptr, *psi0 = nullptr;
    double *q = nullptr, *qB = nullptr;
    bool q_set = false, qB_valid = false, has_psi0 = false;
    // compact integer quality codes (q integer-valued in a small range)
    int q_mode = 0;                    // 0 fp64, 1 int8, 2 int16
    int qmin = 0, qmax = 0;
    void *qc = nullptr, *qcB = nullptr;
    size_t qc_cap = 0, qcB_cap = 0;   // their sizes (reused across uploads: no free / malloc per q)
    bool qcB_valid = false;
    bool q_classified = false;
    double2 *d_tab = nullptr;
    size_t tab_cap = 0;
    double *d_gam = nullptr;
    size_t gam_cap = 0;
    // q permuted into the consumer order of (layout, tile set, register group): see
    // qt_gather_kernel.  Rebuilt lazily after every change of q.
    struct QtEntry {
        std::vector<int> key;  // (sharded layout, tile bits, permuted layout)
        int group, qbytes;
        void *buf;
        size_t bytes;
    };
    std::vector<QtEntry> qt_cache;
    int layout = 0;
    // MaxCut graph of qva_set_qualities_maxcut: q_x = -cut_w(x) is generated inside the tile passes
    // from per-tile records; the fp64 vector q is materialised
    // on demand only (q_dev_valid)
    bool q_graph = false, q_dev_valid = true;
    int g_m = 0;
    bool g_unit = true;
    std::vector<int> g_u, g_v;
    std::vector<double> g_w;
    // ex-QAOA (R25): during one tile-path evolution, the per-layer phase weights
    // gamma_{i,e} w_e ([p][g_m], host); phase passes then use records of those weights
    const double *ex_w = nullptr;
    // fused peer-store exchange (world > 1): both state buffers of every rank, IPC-mapped
    // (index 0: the buffer that was psi at creation, 1: psi_alt); d_bar: barrier word
    bool ipc_ok = false;
    double2 *ipc_own[2] = {nullptr, nullptr};
    double2 *ipc_peer[2][kMaxPeers] = {};
    int *d_bar = nullptr;
    unsigned long long *d_ctr = nullptr;  // per-pass tile claim counters (dynamic tile order)
    int ctr_cap = 0;
    double *q_ex = nullptr;                // step path: per-layer generated term sum
    void *d_ex_edges = nullptr;            // step path: u, v, per-layer weights
    size_t ex_edge_cap = 0;
    struct GenEntry {
        std::vector<int> key;
        int group, mode;
        int wset = -1;                     // -1: the plan's weights; i: ex-QAOA layer i
        std::vector<double> wsig;          // ex-QAOA: the weights the records were built from
        void *rec, *thr, *G;
        size_t rec_bytes;
        std::vector<double> thr_h, G_h;   // host staging (kept alive with the entry)
        std::vector<int> thr_hi, G_hi;
        void *codes = nullptr;             // consumer-order uint8 codes built from the records (lazily)
        int64_t born = 0;                  // run_passes call that created the entry
    };
    int64_t pass_seq = 0;                  // run_passes calls so far (code copies: reused q only)
    std::vector<GenEntry> gen_cache;
    // device buffers of dropped q copies / records, reused by size (a new q every step must not
    // pay cudaFree's device synchronisation and cudaMalloc's mapping cost)
    std::vector<std::pair<size_t, void *>> pool;
    // CUDA graphs of the single-shard evolution: one per (p, buffers,
    // q generation, half-angle pattern); capture staging and per-graph upload offsets
    struct GraphEntry {
        std::vector<int64_t> key;
        cudaGraphExec_t exec;
        int64_t kernels;                   // kernel launches per replay
        unsigned char *stage;
        size_t off[3];
        int n_up;
        double2 *psi_after, *alt_after;
    };
    std::vector<GraphEntry> graphs;
    std::vector<int64_t> graph_warm_key;
    unsigned char *graph_stage = nullptr;
    size_t graph_pos = 0, graph_cap = 0;
    std::vector<size_t> graph_offs;
    bool graph_capture_dirty = false;     // a graph-referenced buffer was dropped during capture
    int64_t q_gen_id = 0;                 // bumped whenever q copies / records are dropped
    double2 *d_mult = nullptr;
    size_t mult_cap = 0;
    void *d_edges = nullptr;              // on-demand q generation: edge list
    size_t edge_cap = 0;
    void *d_gen_edges = nullptr;          // generator records: classified edge lists
    size_t gen_edge_cap = 0;
    void *scratch = nullptr;              // scratch_get
    size_t scratch_cap = 0;
    double2 *small_batch = nullptr;       // batched small-state evolutions
    size_t small_batch_cap = 0;
    // pinned host ring for small per-step uploads (angles, tables, generator records): a copy from
    // pageable memory would synchronise the stream before it starts
    unsigned char *ring = nullptr;
    size_t ring_size = 0, ring_pos = 0;
    // permuted layout of the single-shard state (physical bit -> logical qubit); empty = natural
    std::vector<int> perm;
    std::map<int, std::pair<std::vector<PassPlan>, std::vector<int>>> perm_sched;  // p -> (passes, final layout)
    struct TmEntry {
        CUtensorMap in, out;
        int dim_src[5], dim_w[5], member_dim;
    };
    std::map<std::vector<int64_t>, TmEntry> tmap_cache;
    bool perm_failed = false;
    double *partials = nullptr;
    uint64_t partials_n = 0;
    double *red = nullptr;             // [max_batch][2]
    PassAngles *d_angles = nullptr;
    size_t angles_cap = 0;
    double *d_thetas = nullptr;
    size_t thetas_cap = 0;
    int *d_flag = nullptr;
    int max_batch = 1;
    double2 *batch_psi = nullptr;
    std::vector<std::vector<int>> sets;
    // circulant
    FftPlan *fft = nullptr;
    int fft_M1 = 0, fft_M2 = 0;   // four-step split (sharded transposes)
    void *xfer = nullptr;         // NCCL staging buffer of the sharded circulant path
    double *lambda_perm = nullptr;
    bool lam_set = false, lam_const = false;
    double lam0 = 0.0, lamc = 0.0;
    std::vector<double> lambda_host;   // natural (forward-bin) order mirror
    // parity (QAOAz): ordered qubit subsequence
    std::vector<int> parity_seq;
    std::vector<ParityWindow> parity_win;  // window passes of the current sequence (built lazily)
    std::vector<int> parity_win_seq;       // the sequence they were built for
    std::map<int, std::vector<PassPlan>> parity_tile_sched;  // tile-pass schedule per p (parity_tile_passes)
    std::vector<int> parity_tile_seq;      // the sequence it was built for
    bool parity_tile_ran = false;          // the last parity evolution ran as tile passes
    std::vector<ParityItem> parity_shard_items;           // sharded QAOAz schedule (one layer)
    std::vector<std::vector<PassStep>> parity_shard_steps;  // its window step lists
    std::vector<int> parity_shard_seq;
    // sparse
    SparseMixer sm;
    bool sparse_set = false;
    // collectives of a world > 1 plan: the NCCL communicator, or the caller's host transport
    // (qva_plan_create_ex); see "multi-process collectives" below
    ncclComm_t comm = nullptr;
    bool host_tp = false;
    qva_transport tp = {};
    bool created = false;                 // qva_plan_create completed (collective teardown allowed)
    double xfer_bytes = 0.0;              // state bytes one shard sent to the other shards since the
                                          // last stats reset (NVLink traffic of a real shard)
    // profiling
    bool prof = false;
    KernelStat stats[kKernelClasses];
    std::vector<PendingEvent> pending;
    std::vector<cudaEvent_t> event_pool;
    int64_t launches = 0;
    bool expect_valid = false;
    double expect_val = 0.0, norm_val = 0.0;
};

namespace {

cudaEvent_t get_event(qva_plan *P) {
    if (!P->event_pool.empty()) {
        cudaEvent_t e = P->event_pool.back();
        P->event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

struct ProfScope {
    qva_plan *P;
    int cls;
    double bytes;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    ProfScope(qva_plan *P_, int cls_, double bytes_, int64_t nlaunch = 1, cudaStream_t st_ = nullptr)
        : P(P_), cls(cls_), bytes(bytes_), st(st_ ? st_ : P_->stream) {
        P->launches += nlaunch;
        if (P->prof) {
            a = get_event(P);
            b = get_event(P);
            cudaEventRecord(a, st);
        }
    }
    ~ProfScope() {
        if (P->prof) {
            cudaEventRecord(b, st);
            P->pending.push_back({a, b, cls, bytes});
        }
    }
};

struct PlanObserver : LaunchObserver {
    qva_plan *P;
    std::vector<ProfScope *> stack;
    explicit PlanObserver(qva_plan *P_) : P(P_) {}
    void begin(int cls, double bytes, cudaStream_t st = nullptr) override {
        stack.push_back(new ProfScope(P, cls, bytes, 1, st));
    }
    void count(int cls, double bytes) override {
        P->launches += 1;
        if (P->prof) {
            P->stats[cls].launches += 1;
            P->stats[cls].bytes += bytes;
        }
    }
    void end() override {
        delete stack.back();
        stack.pop_back();
    }
};

qva_status harvest(qva_plan *P) {
    for (auto &pe : P->pending) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, pe.a, pe.b);
        if (g_trace) fprintf(stderr, "[qva] class %d %.3f ms %.3f GB\n", pe.cls, ms, pe.bytes * 1e-9);
        P->stats[pe.cls].ms += ms;
        P->stats[pe.cls].launches += 1;
        P->stats[pe.cls].bytes += pe.bytes;
        P->event_pool.push_back(pe.a);
        P->event_pool.push_back(pe.b);
    }
    P->pending.clear();
    return QVA_OK;
}

qva_status sync(qva_plan *P) {
    QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
    harvest(P);
    return QVA_OK;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

bool is_pow2(uint64_t x) { return x && !(x & (x - 1)); }
int ilog2(uint64_t x) {
    int r = 0;
    while ((1ull << r) < x) ++r;
    return r;
}

// Every captured CUDA graph bakes in the raw addresses of the plan's scratch buffers
// (partials, angle records, phase tables, claim counters, q copies / records).  Any path that
// frees or recycles one of them first drops the graphs (a replay after a grow would
// read and write freed memory).  A drop during a capture marks the capture dirty; it is then
// discarded and the passes run uncaptured.
void invalidate_graphs(qva_plan *P) {
    if (P->graph_stage) {
        P->graph_capture_dirty = true;
        return;
    }
    if (!P->graphs.empty()) {
        cudaStreamSynchronize(P->stream);  // a replay in flight still reads its staging block
        for (auto &g : P->graphs) {
            cudaGraphExecDestroy(g.exec);
            cudaFreeHost(g.stage);
        }
        P->graphs.clear();
    }
    P->graph_warm_key.clear();
}
// cudaFree of a plan-owned buffer that a captured graph may reference
void plan_free(qva_plan *P, void *p) {
    if (!p) return;
    invalidate_graphs(P);
    cudaFree(p);
}

qva_status ensure_partials(qva_plan *P, uint64_t n) {
    if (P->partials_n >= n) return QVA_OK;
    plan_free(P, P->partials);
    P->partials = nullptr;
    QVA_CUDA_TRY(cudaMalloc(&P->partials, n * 2 * sizeof(double)));
    P->partials_n = n;
    return QVA_OK;
}

qva_status ensure_angles(qva_plan *P, size_t n) {
    if (P->angles_cap >= n) return QVA_OK;
    plan_free(P, P->d_angles);
    P->d_angles = nullptr;
    QVA_CUDA_TRY(cudaMalloc(&P->d_angles, n * sizeof(PassAngles)));
    P->angles_cap = n;
    return QVA_OK;
}

qva_status check_theta(const double *theta, size_t n) {
    for (size_t i = 0; i < n; ++i)
        if (!std::isfinite(theta[i])) {
            set_error("non-finite theta");
            return QVA_ERR_NUMERIC;
        }
    return QVA_OK;
}

// ---- multi-process collectives (world > 1) -------------------------------------------------------
// Every collective of a multi-process plan goes through these four calls.  NCCL runs them on the
// plan's stream (stream-ordered with the kernels around them); a host transport (qva_transport,
// include/qva.h) runs them on host buffers after synchronising the stream.
enum { kCollSum = 0, kCollMax = 1, kCollMin = 2 };

qva_status tp_check(int rc, const char *what) {
    if (rc == 0) return QVA_OK;
    set_error(std::string("host transport ") + what + " failed (" + std::to_string(rc) + ")");
    return QVA_ERR_NCCL;
}
cudaError_t scratch_get(qva_plan *P, void **p, size_t bytes);

// element-wise reduction of n host doubles over ranks, in place.  NCCL stages through `dev` (n
// doubles of device memory; NULL -> the plan's scratch) with stream-ordered copies.
qva_status coll_allreduce_host(qva_plan *P, double *vals, int n, int op, double *dev = nullptr) {
    if (P->world == 1 || n <= 0) return QVA_OK;
    if (P->host_tp) return tp_check(P->tp.allreduce_f64(P->tp.ctx, vals, (uint64_t)n, op), "allreduce");
    double *d = dev;
    if (!d) QVA_CUDA_TRY(scratch_get(P, (void **)&d, n * sizeof(double)));
    const ncclRedOp_t nop = op == kCollMax ? ncclMax : (op == kCollMin ? ncclMin : ncclSum);
    QVA_CUDA_TRY(cudaMemcpyAsync(d, vals, n * sizeof(double), cudaMemcpyHostToDevice, P->stream));
    QVA_NCCL_TRY(ncclAllReduce(d, d, n, ncclDouble, nop, P->comm, P->stream));
    QVA_CUDA_TRY(cudaMemcpyAsync(vals, d, n * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
    return QVA_OK;
}

// all-gather of `bytes` host bytes per rank into out[world * bytes] (rank-major).  NCCL stages
// through `dev` ((world + 1) * bytes of device memory).  Every copy is on the plan's stream, so
// the staging is ordered before the collective (a synchronous cudaMemcpy on the legacy
// stream is not ordered with a non-blocking stream's NCCL kernel).
qva_status coll_allgather_host(qva_plan *P, const void *in, void *out, size_t bytes, unsigned char *dev) {
    if (P->host_tp) return tp_check(P->tp.allgather(P->tp.ctx, in, out, bytes), "allgather");
    QVA_CUDA_TRY(cudaMemcpyAsync(dev, in, bytes, cudaMemcpyHostToDevice, P->stream));
    QVA_NCCL_TRY(ncclAllGather(dev, dev + bytes, bytes, ncclChar, P->comm, P->stream));
    QVA_CUDA_TRY(cudaMemcpyAsync(out, dev + bytes, bytes * P->world, cudaMemcpyDeviceToHost, P->stream));
    QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
    return QVA_OK;
}

// barrier ordered after this rank's stream work: once it completes on every rank, every rank's
// kernels enqueued before it (e.g. stores into our buffers over peer memory, which end with
// __threadfence_system) are done.  NCCL: a one-word all-reduce on the stream (no host wait); host
// transport: synchronise the stream, then a one-value all-reduce.
qva_status coll_stream_barrier(qva_plan *P) {
    if (P->world == 1) return QVA_OK;
    if (P->host_tp) {
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        double z = 0.0;
        return tp_check(P->tp.allreduce_f64(P->tp.ctx, &z, 1, kCollSum), "barrier");
    }
    QVA_CUDA_TRY(cudaMemsetAsync(P->d_bar, 0, sizeof(int), P->stream));
    QVA_NCCL_TRY(ncclAllReduce(P->d_bar, P->d_bar, 1, ncclInt32, ncclSum, P->comm, P->stream));
    return QVA_OK;
}

// all-to-all of device chunks: chunk t of src (chunk_bytes each) goes to rank t, chunk s of dst
// comes from rank s; our own chunk is a local copy.  NCCL: grouped send/recv on the stream.  Host
// transport: the whole src through host memory (fallback / tests only).
qva_status coll_alltoall_dev(qva_plan *P, const void *src, void *dst, size_t chunk_bytes) {
    const char *s = (const char *)src;
    char *d = (char *)dst;
    if (P->host_tp) {
        std::vector<char> hs(chunk_bytes * P->world), hr(chunk_bytes * P->world);
        QVA_CUDA_TRY(cudaMemcpyAsync(hs.data(), s, hs.size(), cudaMemcpyDeviceToHost, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        QVA_TRY(tp_check(P->tp.alltoall(P->tp.ctx, hs.data(), hr.data(), chunk_bytes), "alltoall"));
        QVA_CUDA_TRY(cudaMemcpyAsync(d, hr.data(), hr.size(), cudaMemcpyHostToDevice, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        return QVA_OK;
    }
    QVA_NCCL_TRY(ncclGroupStart());
    for (int t = 0; t < P->world; ++t) {
        if (t == P->rank) continue;
        QVA_NCCL_TRY(ncclSend(s + t * chunk_bytes, chunk_bytes, ncclChar, t, P->comm, P->stream));
        QVA_NCCL_TRY(ncclRecv(d + t * chunk_bytes, chunk_bytes, ncclChar, t, P->comm, P->stream));
    }
    QVA_NCCL_TRY(ncclGroupEnd());
    QVA_CUDA_TRY(cudaMemcpyAsync(d + P->rank * chunk_bytes, s + P->rank * chunk_bytes, chunk_bytes,
                                 cudaMemcpyDeviceToDevice, P->stream));
    return QVA_OK;
}

// ---- exchange (global <-> local qubit swap; COMM-psi) ----------------------
// Every shard r sends chunk t (local index top-g bits = t) to shard t, which stores it as its
// chunk r: a block transpose of the G x G chunk matrix.  The layout flips between A and B.
// all-gather of equal device slices: rank r's `bytes` at src land at dst + r * bytes (NCCL on the
// stream; host transport through host memory)
qva_status coll_allgather_dev(qva_plan *P, const void *src, void *dst, size_t bytes) {
    if (P->host_tp) {
        std::vector<char> hs(bytes), hr(bytes * P->world);
        QVA_CUDA_TRY(cudaMemcpyAsync(hs.data(), src, bytes, cudaMemcpyDeviceToHost, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        QVA_TRY(tp_check(P->tp.allgather(P->tp.ctx, hs.data(), hr.data(), bytes), "allgather"));
        QVA_CUDA_TRY(cudaMemcpyAsync(dst, hr.data(), hr.size(), cudaMemcpyHostToDevice, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        return QVA_OK;
    }
    QVA_NCCL_TRY(ncclAllGather(src, dst, bytes, ncclChar, P->comm, P->stream));
    return QVA_OK;
}

// in-place sum over ranks of n device doubles (NCCL on the stream; host transport via host memory)
qva_status coll_allreduce_dev(qva_plan *P, double *dev, int n) {
    if (P->world == 1) return QVA_OK;
    if (P->host_tp) {
        std::vector<double> h(n);
        QVA_CUDA_TRY(cudaMemcpyAsync(h.data(), dev, n * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        QVA_TRY(tp_check(P->tp.allreduce_f64(P->tp.ctx, h.data(), (uint64_t)n, kCollSum), "allreduce"));
        QVA_CUDA_TRY(cudaMemcpyAsync(dev, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, P->stream));
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));
        return QVA_OK;
    }
    QVA_NCCL_TRY(ncclAllReduce(dev, dev, n, ncclDouble, ncclSum, P->comm, P->stream));
    return QVA_OK;
}
struct PlanCompleteComm : CompleteComm {
    qva_plan *P;
    explicit PlanCompleteComm(qva_plan *P_) : P(P_) {}
    qva_status sum2_dev(double *dev2) override { return coll_allreduce_dev(P, dev2, 2); }
};

// collectives of the row-partitioned sparse mixer (SparseComm, kernels_sparse.cu)
struct PlanSparseComm : SparseComm {
    qva_plan *P;
    explicit PlanSparseComm(qva_plan *P_) : P(P_) {}
    qva_status max2(double *v) override { return coll_allreduce_host(P, v, 2, kCollMax); }
    qva_status gather(const double2 *local, double2 *all, uint64_t stride) override {
        return coll_allgather_dev(P, local, all, stride * sizeof(double2));
    }
};

// cross-shard traffic of one all-to-all of `elem_bytes`-byte elements over the whole (local) array:
// each shard keeps 1/G of its slice and sends the rest, (G-1)/G x slice bytes
void count_xfer(qva_plan *P, double elem_bytes) {
    if (P->G <= 1) return;
    const double slice = (double)P->arr_n / (P->world == 1 ? P->G : 1) * elem_bytes;
    P->xfer_bytes += slice * (P->G - 1) / P->G;
}

template <typename T>
qva_status exchange_buffers(qva_plan *P, T *src, T *dst) {
    uint64_t per_shard = 1ull << P->L;
    uint64_t C = per_shard / P->G;
    count_xfer(P, sizeof(T));
    if (P->world == 1) {
        ProfScope ps(P, K_EXCHANGE, 2.0 * sizeof(T) * (double)P->arr_n);
        QVA_CUDA_TRY(launch_chunk_transpose<T>(dst, src, P->G, C, P->stream));
        return QVA_OK;
    }
    ProfScope ps(P, K_EXCHANGE, 2.0 * sizeof(T) * (double)P->arr_n);
    // chunk t (top local bits = t) goes to rank t, where it becomes chunk `rank` (qva_exchange_plan)
    return coll_alltoall_dev(P, src, dst, C * sizeof(T));
}

qva_status ensure_q_dev(qva_plan *P);
qva_status ensure_q_alloc(qva_plan *P);
qva_status exchange_state(qva_plan *P) {
    QVA_TRY(exchange_buffers<double2>(P, P->psi, P->psi_alt));
    std::swap(P->psi, P->psi_alt);
    P->layout ^= 1;
    return QVA_OK;
}

qva_status ensure_qB(qva_plan *P) {
    if (P->G == 1) return QVA_OK;
    if (!P->qB_valid) {
        QVA_TRY(ensure_q_dev(P));
        if (!P->qB) QVA_CUDA_TRY(cudaMalloc(&P->qB, P->arr_n * sizeof(double)));
        QVA_TRY(exchange_buffers<double>(P, P->q, P->qB));
        P->qB_valid = true;
    }
    if (P->q_mode && !P->qcB_valid) {
        int eb = P->q_mode == 1 ? 1 : 2;
        if (P->qcB_cap < P->arr_n * eb) {
            plan_free(P, P->qcB);
            P->qcB = nullptr;
            P->qcB_cap = 0;
            QVA_CUDA_TRY(cudaMalloc(&P->qcB, P->arr_n * eb));
            P->qcB_cap = P->arr_n * eb;
        }
        uint64_t C = (1ull << P->L) / P->G;
        if (P->world == 1) {
            ProfScope ps(P, K_EXCHANGE, 2.0 * eb * (double)P->arr_n);
            QVA_CUDA_TRY(launch_chunk_transpose_bytes(P->qcB, P->qc, P->G, C, eb, P->stream));
        } else {
            ProfScope ps(P, K_EXCHANGE, 2.0 * eb * (double)P->arr_n);
            QVA_TRY(coll_alltoall_dev(P, P->qc, P->qcB, C * eb));
        }
        P->qcB_valid = true;
    }
    return QVA_OK;
}

// Classify q after an upload: integer-valued within int8/int16 range -> compact codes + phase
// tables (exact: the table entry for k is the same fp64 sincos of fl(gamma*k)).
void drop_qt(qva_plan *P);
qva_status ensure_q_dev(qva_plan *P);
cudaError_t scratch_get(qva_plan *P, void **p, size_t bytes);
static double host_ms();
static int hostprof_env() {
    static int v = [] {
        const char *e = getenv("QVA_HOSTPROF");
        return e ? atoi(e) : 0;
    }();
    return v;
}
qva_status classify_q(qva_plan *P) {
    const double h0 = hostprof_env() ? host_ms() : 0.0;
    drop_qt(P);
    P->q_mode = 0;
    P->qcB_valid = false;
    if ((P->mixer != QVA_MIXER_X && P->mixer != QVA_MIXER_PARITY) || P->L < kTileBits) return QVA_OK;
    QVA_TRY(ensure_q_dev(P));
    int blocks = q_range_blocks(P->arr_n);
    double *mm = nullptr;
    QVA_CUDA_TRY(scratch_get(P, (void **)&mm, 2 * blocks * sizeof(double)));
    QVA_CUDA_TRY(cudaMemsetAsync(P->d_flag, 0, sizeof(int), P->stream));
    {
        ProfScope ps(P, K_OTHER, 8.0 * P->arr_n);
        QVA_CUDA_TRY(launch_q_range(P->q, P->arr_n, P->d_flag, mm, blocks, P->stream));
    }
    std::vector<double> h(2 * blocks);
    int flag = 0;
    QVA_CUDA_TRY(cudaMemcpyAsync(h.data(), mm, h.size() * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    QVA_CUDA_TRY(cudaMemcpyAsync(&flag, P->d_flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    QVA_TRY(sync(P));
    double lo = INFINITY, hi = -INFINITY;
    for (int b = 0; b < blocks; ++b) {
        lo = std::min(lo, h[2 * b]);
        hi = std::max(hi, h[2 * b + 1]);
    }
    if (P->world > 1) {
        double v[3] = {(double)flag, -lo, hi};
        QVA_TRY(coll_allreduce_host(P, v, 3, kCollMax));
        flag = v[0] != 0.0;
        lo = -v[1];
        hi = v[2];
    }
    if (flag || !(hi - lo <= 4095.0)) return QVA_OK;
    int eb = 0;
    if (lo >= -128 && hi <= 127) eb = 1;
    else if (lo >= -32768 && hi <= 32767) eb = 2;
    if (!eb) return QVA_OK;
    if (P->qc_cap < P->arr_n * eb) {
        plan_free(P, P->qc);
        P->qc = nullptr;
        P->qc_cap = 0;
        QVA_CUDA_TRY(cudaMalloc(&P->qc, P->arr_n * eb));
        P->qc_cap = P->arr_n * eb;
    }
    {
        ProfScope ps(P, K_OTHER, (8.0 + eb) * P->arr_n);
        QVA_CUDA_TRY(launch_q_encode(P->q, P->arr_n, P->qc, eb, P->stream));
    }
    P->q_mode = eb == 1 ? 1 : 2;
    P->qmin = (int)lo;
    P->qmax = (int)hi;
    qva_status st = sync(P);
    if (hostprof_env()) fprintf(stderr, "[qva] classify_q %.2f ms (host, incl. sync)\n", host_ms() - h0);
    return st;
}

qva_status to_natural_perm(qva_plan *P);
qva_status to_layout_A(qva_plan *P) {
    QVA_TRY(to_natural_perm(P));
    if (P->layout == 0) return QVA_OK;
    return exchange_state(P);
}

void pool_put(qva_plan *P, void *p, size_t bytes) {
    if (!p) return;
    invalidate_graphs(P);  // the buffer may be handed to another use by pool_get
    P->pool.push_back({bytes, p});
}
// smallest pooled buffer of at least `bytes` (exact-size reuse is the common case), else cudaMalloc
cudaError_t pool_get(qva_plan *P, void **p, size_t bytes) {
    int best = -1;
    for (int i = 0; i < (int)P->pool.size(); ++i)
        if (P->pool[i].first >= bytes && (best < 0 || P->pool[i].first < P->pool[best].first)) best = i;
    if (best >= 0 && P->pool[best].first <= 2 * bytes + 4096) {
        *p = P->pool[best].second;
        P->pool.erase(P->pool.begin() + best);
        return cudaSuccess;
    }
    return cudaMalloc(p, bytes);
}

// H2D copy of a small host buffer through the pinned ring (falls back to a pageable copy when
// larger than the ring); the ring restarts after a stream synchronisation when full
constexpr size_t kRingBytes = 4 << 20;
qva_status upload(qva_plan *P, void *dst, const void *src, size_t bytes) {
    if (!bytes) return QVA_OK;
    if (P->graph_stage) {  // graph capture: the copy node reads this fixed pinned slot on every replay
        const size_t off = (P->graph_pos + 15) & ~(size_t)15;
        if (off + bytes > P->graph_cap) {
            set_error("internal: graph staging overflow");
            return QVA_ERR_INVALID_ARGUMENT;
        }
        memcpy(P->graph_stage + off, src, bytes);
        QVA_CUDA_TRY(cudaMemcpyAsync(dst, P->graph_stage + off, bytes, cudaMemcpyHostToDevice, P->stream));
        P->graph_offs.push_back(off);
        P->graph_pos = off + bytes;
        return QVA_OK;
    }
    if (!P->ring) {
        if (cudaMallocHost((void **)&P->ring, kRingBytes) != cudaSuccess) {
            cudaGetLastError();
            P->ring = nullptr;
        } else {
            P->ring_size = kRingBytes;
        }
    }
    if (!P->ring || bytes > P->ring_size) {
        QVA_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, P->stream));
        return QVA_OK;
    }
    const size_t off = (P->ring_pos + 15) & ~(size_t)15;
    if (off + bytes > P->ring_size) {
        QVA_CUDA_TRY(cudaStreamSynchronize(P->stream));  // earlier copies out of the ring are done
        P->ring_pos = 0;
        return upload(P, dst, src, bytes);
    }
    memcpy(P->ring + off, src, bytes);
    QVA_CUDA_TRY(cudaMemcpyAsync(dst, P->ring + off, bytes, cudaMemcpyHostToDevice, P->stream));
    P->ring_pos = off + bytes;
    return QVA_OK;
}

// persistent device scratch for short-lived buffers of one call (each use completes before the
// call returns); stream-ordered allocation measured host stalls of up to 100+ ms per call
cudaError_t scratch_get(qva_plan *P, void **p, size_t bytes) {
    if (P->scratch_cap < bytes) {
        plan_free(P, P->scratch);
        P->scratch = nullptr;
        P->scratch_cap = 0;
        cudaError_t e = cudaMalloc(&P->scratch, bytes);
        if (e != cudaSuccess) return e;
        P->scratch_cap = bytes;
    }
    *p = P->scratch;
    return cudaSuccess;
}

void drop_qt(qva_plan *P) {
    ++P->q_gen_id;
    for (auto &e : P->qt_cache) pool_put(P, e.buf, e.bytes);
    P->qt_cache.clear();
    for (auto &e : P->gen_cache) {
        pool_put(P, e.rec, e.rec_bytes);
        pool_put(P, e.thr, 128 * 8 * sizeof(double));
        pool_put(P, e.G, 32 * sizeof(double));
        pool_put(P, e.codes, P->arr_n);
    }
    P->gen_cache.clear();
}

// q (8 B per amplitude) is allocated on first use: a max-cut plan on the tile path never needs
// it, which is what lets an n = 33 state (128 GiB) fit one GPU without a 64 GiB q beside it
qva_status ensure_q_alloc(qva_plan *P) {
    if (P->q) return QVA_OK;
    if (cudaMalloc(&P->q, P->arr_n * sizeof(double)) != cudaSuccess) {
        cudaGetLastError();
        set_error("cudaMalloc of the quality vector (" + std::to_string(P->arr_n * sizeof(double)) + " bytes) failed");
        return QVA_ERR_OUT_OF_MEMORY;
    }
    QVA_CUDA_TRY(cudaMemsetAsync(P->q, 0, P->arr_n * sizeof(double), P->stream));
    return QVA_OK;
}

// fp64 q of a graph-defined plan, generated on demand (maxcut_q_kernel, 8 B per amplitude); the
// edge list goes through the pinned upload ring into a persistent buffer, and the stream orders
// the kernel before every consumer (no host synchronisation)
qva_status ensure_q_dev(qva_plan *P) {
    QVA_TRY(ensure_q_alloc(P));
    if (!P->q_graph || P->q_dev_valid) return QVA_OK;
    const int m = P->g_m;
    const size_t need = (size_t)std::max(m, 1) * (2 * sizeof(int32_t) + sizeof(double));
    if (P->edge_cap < need) {
        plan_free(P, P->d_edges);
        P->d_edges = nullptr;
        QVA_CUDA_TRY(cudaMalloc(&P->d_edges, need));
        P->edge_cap = need;
    }
    int32_t *du = reinterpret_cast<int32_t *>(P->d_edges);
    int32_t *dv = du + std::max(m, 1);
    double *dw = reinterpret_cast<double *>(reinterpret_cast<unsigned char *>(P->d_edges) +
                                            (size_t)std::max(m, 1) * 2 * sizeof(int32_t));
    if (m) {
        QVA_TRY(upload(P, du, P->g_u.data(), m * sizeof(int32_t)));
        QVA_TRY(upload(P, dv, P->g_v.data(), m * sizeof(int32_t)));
        if (!P->g_unit) QVA_TRY(upload(P, dw, P->g_w.data(), m * sizeof(double)));
    }
    {
        ProfScope ps(P, K_OTHER, 8.0 * P->arr_n);
        QVA_CUDA_TRY(launch_maxcut_q(P->q, P->arr_n, P->offset, m, du, dv, P->g_unit ? nullptr : dw, P->stream));
    }
    P->q_dev_valid = true;
    return QVA_OK;
}

// physical -> logical bit map as runs (nullptr / empty: identity over n bits)
LayoutRuns layout_runs(const std::vector<int> *lay, int n) {
    LayoutRuns R;
    memset(&R, 0, sizeof(R));
    if (!lay || lay->empty()) {
        R.n = 1;
        R.src[0] = 0;
        R.w[0] = (int8_t)n;
        R.dst[0] = 0;
        return R;
    }
    const std::vector<int> &l = *lay;
    int b = 0;
    while (b < (int)l.size()) {
        int st = b++;
        while (b < (int)l.size() && l[b] == l[b - 1] + 1) ++b;
        if (R.n < kMaxLayoutRuns) {
            R.src[R.n] = (int8_t)st;
            R.w[R.n] = (int8_t)(b - st);
            R.dst[R.n] = (int8_t)l[st];
        }
        ++R.n;
    }
    // bits above the layout (batch members) map to themselves
    if (n > (int)l.size() && R.n < kMaxLayoutRuns) {
        R.src[R.n] = R.dst[R.n] = (int8_t)l.size();
        R.w[R.n] = (int8_t)(n - (int)l.size());
        ++R.n;
    }
    return R;
}

// q in the consumer order of group g for the pass tiles described by tp (tile bits + runs) and
// the permuted layout lay (nullptr: natural / sharded layout P->layout)
qva_status ensure_qt(qva_plan *P, const std::vector<int> &key, const std::vector<int> *lay, int g, int qbytes,
                     const TilePassParams &tp, void **out) {
    for (auto &e : P->qt_cache)
        if (e.key == key && e.group == g && e.qbytes == qbytes) {
            *out = e.buf;
            return QVA_OK;
        }
    const void *src;
    if (qbytes == 8) src = (P->layout == 1) ? (const void *)P->qB : (const void *)P->q;
    else src = (P->layout == 1) ? P->qcB : P->qc;
    const LayoutRuns R = layout_runs(lay, ilog2(P->arr_n));
    if (R.n > kMaxLayoutRuns) {
        set_error("internal: permuted layout has too many runs");
        return QVA_ERR_UNSUPPORTED;
    }
    void *buf = nullptr;
    QVA_CUDA_TRY(pool_get(P, &buf, P->arr_n * (size_t)qbytes));
    {
        ProfScope ps(P, K_OTHER, 2.0 * qbytes * (double)P->arr_n);
        QVA_CUDA_TRY(
            launch_qt_gather(buf, src, qbytes, tp, kGroups[g], P->arr_n >> kTileBits, P->qmin, R, P->stream));
    }
    P->qt_cache.push_back({key, g, qbytes, buf, P->arr_n * (size_t)qbytes});
    *out = buf;
    return QVA_OK;
}

// return a permuted single-shard state to the natural layout (one gather pass; outside the
// evolution, e.g. before get_state or a step-level call)
qva_status to_natural_perm(qva_plan *P) {
    if (P->perm.empty()) return QVA_OK;
    bool ident = true;
    for (size_t b = 0; b < P->perm.size(); ++b) ident &= P->perm[b] == (int)b;
    if (!ident) {
        if (!P->psi_alt) QVA_CUDA_TRY(cudaMalloc(&P->psi_alt, P->arr_n * sizeof(double2)));
        const LayoutRuns R = layout_runs(&P->perm, ilog2(P->arr_n));
        ProfScope ps(P, K_OTHER, 32.0 * P->arr_n);
        QVA_CUDA_TRY(launch_permute_copy(P->psi_alt, P->psi, P->arr_n, R, P->stream));
        std::swap(P->psi, P->psi_alt);
    }
    P->perm.clear();
    return QVA_OK;
}

// ---- generated MaxCut qualities ---------------------------
constexpr int kGenIntMaxEdges = 4000;  // integer path: cut in [0, m], phase table of m + 1 entries
constexpr int kGenF64MinQubits = 26;   // weighted graphs, large batches: generate q from 2^26 amplitudes
constexpr int kGfMembersHost = 24;     // = kGfMembers (kernels_tile.cu): factorised weighted phase

bool use_qgen(const qva_plan *P) {
    static int env = [] {
        const char *e = getenv("QVA_QGEN");
        return e ? atoi(e) : 1;
    }();
    return env != 0 && P->q_graph && (P->mixer == QVA_MIXER_X || P->mixer == QVA_MIXER_PARITY);
}

// q path of a tile-pass sequence: generated integer / fp64 records, or 0 (stored q)
int qgen_mode(const qva_plan *P, int batch) {
    const bool gen_int = P->g_unit && P->g_m <= kGenIntMaxEdges && !P->ex_w;  // ex weights are real
    const bool f64_ok = batch <= kGfMembersHost || P->L >= kGenF64MinQubits || P->d.reserved[1] != 0;
    return use_qgen(P) && (gen_int || f64_ok) ? (gen_int ? kQGenInt : kQGenF64) : 0;
}

// unit-weight generated q read as consumer-order uint8 codes (m <= 255) built once per q and pass
// shape from the records, instead of assembling cut(x) per element in every pass (QVA_QGEN_CODES=0:
// in-pass generation); single members (batches keep the in-pass generator: one code copy would serve
// them too, but their passes are compute-bound, not memory-bound)
bool gen_codes_mode(const qva_plan *P, int gen, int batch) {
    static int env = [] {
        const char *e = getenv("QVA_QGEN_CODES");
        return e ? atoi(e) : 1;
    }();
    return env != 0 && gen == kQGenInt && P->g_m <= 255 && batch == 1;
}

// logical qubit of every physical bit of the arrays a pass reads (n_phys bits) and the logical
// bits that are constant on this process (global qubits of a real shard = its rank bits)
void pass_layout(const qva_plan *P, const PassPlan &pp, int n_phys, std::vector<int> &lay, uint64_t &cmask,
                 uint64_t &cval) {
    lay.resize(n_phys);
    for (int b = 0; b < n_phys; ++b) lay[b] = b;
    cmask = cval = 0;
    if (pp.permuted) {
        for (int b = 0; b < (int)pp.lay_in.size() && b < n_phys; ++b) lay[b] = pp.lay_in[b];
        return;
    }
    if (P->G <= 1) return;
    const int L = P->L, g = P->gbits;
    if (P->world == 1) {  // virtual shards: the shard index is the top physical bits
        if (P->layout == 1)
            for (int i = 0; i < g; ++i) {
                lay[L - g + i] = L + i;
                lay[L + i] = L - g + i;
            }
        return;
    }
    if (P->layout == 0) {
        for (int i = 0; i < g; ++i) cmask |= 1ull << (L + i);
        cval = (uint64_t)P->rank << L;
    } else {
        for (int i = 0; i < g; ++i) lay[L - g + i] = L + i;
        for (int i = 0; i < g; ++i) cmask |= 1ull << (L - g + i);
        cval = (uint64_t)P->rank << (L - g);
    }
}

// per-tile records + per-thread constants of the generated q for one pass shape (cached)
qva_status ensure_gen(qva_plan *P, const std::vector<int> &qkey, const PassPlan &pp, int n_phys, int gq, int mode,
                      const TilePassParams &tp, int wset, const qva_plan::GenEntry **out) {
    // wset >= 0: ex-QAOA layer wset, whose weights change with theta (entries are rebuilt when
    // they differ; stream order makes reusing the buffers safe)
    const double *wts = (wset >= 0 && P->ex_w) ? P->ex_w + (size_t)wset * P->g_m : nullptr;
    for (size_t i = 0; i < P->gen_cache.size(); ++i) {
        auto &e = P->gen_cache[i];
        if (e.key == qkey && e.group == gq && e.mode == mode && e.wset == (wts ? wset : -1)) {
            if (!wts || std::equal(e.wsig.begin(), e.wsig.end(), wts)) {
                *out = &e;
                return QVA_OK;
            }
            pool_put(P, e.rec, e.rec_bytes);
            pool_put(P, e.thr, 128 * 8 * sizeof(double));
            pool_put(P, e.G, 32 * sizeof(double));
            pool_put(P, e.codes, P->arr_n);
            P->gen_cache.erase(P->gen_cache.begin() + i);
            break;
        }
    }
    std::vector<int> lay;
    uint64_t cmask, cval;
    pass_layout(P, pp, n_phys, lay, cmask, cval);
    // tile-local bit k -> logical; tile-number bit -> logical
    int tl[kTileBits];
    std::vector<int> in_tile(64, -1);
    for (int k = 0; k < kTileBits; ++k) {
        tl[k] = lay[tp.tile_bits[k]];
        in_tile[tl[k]] = k;
    }
    std::vector<int> tbit_log;
    for (int r = 0; r < tp.n_runs; ++r)
        for (int j = 0; j < tp.run_w[r]; ++j) {
            const int tb = tp.run_src[r] + j;
            if ((int)tbit_log.size() <= tb) tbit_log.resize(tb + 1, -1);
            tbit_log[tb] = lay[tp.run_dst[r] + j];
        }
    GenPrep gp;
    memset(&gp, 0, sizeof(gp));
    {
        int b = 0;
        while (b < (int)tbit_log.size()) {
            int st = b++;
            while (b < (int)tbit_log.size() && tbit_log[b] == tbit_log[b - 1] + 1) ++b;
            if (gp.tmap.n == kMaxLayoutRuns) {
                set_error("internal: tile-number map has too many runs");
                return QVA_ERR_UNSUPPORTED;
            }
            gp.tmap.src[gp.tmap.n] = (int8_t)st;
            gp.tmap.w[gp.tmap.n] = (int8_t)(b - st);
            gp.tmap.dst[gp.tmap.n] = (int8_t)tbit_log[st];
            ++gp.tmap.n;
        }
    }
    gp.const_val = cval;
    gp.w_unit = (P->g_unit && !wts) ? 1 : 0;
    // classify the edges (self-loops never cut)
    std::vector<int2> tt, tb;
    std::vector<double> ttw, tbw;
    struct TileEdge {
        int a, b;
        double w;
    };
    std::vector<TileEdge> te;
    for (int e = 0; e < P->g_m; ++e) {
        const int u = P->g_u[e], v = P->g_v[e];
        if (u == v) continue;
        const double w = wts ? wts[e] : (P->g_unit ? 1.0 : P->g_w[e]);
        const int ku = in_tile[u], kv = in_tile[v];
        if (ku < 0 && kv < 0) {
            tt.push_back(make_int2(u, v));
            ttw.push_back(w);
        } else if (ku >= 0 && kv >= 0) {
            te.push_back({ku, kv, w});
        } else {
            tb.push_back(ku >= 0 ? make_int2(ku, v) : make_int2(kv, u));
            tbw.push_back(w);
        }
    }
    (void)cmask;
    gp.n_tt = (int)tt.size();
    gp.n_tb = (int)tb.size();
    const bool f64 = mode == kQGenF64;
    const uint64_t n_tiles = P->arr_n >> kTileBits;
    const size_t rec_bytes = f64 ? 112 : 16;
    qva_plan::GenEntry ent;
    ent.key = qkey;
    ent.group = gq;
    ent.mode = mode;
    ent.wset = wts ? wset : -1;
    if (wts) ent.wsig.assign(wts, wts + P->g_m);
    ent.rec = ent.thr = ent.G = nullptr;
    ent.born = P->pass_seq;
    ent.rec_bytes = n_tiles * rec_bytes;
    QVA_CUDA_TRY(pool_get(P, &ent.rec, ent.rec_bytes));
    QVA_CUDA_TRY(pool_get(P, &ent.thr, 128 * 8 * sizeof(double)));
    QVA_CUDA_TRY(pool_get(P, &ent.G, 32 * sizeof(double)));
    const size_t eb = (tt.size() + tb.size()) * (sizeof(int2) + sizeof(double)) + 16;
    if (P->gen_edge_cap < eb) {  // stream order keeps one staging buffer safe across entries
        plan_free(P, P->d_gen_edges);
        P->d_gen_edges = nullptr;
        QVA_CUDA_TRY(cudaMalloc(&P->d_gen_edges, eb));
        P->gen_edge_cap = eb;
    }
    void *d_edges = P->d_gen_edges;
    {
        std::vector<unsigned char> hb(eb, 0);
        size_t off = 0;
        auto put = [&](const void *src, size_t n) {
            memcpy(hb.data() + off, src, n);
            off += n;
        };
        put(tt.data(), tt.size() * sizeof(int2));
        put(tb.data(), tb.size() * sizeof(int2));
        const size_t woff = off;
        put(ttw.data(), ttw.size() * sizeof(double));
        put(tbw.data(), tbw.size() * sizeof(double));
        unsigned char *d = (unsigned char *)d_edges;
        gp.tt_uv = (const int2 *)d;
        gp.tb_ab = (const int2 *)(d + tt.size() * sizeof(int2));
        gp.tt_w = (const double *)(d + woff);
        gp.tb_w = (const double *)(d + woff + ttw.size() * sizeof(double));
        QVA_TRY(upload(P, d_edges, hb.data(), eb));
        ProfScope ps(P, K_OTHER, (double)n_tiles * rec_bytes);
        QVA_CUDA_TRY(launch_gen_records(ent.rec, n_tiles, f64 ? 1 : 0, gp, P->stream));
        // host per-thread constants of group gq: C(c), beta_j(c), and G(e)
        const TileGroup &g = kGroups[gq];
        int role[kTileBits], ridx[kTileBits];  // 0: thread bit, 1: register bit
        for (int j = 0; j < kCT_BITS; ++j) role[g.tbit[j]] = 0, ridx[g.tbit[j]] = j;
        for (int j = 0; j < kGroupBits; ++j) role[g.ebit[j]] = 1, ridx[g.ebit[j]] = j;
        std::vector<double> &thr = ent.thr_h, &G = ent.G_h;
        std::vector<int> &thr_i = ent.thr_hi, &G_i = ent.G_hi;
        thr.assign(128 * 8, 0.0);
        G.assign(32, 0.0);
        thr_i.assign(128 * 8, 0);
        G_i.assign(32, 0);
        for (int c = 0; c < 128; ++c) {
            double C = 0.0, beta[kGroupBits] = {0, 0, 0, 0, 0};
            auto xv = [&](int k) { return (c >> ridx[k]) & 1; };
            for (const TileEdge &x : te) {
                if (role[x.a] == 0 && role[x.b] == 0) {
                    C += x.w * (double)(xv(x.a) ^ xv(x.b));
                } else if (role[x.a] != role[x.b]) {
                    const int h = role[x.a] == 0 ? x.a : x.b, e = role[x.a] == 0 ? x.b : x.a;
                    C += x.w * xv(h);
                    beta[ridx[e]] += x.w * (1.0 - 2.0 * xv(h));
                }
            }
            thr[c * 8] = C;
            thr_i[c * 8] = (int)C;
            for (int j = 0; j < kGroupBits; ++j) {
                thr[c * 8 + 1 + j] = beta[j];
                thr_i[c * 8 + 1 + j] = (int)beta[j];
            }
        }
        for (int e = 0; e < 32; ++e) {
            double s = 0.0;
            for (const TileEdge &x : te)
                if (role[x.a] == 1 && role[x.b] == 1) s += x.w * (double)(((e >> ridx[x.a]) ^ (e >> ridx[x.b])) & 1);
            G[e] = s;
            G_i[e] = (int)s;
        }
        if (f64) {
            QVA_TRY(upload(P, ent.thr, thr.data(), thr.size() * sizeof(double)));
            QVA_TRY(upload(P, ent.G, G.data(), G.size() * sizeof(double)));
        } else {
            QVA_TRY(upload(P, ent.thr, thr_i.data(), thr_i.size() * sizeof(int)));
            QVA_TRY(upload(P, ent.G, G_i.data(), G_i.size() * sizeof(int)));
        }
    }
    P->gen_cache.push_back(ent);
    *out = &P->gen_cache.back();
    return QVA_OK;
}

// ---- tile-pass execution of a pass list -----------------------------------------------------
// thetas: [batch][2p]; psi_base/stride: states of the batch members
// Host data of one pass sequence for one theta set: per-pass angle records, half-angle flags,
// phase-table rows (gammas + deferred scalar factors) and which passes apply the carried scale.
// The structure (flags) decides the step programs; the values are what a replayed graph uploads.
struct PassHostData {
    std::vector<PassAngles> ang;
    std::vector<char> half1, half2, apply_scale;
    std::vector<double> gam;
    std::vector<double2> tab_mult;
    std::vector<int> tab_index;
};
static void pass_host_data(const std::vector<PassPlan> &passes, const double *thetas, int p, int batch,
                           bool int_table, int n_tile_passes, PassHostData &H, bool fold_gf = false) {
    std::vector<PassAngles> &ang = H.ang;
    ang.assign((size_t)n_tile_passes * batch, PassAngles{});
    std::vector<char> &half1 = H.half1, &half2 = H.half2;
    half1.assign(n_tile_passes, 0);
    half2.assign(n_tile_passes, 0);
    {
        int j = 0;
        for (const PassPlan &pp : passes) {
            if (pp.exchange) continue;
            for (int b = 0; b < batch; ++b) {
                const double *th = thetas + (size_t)b * 2 * p;
                if (pp.a1 >= 0 && fabs(cos(th[2 * pp.a1 + 1])) < 0x1p-10) half1[j] = 1;
                if (pp.a2 >= 0 && fabs(cos(th[2 * pp.a2 + 1])) < 0x1p-10) half2[j] = 1;
            }
            ++j;
        }
    }
    std::vector<double> &gam = H.gam;  // [phase pass][batch]
    gam.clear();
    std::vector<int> &tab_index = H.tab_index;
    tab_index.assign(passes.size(), -1);
    {
        int j = 0, np = 0;
        for (size_t pi = 0; pi < passes.size(); ++pi) {
            const PassPlan &pp = passes[pi];
            if (pp.exchange) continue;
            if (pp.phase >= 0 && int_table) tab_index[pi] = np++;
            int n1 = __builtin_popcount(pp.r1), n2 = __builtin_popcount(pp.r2);
            for (int b = 0; b < batch; ++b) {
                const double *th = thetas + (size_t)b * 2 * p;
                PassAngles &a = ang[(size_t)j * batch + b];
                memset(&a, 0, sizeof(a));
                double sr = 1.0, si = 0.0;  // accumulated dropped factor
                // factored rotation: t = tan(beta), dropped factor cos(beta) per rotated qubit;
                // |cos beta| < 2^-10: two steps of beta/2 (for every member of the slot)
                auto factor = [&](int layer, int count, bool half, double &t) {
                    double beta = th[2 * layer + 1];
                    if (half) beta *= 0.5;
                    const double c = cos(beta);
                    t = sin(beta) / c;
                    for (int k = 0; k < (half ? 2 : 1) * count; ++k) sr *= c;
                };
                if (pp.a1 >= 0) factor(pp.a1, n1, half1[j], a.t1);
                if (pp.a2 >= 0) factor(pp.a2, n2, half2[j], a.t2);
                if (pp.parity && pp.play >= 0) {  // Givens pair terms: cos 2t, sin 2t (R19)
                    a.t1 = cos(2.0 * th[2 * pp.play + 1]);
                    a.t2 = sin(2.0 * th[2 * pp.play + 1]);
                }
                a.scale = make_double2(sr, si);
                if (pp.phase >= 0) {
                    a.gamma = th[2 * pp.phase];
                    if (int_table) gam.push_back(a.gamma);
                }
            }
            ++j;
        }
    }
    // The dropped rotation factors are scalars per member, so they commute with every pass: carry
    // them forward and fold them into the next integer phase table (free) or apply them at the
    // next fp64 phase / the last pass, instead of a complex multiply per amplitude in every pass.
    std::vector<char> &apply_scale = H.apply_scale;
    apply_scale.assign(n_tile_passes, 0);
    std::vector<double2> &tab_mult = H.tab_mult;  // [phase table row][batch]
    tab_mult.clear();
    {
        std::vector<double2> carry(batch, make_double2(1.0, 0.0));
        int j = 0;
        for (size_t pi = 0; pi < passes.size(); ++pi) {
            const PassPlan &pp = passes[pi];
            if (pp.exchange) continue;
            const bool last = (j == n_tile_passes - 1);
            const bool fold_tab = pp.phase >= 0 && int_table;
            const bool fold_here = (pp.phase >= 0 && !int_table) || last;
            // factorised fp64 generated phase: the factor rides on the per-member G table (free)
            const bool into_gf = fold_gf && pp.phase >= 0 && !int_table;
            for (int b = 0; b < batch; ++b) {
                PassAngles &a = ang[(size_t)j * batch + b];
                const double2 f = a.scale, c = carry[b];
                carry[b] = make_double2(c.x * f.x - c.y * f.y, c.x * f.y + c.y * f.x);
                if (fold_tab) tab_mult.push_back(carry[b]);
                if (fold_here) a.scale = carry[b];
                if (fold_tab || fold_here) carry[b] = make_double2(1.0, 0.0);
            }
            apply_scale[j] = into_gf ? 2 : (fold_here ? 1 : 0);
            ++j;
        }
    }
}

static int g_hostprof = [] {
    const char *e = getenv("QVA_HOSTPROF");
    return e ? atoi(e) : 0;
}();
static double host_ms() {
    timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

qva_status run_passes(qva_plan *P, const std::vector<PassPlan> &passes, const double *thetas, int p, int batch,
                      double2 *psi_base, uint64_t stride, int init_mode, double *expect_out /*[batch][2] host*/) {
    ++P->pass_seq;
    const double hp0 = g_hostprof ? host_ms() : 0.0;
    double hp_first = -1.0;
    int n_tile_passes = 0;
    for (auto &pp : passes) n_tile_passes += !pp.exchange;
    // graph-defined q: generated inside the passes (integer table path for unit weights)
    // (weighted graphs: the factorised phase needs a per-member G table, held in smem for batches
    // <= kGfMembers (cfg2: 1.17 vs 1.63 ms stored); larger batches pay one sincos per amplitude
    // plus the record arithmetic, which only pays where HBM bounds the pass)
    const int gen = qgen_mode(P, batch);
    if (!gen && P->q_set && !P->q_classified) {
        QVA_TRY(classify_q(P));
        P->q_classified = true;
    }
    const bool int_table = gen == kQGenInt || (!gen && P->q_mode != 0);
    const int tab_qmin = gen == kQGenInt ? -P->g_m : P->qmin;
    QVA_TRY(ensure_angles(P, (size_t)n_tile_passes * batch));
    PassHostData H;
    pass_host_data(passes, thetas, p, batch, int_table, n_tile_passes, H,
                   gen == kQGenF64 && batch <= kGfMembersHost);
    const std::vector<PassAngles> &ang = H.ang;
    const std::vector<char> &half1 = H.half1, &half2 = H.half2, &apply_scale = H.apply_scale;
    const std::vector<double> &gam = H.gam;
    const std::vector<double2> &tab_mult = H.tab_mult;
    const std::vector<int> &tab_index = H.tab_index;
    QVA_TRY(upload(P, P->d_angles, ang.data(), ang.size() * sizeof(PassAngles)));
    const int ntab = gen == kQGenInt ? P->g_m + 1 : (int_table ? (P->qmax - P->qmin + 1) : 0);
    if (!gam.empty()) {
        if (P->gam_cap < gam.size()) {
            plan_free(P, P->d_gam);
            P->d_gam = nullptr;
            QVA_CUDA_TRY(cudaMalloc(&P->d_gam, gam.size() * sizeof(double)));
            P->gam_cap = gam.size();
        }
        if (P->tab_cap < gam.size() * ntab) {
            plan_free(P, P->d_tab);
            P->d_tab = nullptr;
            QVA_CUDA_TRY(cudaMalloc(&P->d_tab, gam.size() * ntab * sizeof(double2)));
            P->tab_cap = gam.size() * ntab;
        }
        QVA_TRY(upload(P, P->d_gam, gam.data(), gam.size() * sizeof(double)));
        if (P->mult_cap < gam.size()) {
            plan_free(P, P->d_mult);
            P->d_mult = nullptr;
            QVA_CUDA_TRY(cudaMalloc(&P->d_mult, gam.size() * sizeof(double2)));
            P->mult_cap = gam.size();
        }
        QVA_TRY(upload(P, P->d_mult, tab_mult.data(), gam.size() * sizeof(double2)));
        {
            ProfScope ps(P, K_OTHER, 16.0 * gam.size() * ntab);
            QVA_CUDA_TRY(launch_phase_table(P->d_tab, P->d_gam, P->d_mult, (int)gam.size(), tab_qmin, ntab, P->stream));
        }
    }
    uint64_t n_tiles = P->arr_n >> kTileBits;
    bool any_expect = false;
    for (auto &pp : passes) any_expect |= pp.expect;
    const int grid = tile_pass_grid(n_tiles * (uint64_t)batch);
    const int nslot = grid * tile_consumer_warps();
    if (any_expect) QVA_TRY(ensure_partials(P, (uint64_t)nslot * batch));
    const int n_phys = ilog2(P->arr_n);
    const int qbytes = gen ? gen : (P->q_mode == 1 ? 1 : (P->q_mode == 2 ? 2 : 8));
    // dynamic tile claiming: one zeroed counter per tile pass (one memset for the sequence)
    static int g_dyn = [] {
        const char *e = getenv("QVA_DYN");
        return e ? atoi(e) : 1;
    }();
    static const bool g_dyn_all = getenv("QVA_DYN") != nullptr;  // explicit QVA_DYN: as given
    if (g_dyn) {
        if (P->ctr_cap < n_tile_passes) {
            plan_free(P, P->d_ctr);
            P->d_ctr = nullptr;
            const int cap = std::max(n_tile_passes, 64);
            QVA_CUDA_TRY(cudaMalloc(&P->d_ctr, cap * sizeof(unsigned long long)));
            P->ctr_cap = cap;
        }
        QVA_CUDA_TRY(cudaMemsetAsync(P->d_ctr, 0, n_tile_passes * sizeof(unsigned long long), P->stream));
    }
    int j = 0;
    bool first = true;
    bool exchanged = false;  // the previous pass already wrote the exchanged layout (fused exchange)
    static int g_fuse_x = [] {
        const char *e = getenv("QVA_FUSE_EXCHANGE");
        return e ? atoi(e) : 1;
    }();
    for (size_t pi = 0; pi < passes.size(); ++pi) {
        const PassPlan &pp = passes[pi];
        if (pp.exchange) {
            if (batch != 1 || psi_base != P->psi) {
                set_error("internal: exchange in batched pass list");
                return QVA_ERR_INVALID_ARGUMENT;
            }
            if (exchanged) {
                exchanged = false;
                continue;
            }
            QVA_TRY(exchange_state(P));
            psi_base = P->psi;
            continue;
        }
        // global <-> local exchange fused into the store of the pass before it (virtual shards):
        // the exchange swaps the physical bit fields [L-g, L) and [L, L+g), which the tile's TMA
        // store applies as an output bit permutation into psi_alt -- no transpose pass
        std::vector<int> xbit;
        if (g_fuse_x && !pp.permuted && batch == 1 && P->G > 1 && P->world == 1 && pi + 1 < passes.size() &&
            passes[pi + 1].exchange && P->psi_alt) {
            xbit.resize(n_phys);
            for (int b = 0; b < n_phys; ++b) xbit[b] = b;
            for (int i = 0; i < P->gbits; ++i) {
                xbit[P->L - P->gbits + i] = P->L + i;
                xbit[P->L + i] = P->L - P->gbits + i;
            }
            // the permuted store must stay one <= 5-D TMA box (else the transpose pass runs)
            if (tile_tma_dims(P->sets[pp.set].data(), n_phys, xbit.data()) > 5) xbit.clear();
        }
        // real shards: the same exchange done by stores into the receiving ranks' buffers (peer
        // memory); needs the chunk bits [L-g, L) outside the tile (they name the receiver)
        bool xpeer = false;
        const bool xvirt = P->world == 1 && P->d.reserved[3] != 0;  // test mode: virtual shards as peers
        if (xvirt) xbit.clear();
        if (g_fuse_x && (P->ipc_ok || xvirt) && !pp.permuted && batch == 1 && P->G > 1 && P->G <= kMaxPeers &&
            pi + 1 < passes.size() && passes[pi + 1].exchange) {
            xpeer = true;
            for (int k = 0; k < kTileBits; ++k)
                if (P->sets[pp.set][k] >= P->L - P->gbits) xpeer = false;
        }
        TilePassParams tp;
        memset(&tp, 0, sizeof(tp));
        const std::vector<int> &s = (pp.permuted || pp.parity) ? pp.tbits : P->sets[pp.set];
        uint64_t tmask = 0;
        for (int k = 0; k < kTileBits; ++k) {
            tp.tile_bits[k] = s[k];
            tmask |= 1ull << s[k];
        }
        // runs of non-tile physical bits: tile number bits -> physical positions
        {
            int src = 0, b = 0;
            tp.n_runs = 0;
            while (b < n_phys) {
                if ((tmask >> b) & 1) { ++b; continue; }
                int st = b;
                while (b < n_phys && !((tmask >> b) & 1)) ++b;
                if (tp.n_runs == kMaxRuns) {
                    set_error("internal: tile set leaves more than 4 runs of non-tile bits");
                    return QVA_ERR_UNSUPPORTED;
                }
                tp.run_src[tp.n_runs] = src;
                tp.run_dst[tp.n_runs] = st;
                tp.run_w[tp.n_runs] = b - st;
                tp.run_mask[tp.n_runs] = (1ull << (b - st)) - 1;
                src += b - st;
                ++tp.n_runs;
            }
        }
        tp.n_tiles = n_tiles;
        tp.log2_tiles = ilog2(n_tiles);
        tp.batch = batch;
        tp.member_stride = stride;
        tp.psi_out = psi_base;
        const double2 *psi_in = (first && init_mode == 2) ? P->psi0 : psi_base;
        tp.init = (first && init_mode == 1) ? 1 : 0;
        // permuted passes write out of place (except a first pass, whose input is not psi_base)
        const bool swap_after = (pp.permuted && !(first && init_mode != 0)) || !xbit.empty() || xpeer;
        if (swap_after) tp.psi_out = P->psi_alt;
        tp.amp0 = 1.0 / sqrt((double)P->N);
        const bool needs_q = pp.phase >= 0 || pp.expect;
        // q copies are keyed by (sharded layout, tile bits, permuted layout)
        std::vector<int> qkey = {P->layout};
        qkey.insert(qkey.end(), s.begin(), s.end());
        if (pp.permuted) qkey.insert(qkey.end(), pp.lay_in.begin(), pp.lay_in.end());
        int pref = -1;
        if (needs_q)
            for (auto &e : P->qt_cache)
                if (e.key == qkey && e.qbytes == qbytes) pref = e.group;
        if (pp.parity) build_parity_steps(pp, tp);
        else build_steps(pp, tp, pref, half1[j], half2[j]);
        int launch_qb = 0;  // q mode of this launch when it differs from the sequence's (generated codes)
        if (needs_q && gen) {
            const qva_plan::GenEntry *ge = nullptr;
            if (P->ex_w && pp.phase >= 0 && pp.expect) {
                set_error("internal: ex-QAOA phase and <Q> in one pass");
                return QVA_ERR_UNSUPPORTED;
            }
            QVA_TRY(ensure_gen(P, qkey, pp, n_phys, tp.gq, gen, tp, (P->ex_w && pp.phase >= 0) ? pp.phase : -1, &ge));
            tp.qt = ge->rec;
            // phase passes read 1-B codes built from the records (stored-code pass); an expectation-only
            // pass keeps the in-pass generator (A/B, cfg4: 5.19 vs 5.34 ms -- it is memory-bound)
            // (built only for a q that outlived the evolution that made its records: a q set anew for
            // every evaluation keeps the in-pass generator, the cheaper one when used once)
            if (pp.phase >= 0 && gen_codes_mode(P, gen, batch) && ge->born < P->pass_seq) {
                qva_plan::GenEntry *gm = const_cast<qva_plan::GenEntry *>(ge);
                if (!gm->codes && P->graph_stage) {
                    // never built inside a graph capture (the replays would rebuild them): the capture
                    // is dropped, the uncaptured rerun builds them and a later call captures the
                    // code-reading passes
                    P->graph_capture_dirty = true;
                } else {
                    if (!gm->codes) {
                        QVA_CUDA_TRY(pool_get(P, &gm->codes, P->arr_n));
                        ProfScope ps(P, K_OTHER, (double)P->arr_n);
                        QVA_CUDA_TRY(launch_gen_codes(gm->codes, gm->rec, P->arr_n >> kTileBits, gm->thr, gm->G,
                                                      kGroups[tp.gq], P->g_m, P->stream));
                    }
                    tp.qt = gm->codes;
                    launch_qb = 1;
                }
            }
            tp.gen_thr = ge->thr;
            tp.gen_G = ge->G;
            tp.gen_m = P->g_m;
            tp.qmin = tab_qmin;
            tp.ntab = ntab;
            if (tab_index[pi] >= 0) tp.tab = P->d_tab + (size_t)tab_index[pi] * batch * ntab;
        } else if (needs_q) {
            if (P->layout == 1) QVA_TRY(ensure_qB(P));
            void *qt = nullptr;
            QVA_TRY(ensure_qt(P, qkey, pp.permuted ? &pp.lay_in : nullptr, tp.gq, qbytes, tp, &qt));
            tp.qt = qt;
            tp.qmin = P->qmin;
            tp.ntab = ntab;
            if (tab_index[pi] >= 0) tp.tab = P->d_tab + (size_t)tab_index[pi] * batch * ntab;
        } else {
            tp.gq = -1;
        }
        tp.angles = P->d_angles + (size_t)j * batch;
        // claimed tiles level the SMs of the load-bound passes; the write-only first pass (no state
        // to load, uniform work per tile) keeps the static interleaved split, which spares its
        // claiming thread an atomic round trip per tile (A/B on one box, cfg4 init pass: 3.93 ->
        // 3.76 ms; QVA_DYN=1 claims in every pass)
        const bool dyn_default = g_dyn == 1 && !(tp.init == 1 && !g_dyn_all);
        tp.work_ctr = (dyn_default || (g_dyn > 1 && ((g_dyn >> 1) >> j) & 1)) ? P->d_ctr + j : nullptr;
        tp.expect = pp.expect ? 1 : 0;
        tp.partials = P->partials;
        // default 2: the thread that issued a tile's TMA store waits for its shared-memory read
        // (and refills the stage) at the warpgroup's next barrier instead of right after the
        // store, so its warp no longer arrives late at the next transpose (A/B on one box, cfg4:
        // boundary passes 6.34 -> 6.20 ms, init 3.94 -> 3.92 ms, 37.74 -> 37.46 ms per evaluation)
        static int g_tail = [] {
            const char *e = getenv("QVA_TAIL");
            return e ? atoi(e) : 2;
        }();
        tp.tail_mode = g_tail;
        tp.apply_scale = apply_scale[j] == 1 ? 1 : 0;
        tp.fold_scale_gf = apply_scale[j] == 2 ? 1 : 0;
        // last step touching shared memory: a group switch (smem transpose) or the phase (q stage)
        tp.release_step = (tp.init == 1 && tp.gq < 0) ? -1 : 0;
        for (int k = 0; k < tp.n_steps; ++k)
            if ((k > 0 && tp.steps[k].group != tp.steps[k - 1].group) || tp.steps[k].phase) tp.release_step = k;
        if (tp.expect) tp.release_step = tp.n_steps;
        const int prog = match_prog(tp);
        // tiles go back through a TMA tensor store (measured faster than st.global from registers for
        // every tile shape; env QVA_TSTORE=0 selects the register stores for comparison)
        tp.tma_store = (g_tstore >= 0) ? g_tstore : 1;
        CUtensorMap map, map_out;
        if (pp.permuted || !xbit.empty()) tp.tma_store = 1;  // the permuted store is a TMA store map
        const int *obit = pp.permuted ? pp.obit.data() : (xbit.empty() ? nullptr : xbit.data());
        if (xpeer) {
            tp.tma_store = 0;  // register stores: each tile's destination is a peer pointer
            if (xvirt) {  // shard t's buffer is psi_alt's t-th 2^L block
                for (int t = 0; t < P->G; ++t) tp.xpeer[t] = P->psi_alt + ((uint64_t)t << P->L);
                tp.xvirt = 1;
            } else {
                const int k = (P->psi_alt == P->ipc_own[0]) ? 0 : 1;  // every rank swaps in lockstep
                for (int t = 0; t < P->world; ++t) tp.xpeer[t] = P->ipc_peer[k][t];
            }
            tp.xg = P->G;
            tp.xrank = P->rank;
            tp.xshift = P->L - P->gbits;
        }
        {
            // tensor maps depend on (tile bits, store permutation, buffers, sizes): encoded once
            std::vector<int64_t> key = {(int64_t)(uintptr_t)psi_in, (int64_t)(uintptr_t)tp.psi_out, n_phys, batch};
            key.insert(key.end(), s.begin(), s.end());
            if (obit) key.insert(key.end(), obit, obit + n_phys);
            auto it = P->tmap_cache.find(key);
            if (it == P->tmap_cache.end()) {
                qva_plan::TmEntry te;
                QVA_TRY(make_tile_tensor_maps(psi_in, tp.psi_out, n_phys, batch, tp, obit, &te.in, &te.out));
                memcpy(te.dim_src, tp.dim_src, sizeof(te.dim_src));
                memcpy(te.dim_w, tp.dim_w, sizeof(te.dim_w));
                te.member_dim = tp.member_dim;
                if (P->tmap_cache.size() > 256) P->tmap_cache.clear();
                it = P->tmap_cache.emplace(std::move(key), te).first;
            }
            map = it->second.in;
            map_out = it->second.out;
            memcpy(tp.dim_src, it->second.dim_src, sizeof(tp.dim_src));
            memcpy(tp.dim_w, it->second.dim_w, sizeof(tp.dim_w));
            tp.member_dim = it->second.member_dim;
        }
        if (g_trace > 1) {
            fprintf(stderr, "[qva] pass set %d prog %d init %d gq %d expect %d release %d steps:", pp.set, prog, tp.init,
                    tp.gq, tp.expect, tp.release_step);
            for (int k = 0; k < tp.n_steps; ++k)
                fprintf(stderr, " (g%d m%02x a%d p%d)", tp.steps[k].group, tp.steps[k].mask, tp.steps[k].angle,
                        tp.steps[k].phase);
            fprintf(stderr, " dims:");
            for (int d = 0; d < 5; ++d) fprintf(stderr, " [%d,%d]", tp.dim_src[d], tp.dim_w[d]);
            fprintf(stderr, "\n");
        }
        // algorithmic bytes: the state round trip plus stored q (generated q: the per-tile records)
        const double qb = gen ? (gen == kQGenInt ? 16.0 : 112.0) / (double)(1 << kTileBits) : (double)qbytes;
        double bytes = (double)P->arr_n * batch *
                       ((tp.init == 1 ? 16.0 : 32.0) + ((pp.phase >= 0 || pp.expect) ? qb : 0.0) / batch);
        if (pp.expect)
            QVA_CUDA_TRY(cudaMemsetAsync(P->partials, 0, (size_t)nslot * batch * 2 * sizeof(double), P->stream));
        {
            ProfScope ps(P, K_TILE, bytes);
            QVA_CUDA_TRY(launch_tile_pass(map, map_out, tp, needs_q ? (launch_qb ? launch_qb : qbytes) : 0, prog, grid,
                                          P->stream));
            if (g_hostprof && hp_first < 0) hp_first = host_ms() - hp0;
        }
        first = false;
        ++j;
        if (swap_after) {
            std::swap(P->psi, P->psi_alt);
            psi_base = P->psi;
        }
        if (xpeer && !xvirt) {
            // every rank's stores into our buffer are done once every rank's pass has finished:
            // a one-word all-reduce on the stream is that barrier
            QVA_TRY(coll_stream_barrier(P));
        }
        if (!xbit.empty() || xpeer) {
            P->layout ^= 1;  // what exchange_state would have done
            exchanged = true;
            count_xfer(P, sizeof(double2) * batch);
        }
        if (pp.expect) {
            ProfScope ps(P, K_REDUCE, 16.0 * nslot * batch);
            QVA_CUDA_TRY(launch_reduce_partials(P->partials, nslot, batch, P->red, P->stream));
        }
    }
    if (expect_out) {
        QVA_CUDA_TRY(cudaMemcpyAsync(expect_out, P->red, sizeof(double) * 2 * batch, cudaMemcpyDeviceToHost,
                                     P->stream));
    }
    if (g_hostprof)
        fprintf(stderr, "[qva host] run_passes: %.3f ms to the first launch, %.3f ms total enqueue\n", hp_first,
                host_ms() - hp0);
    return QVA_OK;
}

// ---- graph replay of the single-shard evolution ------------------
// The launch sequence of an evolution depends only on (p, schedule, buffers, q copies /
// records, half-angle pattern); the theta-dependent data are three uploads (angle records,
// phase-table gammas and scalar factors).  The first call with a new key runs normally (warming
// every cache); the second captures run_passes into a CUDA graph whose copy nodes read a fixed
// pinned staging block; later calls refill that block and launch the graph: one launch per
// evaluation instead of ~10 launches and their host-side preparation.
qva_status run_passes_graph(qva_plan *P, const std::vector<PassPlan> &passes, const double *theta, int p,
                            int init_mode) {
    static int env = [] {
        const char *e = getenv("QVA_GRAPH");
        return e ? atoi(e) : 1;
    }();
    if (!env || P->prof || g_trace || g_hostprof)
        return run_passes(P, passes, theta, p, 1, P->psi, 0, init_mode, nullptr);
    int n_tile_passes = 0;
    for (auto &pp : passes) n_tile_passes += !pp.exchange;
    const int gen = qgen_mode(P, 1);
    const bool int_table = gen == kQGenInt || (!gen && P->q_mode != 0);
    PassHostData H;
    pass_host_data(passes, theta, p, 1, int_table, n_tile_passes, H, gen == kQGenF64);
    std::vector<int64_t> key = {p, (int64_t)(uintptr_t)P->psi, (int64_t)(uintptr_t)P->psi_alt, init_mode,
                                P->q_gen_id, gen, (int64_t)P->q_classified, (int64_t)P->q_mode,
                                (int64_t)(uintptr_t)&passes};
    for (int j = 0; j < n_tile_passes; ++j) key.push_back(H.half1[j] * 2 + H.half2[j]);
    const void *srcs[3] = {H.ang.data(), H.gam.data(), H.tab_mult.data()};
    const size_t sizes[3] = {H.ang.size() * sizeof(PassAngles), H.gam.size() * sizeof(double),
                             H.gam.size() * sizeof(double2)};
    for (auto &g : P->graphs)
        if (g.key == key) {
            for (int k = 0; k < g.n_up; ++k) memcpy(g.stage + g.off[k], srcs[k], sizes[k]);
            QVA_CUDA_TRY(cudaGraphLaunch(g.exec, P->stream));
            P->launches += g.kernels;
            P->psi = g.psi_after;
            P->psi_alt = g.alt_after;
            return QVA_OK;
        }
    if (key != P->graph_warm_key) {  // first call with this key: run normally, warming the caches
        P->graph_warm_key = key;
        return run_passes(P, passes, theta, p, 1, P->psi, 0, init_mode, nullptr);
    }
    // second call: capture
    qva_plan::GraphEntry g;
    g.key = key;
    const size_t cap = sizes[0] + sizes[1] + sizes[2] + 64;
    QVA_CUDA_TRY(cudaMallocHost((void **)&g.stage, cap));
    double2 *psi0 = P->psi, *alt0 = P->psi_alt;
    P->graph_stage = g.stage;
    P->graph_pos = 0;
    P->graph_cap = cap;
    P->graph_offs.clear();
    P->graph_capture_dirty = false;
    cudaGraph_t graph = nullptr;
    QVA_CUDA_TRY(cudaStreamBeginCapture(P->stream, cudaStreamCaptureModeThreadLocal));
    const int64_t launches0 = P->launches;
    qva_status st = run_passes(P, passes, theta, p, 1, P->psi, 0, init_mode, nullptr);
    cudaError_t ce = cudaStreamEndCapture(P->stream, &graph);
    P->graph_stage = nullptr;
    g.kernels = P->launches - launches0;
    P->launches = launches0;
    g.psi_after = P->psi;
    g.alt_after = P->psi_alt;
    P->psi = psi0;
    P->psi_alt = alt0;
    if (st != QVA_OK || ce != cudaSuccess || P->graph_offs.size() > 3 || P->graph_capture_dirty) {
        P->graph_capture_dirty = false;
        if (graph) cudaGraphDestroy(graph);
        cudaFreeHost(g.stage);
        cudaGetLastError();
        P->graph_warm_key.clear();
        if (st != QVA_OK) return st;
        return run_passes(P, passes, theta, p, 1, P->psi, 0, init_mode, nullptr);
    }
    g.n_up = (int)P->graph_offs.size();
    for (int k = 0; k < g.n_up; ++k) g.off[k] = P->graph_offs[k];
    ce = cudaGraphInstantiate(&g.exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
        cudaFreeHost(g.stage);
        set_error(std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ce));
        return QVA_ERR_CUDA;
    }
    if (P->graphs.size() >= 8) {
        cudaGraphExecDestroy(P->graphs.front().exec);
        cudaFreeHost(P->graphs.front().stage);
        P->graphs.erase(P->graphs.begin());
    }
    P->graphs.push_back(g);
    QVA_CUDA_TRY(cudaGraphLaunch(g.exec, P->stream));
    P->launches += g.kernels;
    P->psi = g.psi_after;
    P->psi_alt = g.alt_after;
    return QVA_OK;
}

bool fuse_exchange_enabled() {
    static int env = [] {
        const char *e = getenv("QVA_FUSE_EXCHANGE");
        return e ? atoi(e) : 1;
    }();
    return env != 0;
}

// Fused exchange over peer memory: every rank's two state buffers are exported as CUDA IPC
// handles, all-gathered over the plan's NCCL communicator and mapped (NVLink P2P), so the pass
// before a global<->local exchange can store each tile straight into its receiving rank's
// buffer.  Any failure leaves ipc_ok = false and the exchange runs as NCCL send/recv.
// unmap every peer buffer this rank opened (ours are not IPC mappings)
void close_peer_maps(qva_plan *P) {
    for (int k = 0; k < 2; ++k)
        for (int t = 0; t < kMaxPeers; ++t) {
            double2 *ptr = P->ipc_peer[k][t];
            if (ptr && ptr != P->ipc_own[k]) cudaIpcCloseMemHandle(ptr);
            P->ipc_peer[k][t] = nullptr;
        }
    cudaGetLastError();
}

void setup_peer_exchange(qva_plan *P) {
    if ((!fuse_exchange_enabled() && P->mixer != QVA_MIXER_PARITY) || P->world > kMaxPeers || !P->psi ||
        !P->psi_alt || (!P->comm && !P->host_tp))
        return;
    P->ipc_own[0] = P->psi;
    P->ipc_own[1] = P->psi_alt;
    // every rank takes part in both collectives below whatever happens locally (a rank that
    // skipped one would leave the others blocked in it); the final min-reduce decides
    const size_t hb = sizeof(cudaIpcMemHandle_t);
    std::vector<unsigned char> mine(2 * hb, 0), all(2 * hb * P->world, 0);
    bool ok = cudaIpcGetMemHandle((cudaIpcMemHandle_t *)mine.data(), P->psi) == cudaSuccess &&
              cudaIpcGetMemHandle((cudaIpcMemHandle_t *)(mine.data() + hb), P->psi_alt) == cudaSuccess;
    cudaGetLastError();
    // NCCL staging in the (not yet used) receive buffer: no allocation that could fail on one rank
    unsigned char *dbuf = reinterpret_cast<unsigned char *>(P->psi_alt);
    const bool g = coll_allgather_host(P, mine.data(), all.data(), 2 * hb, dbuf) == QVA_OK;
    ok = ok && g;
    // a rank whose handles failed sent zeros: opening those fails here, and the vote below
    // turns the fused path off everywhere
    for (int t = 0; ok && t < P->world; ++t)
        for (int k = 0; ok && k < 2; ++k) {
            if (t == P->rank) {
                P->ipc_peer[k][t] = P->ipc_own[k];
                continue;
            }
            cudaIpcMemHandle_t h;
            memcpy(&h, all.data() + (2 * t + k) * hb, hb);
            void *ptr = nullptr;
            ok = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
            P->ipc_peer[k][t] = (double2 *)ptr;
        }
    if (ok && !P->host_tp) ok = cudaMalloc(&P->d_bar, sizeof(int)) == cudaSuccess;
    cudaGetLastError();
    // every rank must agree, or the ranks would run different exchange code
    double flag = ok ? 1.0 : 0.0;
    if (coll_allreduce_host(P, &flag, 1, kCollMin, reinterpret_cast<double *>(P->psi_alt)) != QVA_OK) flag = 0.0;
    cudaGetLastError();
    P->ipc_ok = flag == 1.0;
    if (!P->ipc_ok) close_peer_maps(P);
}

qva_status allreduce_host(qva_plan *P, double *vals, int n) { return coll_allreduce_host(P, vals, n, kCollSum); }

// generic (non-tile) expectation over this process's arrays
qva_status expect_generic(qva_plan *P, const double2 *psi, uint64_t n, const double *q, double *out2) {
    int blocks = expect_partial_blocks(n);
    QVA_TRY(ensure_partials(P, blocks));
    {
        ProfScope ps(P, K_REDUCE, 24.0 * n);
        QVA_CUDA_TRY(launch_expect_partials(psi, q, n, P->partials, blocks, P->stream));
    }
    {
        ProfScope ps(P, K_REDUCE, 16.0 * blocks);
        QVA_CUDA_TRY(launch_reduce_partials(P->partials, blocks, 1, P->red, P->stream));
    }
    QVA_CUDA_TRY(cudaMemcpyAsync(out2, P->red, 2 * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    return sync(P);
}

// opt-in closed form of the complete-graph-family circulant (desc.reserved[4], kernels_complete.cu):
// single shard, spectrum given as (lambda_0, c) by qva_set_circulant_eigenvalues_const
bool use_complete_closed_form(const qva_plan *P) {
    return P->mixer == QVA_MIXER_CIRCULANT && P->d.reserved[4] != 0 && P->lam_const;
}

bool use_small(const qva_plan *P) { return P->mixer == QVA_MIXER_X && P->n <= kSmallMaxQubits && P->G == 1; }

// permuted out-of-place schedule: single shard, >= 21 qubits
// (a 9-bit read window above the contiguous tile), room for the ping-pong buffer.
// QVA_PERM=0 selects the in-place schedule.
bool use_permuted(const qva_plan *P) {
    static int env = [] {
        const char *e = getenv("QVA_PERM");
        return e ? atoi(e) : 1;
    }();
    return env != 0 && P->mixer == QVA_MIXER_X && P->G == 1 && P->L >= 21 && !P->perm_failed;
}

// ---- sharded circulant transport: row layout <-> column layout ----------------
// Row layout: shard s holds rows [s M1/G, (s+1) M1/G) of the M1 x M2 natural matrix; column
// layout: all rows of columns [s M2/G, (s+1) M2/G).  Virtual shards (one GPU): one block transpose
// of the whole array.  Real ranks: pack (block transpose) + grouped NCCL send/recv (+ unpack).
template <typename T>
qva_status shard_to_col(qva_plan *P, const T *row, T *col) {
    const int G = P->G;
    const uint64_t M1 = P->fft_M1, M2 = P->fft_M2, M1s = M1 / G, M2s = M2 / G;
    ProfScope ps(P, K_EXCHANGE, 2.0 * sizeof(T) * (double)P->arr_n);
    if (P->world == 1) {
        QVA_CUDA_TRY(launch_block_transpose<T>(col, row, M1, (uint64_t)G, M2s, P->stream));
        return QVA_OK;
    }
    T *snd = reinterpret_cast<T *>(P->xfer);
    QVA_CUDA_TRY(launch_block_transpose<T>(snd, row, M1s, (uint64_t)G, M2s, P->stream));
    return coll_alltoall_dev(P, snd, col, M1s * M2s * sizeof(T));
}
template <typename T>
qva_status shard_to_row(qva_plan *P, const T *col, T *row) {
    const int G = P->G;
    const uint64_t M1 = P->fft_M1, M2 = P->fft_M2, M1s = M1 / G, M2s = M2 / G;
    ProfScope ps(P, K_EXCHANGE, 2.0 * sizeof(T) * (double)P->arr_n);
    if (P->world == 1) {
        QVA_CUDA_TRY(launch_block_transpose<T>(row, col, (uint64_t)G, M1, M2s, P->stream));
        return QVA_OK;
    }
    T *rcv = reinterpret_cast<T *>(P->xfer);
    QVA_TRY(coll_alltoall_dev(P, col, rcv, M1s * M2s * sizeof(T)));
    QVA_CUDA_TRY(launch_block_transpose<T>(row, rcv, (uint64_t)G, M1s, M2s, P->stream));
    return QVA_OK;
}

struct PlanShardIO : FftShardIO {
    qva_plan *P;
    explicit PlanShardIO(qva_plan *P_) : P(P_) {}
    qva_status to_col(const double2 *row, double2 *col) override {
        count_xfer(P, sizeof(double2));
        return shard_to_col<double2>(P, row, col);
    }
    qva_status to_row(const double2 *col, double2 *row) override {
        count_xfer(P, sizeof(double2));
        return shard_to_row<double2>(P, col, row);
    }
    qva_status barrier() override {  // ends a transpose fused into the pass stores
        count_xfer(P, sizeof(double2));
        if (P->world == 1) return QVA_OK;  // virtual shards: stream order
        return coll_stream_barrier(P);
    }
};

// buffers of the sharded circulant path: column-layout work array (psi_alt), q in the column
// layout (qB), NCCL staging (xfer)
qva_status circ_shard_setup(qva_plan *P, PlanShardIO &io) {
    if (!P->psi_alt) QVA_CUDA_TRY(cudaMalloc(&P->psi_alt, P->arr_n * sizeof(double2)));
    if (P->world > 1 && !P->xfer) QVA_CUDA_TRY(cudaMalloc(&P->xfer, P->arr_n * sizeof(double2)));
    if (P->q_set && !P->qB_valid) {
        QVA_TRY(ensure_q_dev(P));
        if (!P->qB) QVA_CUDA_TRY(cudaMalloc(&P->qB, P->arr_n * sizeof(double)));
        QVA_TRY(shard_to_col<double>(P, P->q, P->qB));
        P->qB_valid = true;
    }
    io.G = P->G;
    io.local = P->world == 1 ? P->G : 1;
    io.first = P->world == 1 ? 0 : P->rank;
    io.col = P->psi_alt;
    io.q_col = P->qB;
    // transposes fused into the pass stores: virtual shards address blocks of psi / psi_alt, real
    // shards the IPC-mapped peer buffers (psi and psi_alt never swap on the circulant path)
    // (virtual shards only with peer_store_exchange: on one GPU the L2-resident block transposes
    // measured faster, cfg3 G = 2: 1.33 vs 1.41 ms; the flag runs the multi-GPU store path)
    io.fused = fuse_exchange_enabled() && P->G <= kMaxPeers &&
               (P->world == 1 ? P->d.reserved[3] != 0 : P->ipc_ok);
    if (io.fused) {
        const uint64_t NG = P->N / P->G;
        for (int t = 0; t < P->G; ++t) {
            io.row_dst[t] = P->world == 1 ? P->psi + t * NG : P->ipc_peer[0][t];
            io.col_dst[t] = P->world == 1 ? P->psi_alt + t * NG : P->ipc_peer[1][t];
        }
    }
    return QVA_OK;
}

// QAOAz parity mixer U(t) = e^{-itB_last} e^{-itB_even} e^{-itB_odd} (reading R19).  The pair
// terms of one group act on disjoint qubits and commute; a term only has to follow the terms of
// earlier groups it shares a qubit with.  Windows of <= 12 physical bits (0..2 always, for
// 128-B rows) each take, greedily in group order, every term whose qubits fit and whose
// predecessors are done or earlier in the same window: one HBM round trip per window instead of
// one per term (default sequence, n = 28: 5 windows for 27 terms).
static std::vector<ParityWinPlan> parity_window_plan(int n, const std::vector<int> &s);
// Sharded state (qubits >= nl are rank bits): windows over local bits take the ready local terms
// (as parity_window_plan); when no local term is ready, every ready term touching a rank qubit
// becomes one peer pass.  One layer of the mixer.
static std::vector<ParityItem> parity_shard_items(int n, int nl, const std::vector<int> &s) {
    const int K = (int)s.size();
    std::vector<std::pair<int, int>> terms;
    std::vector<int> grp;
    for (int m = 0; m + 1 < K; m += 2) terms.push_back({s[m], s[m + 1]}), grp.push_back(0);
    for (int m = 1; m + 1 < K; m += 2) terms.push_back({s[m], s[m + 1]}), grp.push_back(1);
    if (K >= 3 && (K & 1)) terms.push_back({s[K - 1], s[0]}), grp.push_back(2);
    const int T = (int)terms.size();
    std::vector<std::vector<int>> deps(T);
    for (int k = 0; k < T; ++k)
        for (int j = 0; j < k; ++j)
            if (grp[j] < grp[k] && (terms[j].first == terms[k].first || terms[j].first == terms[k].second ||
                                    terms[j].second == terms[k].first || terms[j].second == terms[k].second))
                deps[k].push_back(j);
    auto local = [&](int k) { return terms[k].first < nl && terms[k].second < nl; };
    std::vector<char> done(T, 0);
    std::vector<ParityItem> out;
    const int wmax = std::min(nl, kWinMaxBits);
    for (int left = T; left > 0;) {
        std::vector<char> inw(n, 0), placed(T, 0);
        int w = 0;
        for (int b = 0; b < std::min(3, nl); ++b) inw[b] = 1, ++w;
        std::vector<int> plan;
        for (int k = 0; k < T && (int)plan.size() < kWinMaxPairs; ++k) {
            if (done[k] || !local(k)) continue;
            bool ready = true;
            for (int j : deps[k]) ready = ready && (done[j] || placed[j]);
            if (!ready) continue;
            const int need = !inw[terms[k].first] + !inw[terms[k].second];
            if (w + need > wmax) continue;
            inw[terms[k].first] = inw[terms[k].second] = 1;
            w += need;
            placed[k] = 1;
            plan.push_back(k);
        }
        if (!plan.empty()) {
            for (int b = 0; b < nl && w < wmax; ++b)
                if (!inw[b]) inw[b] = 1, ++w;
            ParityItem it;
            for (int b = 0; b < nl; ++b)
                if (inw[b]) it.win.bits.push_back(b);
            for (int k : plan) {
                it.win.ta.push_back(terms[k].first);
                it.win.tb.push_back(terms[k].second);
                it.win.cls.push_back(grp[k]);
                done[k] = 1;
            }
            left -= (int)plan.size();
            out.push_back(it);
            continue;
        }
        int got = 0;
        std::vector<int> ready_g;
        for (int k = 0; k < T; ++k) {
            if (done[k] || local(k)) continue;
            bool ready = true;
            for (int j : deps[k]) ready = ready && done[j];
            if (ready) ready_g.push_back(k);
        }
        for (int k : ready_g) {
            ParityItem it;
            it.global = true;
            it.a = terms[k].first;
            it.b = terms[k].second;
            out.push_back(it);
            done[k] = 1;
            ++got;
        }
        left -= got;
        if (!got) return {};  // cannot happen: some term is always ready
    }
    return out;
}

static std::vector<ParityWinPlan> parity_window_plan(int n, const std::vector<int> &s) {
    const int K = (int)s.size();
    std::vector<std::pair<int, int>> terms;
    std::vector<int> grp;
    for (int m = 0; m + 1 < K; m += 2) terms.push_back({s[m], s[m + 1]}), grp.push_back(0);
    for (int m = 1; m + 1 < K; m += 2) terms.push_back({s[m], s[m + 1]}), grp.push_back(1);
    if (K >= 3 && (K & 1)) terms.push_back({s[K - 1], s[0]}), grp.push_back(2);
    const int T = (int)terms.size();
    std::vector<std::vector<int>> deps(T);
    for (int k = 0; k < T; ++k)
        for (int j = 0; j < k; ++j)
            if (grp[j] < grp[k] && (terms[j].first == terms[k].first || terms[j].first == terms[k].second ||
                                    terms[j].second == terms[k].first || terms[j].second == terms[k].second))
                deps[k].push_back(j);
    std::vector<char> done(T, 0);
    std::vector<ParityWinPlan> out;
    const int wmax = std::min(n, kWinMaxBits);
    for (int left = T; left > 0;) {
        std::vector<char> inw(n, 0), placed(T, 0);
        int w = 0;
        for (int b = 0; b < std::min(3, n); ++b) inw[b] = 1, ++w;
        std::vector<int> plan;
        for (int k = 0; k < T && (int)plan.size() < kWinMaxPairs; ++k) {
            if (done[k]) continue;
            bool ready = true;
            for (int j : deps[k]) ready = ready && (done[j] || placed[j]);
            if (!ready) continue;
            const int need = !inw[terms[k].first] + !inw[terms[k].second];
            if (w + need > wmax) continue;
            inw[terms[k].first] = inw[terms[k].second] = 1;
            w += need;
            placed[k] = 1;
            plan.push_back(k);
        }
        // pad the window to wmax bits with the lowest free bits (longer rows, fewer tiles)
        for (int b = 0; b < n && w < wmax; ++b)
            if (!inw[b]) inw[b] = 1, ++w;
        ParityWinPlan W;
        for (int b = 0; b < n; ++b)
            if (inw[b]) W.bits.push_back(b);
        for (int k : plan) {
            W.ta.push_back(terms[k].first);
            W.tb.push_back(terms[k].second);
            W.cls.push_back(grp[k]);
            done[k] = 1;
        }
        left -= (int)plan.size();
        out.push_back(W);
    }
    return out;
}

// A window plan as run tables for the register-free parity_window_kernel on a state of n bits.
// false if too fragmented for the run tables (the caller takes the per-term passes).
static bool parity_window_of(int n, const ParityWinPlan &P, ParityWindow &W) {
    std::vector<char> inw(n, 0);
    for (int b : P.bits) inw[b] = 1;
    memset(&W, 0, sizeof(W));
    W.n = n;
    W.w = (int)P.bits.size();
    std::vector<int> local(n, -1);
    for (int i = 0; i < (int)P.bits.size(); ++i) local[P.bits[i]] = i;
    auto runs = [&](bool in_window, int *src, int *wd, int *dst, int cap, int &nr) {
        nr = 0;
        int idx = 0;  // running index in the window (or the tile number)
        for (int b = 0; b < n;) {
            if ((bool)inw[b] != in_window) { ++b; continue; }
            int st = b;
            while (b < n && (bool)inw[b] == in_window) ++b;
            if (nr == cap) return false;
            src[nr] = idx;
            wd[nr] = b - st;
            dst[nr] = st;
            idx += b - st;
            ++nr;
        }
        return true;
    };
    if (!runs(true, W.in_src, W.in_w, W.in_dst, kWinMaxRuns, W.n_in) ||
        !runs(false, W.out_src, W.out_w, W.out_dst, kWinMaxRuns + 1, W.n_out))
        return false;
    W.np = (int)P.ta.size();
    for (int i = 0; i < W.np; ++i) {
        W.pa[i] = (int8_t)local[P.ta[i]];
        W.pb[i] = (int8_t)local[P.tb[i]];
    }
    return true;
}

// Windows of <= 12 physical bits for the register-free parity_window_kernel.
static std::vector<ParityWindow> parity_windows(int n, const std::vector<int> &s) {
    std::vector<ParityWindow> out;
    for (const ParityWinPlan &P : parity_window_plan(n, s)) {
        ParityWindow W;
        if (!parity_window_of(n, P, W)) return {};
        out.push_back(W);
    }
    return out;
}

// The window's pair terms as register-group steps of a tile pass (window bit i = tile bit i): at
// each step the group (X, Y, W, V, Z) that can apply the most remaining terms -- both qubits among
// its register bits, every earlier-class term of the window sharing a qubit already applied --
// takes them in window order (ties: stay in the current group, i.e. no smem transpose).
// false if some term fits no group (the caller keeps the register-free window kernel).
static bool parity_group_steps(const ParityWinPlan &W, std::vector<PassStep> &steps) {
    const int T = (int)W.ta.size();
    if (T > 64) return false;
    std::vector<int> tbit(64, -1);
    for (int i = 0; i < (int)W.bits.size(); ++i) tbit[W.bits[i]] = i;
    std::vector<uint64_t> dep(T, 0);  // earlier-class terms of the window sharing a qubit
    for (int k = 0; k < T; ++k)
        for (int j = 0; j < T; ++j)
            if (W.cls[j] < W.cls[k] && (W.ta[j] == W.ta[k] || W.ta[j] == W.tb[k] || W.tb[j] == W.ta[k] ||
                                        W.tb[j] == W.tb[k]))
                dep[k] |= 1ull << j;
    uint64_t fits[kMaxGroups] = {};  // terms whose two qubits are register bits of group g
    for (int g = 0; g < kMaxGroups; ++g)
        for (int k = 0; k < T; ++k)
            if (ebit_index(g, tbit[W.ta[k]]) >= 0 && ebit_index(g, tbit[W.tb[k]]) >= 0) fits[g] |= 1ull << k;
    const uint64_t all = T == 64 ? ~0ull : (1ull << T) - 1;
    // a step in group g takes every applicable term in window order (taking a term never delays
    // another), so a plan is a group sequence; iterative deepening finds the fewest steps
    auto step = [&](uint64_t done, int g) {
        for (int k = 0; k < T; ++k)
            if (!((done >> k) & 1) && ((fits[g] >> k) & 1) && (dep[k] & ~done) == 0) done |= 1ull << k;
        return done;
    };
    std::vector<int> seq;
    std::function<bool(uint64_t, int)> dfs = [&](uint64_t done, int depth) -> bool {
        if (done == all) return true;
        if (depth == 0) return false;
        for (int g = 0; g < kMaxGroups; ++g) {
            if (!seq.empty() && seq.back() == g) continue;
            const uint64_t nd = step(done, g);
            if (nd == done) continue;
            seq.push_back(g);
            if (dfs(nd, depth - 1)) return true;
            seq.pop_back();
        }
        return false;
    };
    bool found = false;
    for (int depth = 1; depth <= 8 && !found; ++depth) {
        seq.clear();
        found = dfs(0, depth);
    }
    if (!found) return false;
    uint64_t done = 0;
    for (int g : seq) {
        const uint64_t nd = step(done, g);
        std::vector<int> take;
        for (int k = 0; k < T; ++k)
            if (((nd & ~done) >> k) & 1) take.push_back(k);
        // within the step, a term follows the terms it depends on (window order already does)
        for (size_t i = 0; i < take.size(); i += kMaxStepPairs) {
            PassStep st;
            memset(&st, 0, sizeof(st));
            st.group = (int8_t)g;
            for (size_t k = i; k < take.size() && k < i + kMaxStepPairs; ++k) {
                int ja = ebit_index(g, tbit[W.ta[take[k]]]), jb = ebit_index(g, tbit[W.tb[take[k]]]);
                if (ja > jb) std::swap(ja, jb);
                st.pair[st.npair++] = (int8_t)(ja * 8 + jb);
            }
            steps.push_back(st);
        }
        done = nd;
    }
    return true;
}

// QAOAz evolution as tile passes (one HBM round trip per window, pair terms on register groups,
// phase fused into the first window of each layer, <Q> into the last): single shard, n >= 12,
// every window plannable.  Returns false when the sequence needs the register-free path.
static bool parity_tile_passes(int n, int L, int G, const std::vector<int> &s, int p, std::vector<PassPlan> &out) {
    out.clear();
    if (G != 1 || L < kTileBits || n != L || p < 1) return false;
    const std::vector<ParityWinPlan> wins = parity_window_plan(n, s);
    if (wins.empty()) return false;
    std::vector<std::vector<PassStep>> wsteps(wins.size());
    for (size_t w = 0; w < wins.size(); ++w) {
        if ((int)wins[w].bits.size() != kTileBits) return false;
        if (!parity_group_steps(wins[w], wsteps[w]) || wsteps[w].empty()) return false;
        if (tile_tma_dims(wins[w].bits.data(), n, nullptr) > 5) return false;
        int runs = 0;  // non-tile runs (TilePassParams::run_*)
        for (int b = 0; b < n;) {
            if (std::find(wins[w].bits.begin(), wins[w].bits.end(), b) != wins[w].bits.end()) { ++b; continue; }
            ++runs;
            while (b < n && std::find(wins[w].bits.begin(), wins[w].bits.end(), b) == wins[w].bits.end()) ++b;
        }
        if (runs > kMaxRuns) return false;
    }
    for (int k = 0; k < p; ++k)
        for (size_t w = 0; w < wins.size(); ++w) {
            PassPlan pp;
            pp.parity = true;
            pp.tbits = wins[w].bits;
            pp.play = k;
            pp.phase = (w == 0) ? k : -1;
            pp.expect = (k == p - 1 && w + 1 == wins.size());
            pp.psteps = wsteps[w];
            if (pp.phase >= 0) {  // the layer's phase on load: in a step, phase precedes its pair terms
                pp.psteps.front().phase = 1;
                if (pp.expect && pp.psteps.back().group != pp.psteps.front().group) {  // one q group per pass
                    PassStep e;
                    memset(&e, 0, sizeof(e));
                    e.group = pp.psteps.front().group;
                    pp.psteps.push_back(e);
                }
            }
            if ((int)pp.psteps.size() > kMaxSteps) return false;
            out.push_back(pp);
        }
    return true;
}

qva_status reset_state(qva_plan *P);
qva_status run_passes(qva_plan *P, const std::vector<PassPlan> &passes, const double *thetas, int p, int batch,
                      double2 *psi_base, uint64_t stride, int init_mode, double *expect_out);
// QAOAz on a sharded state (world > 1; rank = the top g qubits).  Per layer the items of
// parity_shard_items: windows of local bits run as tile passes (pair terms on register groups,
// phase fused into the layer's first window, <Q> into the last), and each term touching a rank
// qubit runs as one peer pass that reads the partner rank's IPC-mapped buffer (parity_peer_kernel),
// after a barrier (every rank's previous writes are done).  t_only != nullptr: one mixer step on the
// current state (no phase, no expectation).
static qva_status parity_sharded_run(qva_plan *P, const double *theta, int p, bool *have_red, const double *t_only) {
    *have_red = false;
    if (!P->ipc_ok) {
        set_error("sharded QAOAz mixer needs the peers' buffers mapped (CUDA IPC)");
        return QVA_ERR_UNSUPPORTED;
    }
    if (P->parity_shard_seq != P->parity_seq) {
        P->parity_shard_items = parity_shard_items(P->n, P->L, P->parity_seq);
        P->parity_shard_steps.assign(P->parity_shard_items.size(), {});
        for (size_t i = 0; i < P->parity_shard_items.size(); ++i) {  // no steps: the register-free path
            const ParityItem &it = P->parity_shard_items[i];
            if (it.global) continue;
            if ((int)it.win.bits.size() != kTileBits || tile_tma_dims(it.win.bits.data(), P->L, nullptr) > 5 ||
                !parity_group_steps(it.win, P->parity_shard_steps[i]))
                P->parity_shard_steps[i].clear();
        }
        P->parity_shard_seq = P->parity_seq;
    }
    const auto &items = P->parity_shard_items;
    if (items.empty()) {
        set_error("sharded QAOAz: no window plan for this qubit sequence");
        return QVA_ERR_UNSUPPORTED;
    }
    std::vector<double> th1;
    if (t_only) {
        th1 = {0.0, *t_only};
        theta = th1.data();
        p = 1;
    }
    const bool evolving = t_only == nullptr;
    bool first = evolving;  // the evolution's first pass starts from |+> / psi0
    std::vector<PassPlan> run;
    auto flush = [&]() -> qva_status {
        if (run.empty()) return QVA_OK;
        QVA_TRY(run_passes(P, run, theta, p, 1, P->psi, 0, first ? (P->has_psi0 ? 2 : 1) : 0, nullptr));
        first = false;
        run.clear();
        return QVA_OK;
    };
    for (int k = 0; k < p; ++k) {
        bool phase_pending = evolving;
        for (size_t i = 0; i < items.size(); ++i) {
            const ParityItem &it = items[i];
            const bool last = evolving && k == p - 1 && i + 1 == items.size();
            if (!it.global && !P->parity_shard_steps[i].empty()) {
                PassPlan pp;
                pp.parity = true;
                pp.tbits = it.win.bits;
                pp.play = k;
                pp.psteps = P->parity_shard_steps[i];
                if (phase_pending) {
                    pp.phase = k;
                    pp.psteps.front().phase = 1;
                    phase_pending = false;
                }
                pp.expect = last;
                if (pp.expect && pp.phase >= 0 && pp.psteps.back().group != pp.psteps.front().group) {
                    PassStep e;
                    memset(&e, 0, sizeof(e));
                    e.group = pp.psteps.front().group;
                    pp.psteps.push_back(e);
                }
                if ((int)pp.psteps.size() > kMaxSteps) {
                    set_error("sharded QAOAz: window pass has too many steps");
                    return QVA_ERR_UNSUPPORTED;
                }
                run.push_back(pp);
                if (last) *have_red = true;
                continue;
            }
            QVA_TRY(flush());
            if (first) {
                QVA_TRY(reset_state(P));
                first = false;
            }
            if (!it.global) {  // a local window no tile plan covers: window kernel (phase fused), else per term
                const double t = theta[2 * k + 1];
                ParityWindow W;
                if (parity_window_of(P->L, it.win, W)) {
                    if (phase_pending) QVA_TRY(ensure_q_dev(P));
                    W.c = cos(2.0 * t);
                    W.s = sin(2.0 * t);
                    W.q = phase_pending ? P->q : nullptr;
                    W.gamma = theta[2 * k];
                    phase_pending = false;
                    ProfScope ps(P, K_OTHER, (32.0 + (W.q ? 8.0 : 0.0)) * P->arr_n);
                    QVA_CUDA_TRY(launch_parity_window(P->psi, W, P->stream));
                    continue;
                }
                if (phase_pending) {
                    QVA_TRY(ensure_q_dev(P));
                    ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
                    QVA_CUDA_TRY(launch_phase(P->psi, P->q, P->arr_n, theta[2 * k], P->stream));
                    phase_pending = false;
                }
                for (size_t m = 0; m < it.win.ta.size(); ++m) {
                    ProfScope ps(P, K_OTHER, 32.0 * P->arr_n);
                    QVA_CUDA_TRY(launch_parity_pair(P->psi, P->arr_n, it.win.ta[m], it.win.tb[m], t, P->stream));
                }
                continue;
            }
            if (phase_pending) {  // the layer opens with a rank-qubit term: a standalone phase
                QVA_TRY(ensure_q_dev(P));
                ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
                QVA_CUDA_TRY(launch_phase(P->psi, P->q, P->arr_n, theta[2 * k], P->stream));  // layout A
                phase_pending = false;
            }
            QVA_TRY(coll_stream_barrier(P));  // every rank's state is final before anyone reads it
            ParityPeer pr{};
            pr.L = P->L;
            pr.rank = P->rank;
            pr.a = it.a;
            pr.b = it.b;
            pr.c = cos(2.0 * theta[2 * k + 1]);
            pr.s = sin(2.0 * theta[2 * k + 1]);
            const int kb = (P->psi == P->ipc_own[0]) ? 0 : 1;  // every rank swaps in lockstep
            for (int t = 0; t < P->world; ++t) pr.peer[t] = P->ipc_peer[kb][t];
            {
                ProfScope ps(P, K_EXCHANGE, 48.0 * P->arr_n);
                QVA_CUDA_TRY(launch_parity_peer(P->psi_alt, P->psi, pr, P->stream));
            }
            std::swap(P->psi, P->psi_alt);
            count_xfer(P, sizeof(double2) * 2);  // about half the elements read remotely
        }
    }
    QVA_TRY(flush());
    if (first) QVA_TRY(reset_state(P));  // p = 0: the initial state
    return QVA_OK;
}

// one mixer step; q != nullptr also applies the phase exp(-i gamma q) first (fused into the
// first window's loads)
qva_status parity_mix(qva_plan *P, double t, const double *q = nullptr, double gamma = 0.0, bool from_psi0 = false) {
    if (P->world > 1 && !P->replicated) {  // sharded state
        if (from_psi0) QVA_TRY(reset_state(P));
        if (q) {
            ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
            QVA_CUDA_TRY(launch_phase(P->psi, q, P->arr_n, gamma, P->stream));
        }
        bool dummy = false;
        return parity_sharded_run(P, nullptr, 1, &dummy, &t);
    }
    const std::vector<int> &s = P->parity_seq;
    const int K = (int)s.size();
    static int win_env = [] {
        const char *e = getenv("QVA_PARITY_WINDOWS");
        return e ? atoi(e) : 1;
    }();
    if (win_env && P->arr_n == (1ull << P->n)) {
        if (P->parity_win_seq != s) {
            P->parity_win = parity_windows(P->n, s);
            P->parity_win_seq = s;
        }
        if (!P->parity_win.empty()) {
            for (size_t i = 0; i < P->parity_win.size(); ++i) {
                ParityWindow W = P->parity_win[i];
                W.c = cos(2.0 * t);
                W.s = sin(2.0 * t);
                W.q = (i == 0) ? q : nullptr;
                W.gamma = gamma;
                if (i == 0 && from_psi0) {  // the first window also stands in for reset_state
                    if (P->has_psi0) W.src = P->psi0;
                    else W.init_amp = 1.0 / sqrt((double)P->N);
                }
                ProfScope ps(P, K_OTHER, (32.0 + (W.q ? 8.0 : 0.0)) * P->arr_n);
                QVA_CUDA_TRY(launch_parity_window(P->psi, W, P->stream));
            }
            return QVA_OK;
        }
    }
    if (from_psi0) QVA_TRY(reset_state(P));
    if (q) {
        ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
        QVA_CUDA_TRY(launch_phase(P->psi, q, P->arr_n, gamma, P->stream));
    }
    auto pair = [&](int a, int b) -> qva_status {
        ProfScope ps(P, K_OTHER, 16.0 * P->arr_n);
        QVA_CUDA_TRY(launch_parity_pair(P->psi, P->arr_n, a, b, t, P->stream));
        return QVA_OK;
    };
    for (int m = 0; m + 1 < K; m += 2) QVA_TRY(pair(s[m], s[m + 1]));
    for (int m = 1; m + 1 < K; m += 2) QVA_TRY(pair(s[m], s[m + 1]));
    if (K >= 3 && (K & 1)) QVA_TRY(pair(s[K - 1], s[0]));
    return QVA_OK;
}

// apply one mixer on the current state (no phase)
qva_status apply_mixer_impl(qva_plan *P, double beta) {
    if (P->mixer == QVA_MIXER_X) {
        if (use_small(P)) {
            QVA_TRY(ensure_q_alloc(P));  // the small-state kernel stages q even when it only mixes
            SmallEvolveParams sp{};
            sp.psi = P->psi;
            sp.q = P->q;
            sp.n = P->n;
            sp.p = 1;
            sp.mode = 2;
            double th = beta;
            QVA_CUDA_TRY(cudaMemcpyAsync(P->d_thetas, &th, sizeof(double), cudaMemcpyHostToDevice, P->stream));
            sp.thetas = P->d_thetas;
            ProfScope ps(P, K_SMALL, 32.0 * P->arr_n);
            QVA_CUDA_TRY(launch_small_evolve(sp, 1, P->stream));
            return QVA_OK;
        }
        auto toks = mixer_tokens(P->L, P->gbits);
        auto passes = cut_passes(toks, P->sets, false);
        double th[2] = {0.0, beta};
        QVA_TRY(run_passes(P, passes, th, 1, 1, P->psi, 0, 0, nullptr));
        return QVA_OK;
    }
    if (P->mixer == QVA_MIXER_CIRCULANT) {
        if (!P->lam_set) {
            set_error("circulant spectrum not set");
            return QVA_ERR_NOT_READY;
        }
        FftRun r;
        r.psi = P->psi;
        r.q = P->q;
        r.lambda_perm = P->lam_const ? nullptr : P->lambda_perm;
        r.lam0 = P->lam0;
        r.lamc = P->lamc;
        r.theta = &beta;
        r.mode = 1;
        PlanObserver obs(P);
        if (use_complete_closed_form(P)) {
            double *scr = nullptr;
            QVA_CUDA_TRY(scratch_get(P, (void **)&scr, complete_scratch_doubles(P->arr_n) * sizeof(double)));
            PlanCompleteComm cc(P);
            return complete_run(r, P->arr_n, P->N, scr, P->stream, &obs, P->world > 1 ? &cc : nullptr);
        }
        if (P->G > 1) {
            PlanShardIO io(P);
            QVA_TRY(circ_shard_setup(P, io));
            return fft_run_sharded(P->fft, r, io, P->stream, &obs);
        }
        return fft_run(P->fft, r, P->stream, &obs);
    }
    if (P->mixer == QVA_MIXER_PARITY) return parity_mix(P, beta);
    if (P->mixer == QVA_MIXER_SPARSE) {
        if (!P->sparse_set) {
            set_error("sparse mixer not set");
            return QVA_ERR_NOT_READY;
        }
        int terms = 0;
        PlanObserver obs(P);
        PlanSparseComm comm(P);
        return sparse_apply_mixer(P->sm, P->psi, beta, P->stream, &obs, &terms,
                                  (P->world > 1 && !P->replicated) ? &comm : nullptr);
    }
    return QVA_ERR_UNSUPPORTED;
}

qva_status reset_state(qva_plan *P) {
    if (P->has_psi0) {
        QVA_CUDA_TRY(cudaMemcpyAsync(P->psi, P->psi0, P->arr_n * sizeof(double2), cudaMemcpyDeviceToDevice, P->stream));
    } else {
        QVA_CUDA_TRY(launch_fill_uniform(P->psi, P->arr_n, 1.0 / sqrt((double)P->N), P->stream));
    }
    P->layout = 0;
    P->perm.clear();
    return QVA_OK;
}

qva_status check_range(const qva_plan *P, uint64_t offset, uint64_t count, uint64_t *local_off) {
    uint64_t lo = P->offset, hi = P->offset + P->local_n;
    if (offset < lo || offset + count > hi || offset + count < offset) {
        set_error("range [" + std::to_string(offset) + ", " + std::to_string(offset + count) +
                  ") outside this rank's partition [" + std::to_string(lo) + ", " + std::to_string(hi) + ")");
        return QVA_ERR_SIZE_MISMATCH;
    }
    *local_off = offset - lo;
    return QVA_OK;
}

}  // namespace

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

const char *qva_version(void) { return "qva-b200 0.1 (sm_100a)"; }

const char *qva_status_string(qva_status s) {
    switch (s) {
        case QVA_OK: return "QVA_OK";
        case QVA_ERR_INVALID_ARGUMENT: return "QVA_ERR_INVALID_ARGUMENT";
        case QVA_ERR_SIZE_MISMATCH: return "QVA_ERR_SIZE_MISMATCH";
        case QVA_ERR_NOT_READY: return "QVA_ERR_NOT_READY";
        case QVA_ERR_NUMERIC: return "QVA_ERR_NUMERIC";
        case QVA_ERR_UNSUPPORTED: return "QVA_ERR_UNSUPPORTED";
        case QVA_ERR_OUT_OF_MEMORY: return "QVA_ERR_OUT_OF_MEMORY";
        case QVA_ERR_CUDA: return "QVA_ERR_CUDA";
        case QVA_ERR_NCCL: return "QVA_ERR_NCCL";
    }
    return "QVA_ERR_UNKNOWN";
}

const char *qva_last_error(void) { return g_last_error.c_str(); }

qva_status qva_partition(uint64_t dim, int32_t world, int32_t rank, uint64_t *local_n, uint64_t *offset) {
    if (!local_n || !offset || world < 1 || rank < 0 || rank >= world || dim == 0) {
        set_error("qva_partition: invalid argument");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    // Eqs. local_i / offset; remainder to the lowest ranks (reading R16)
    uint64_t base = dim / world, rem = dim % world;
    *local_n = base + ((uint64_t)rank < rem ? 1 : 0);
    *offset = base * rank + std::min<uint64_t>(rank, rem);
    return QVA_OK;
}

qva_status qva_batch_partition(int32_t B, int32_t world, int32_t rank, int32_t *first, int32_t *count) {
    if (!first || !count || B < 0 || world < 1 || rank < 0 || rank >= world) {
        set_error("qva_batch_partition: invalid argument");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    int32_t base = B / world, rem = B % world;
    *count = base + (rank < rem ? 1 : 0);
    *first = base * rank + std::min(rank, rem);
    return QVA_OK;
}

qva_status qva_exchange_plan(int32_t G, int32_t rank, int32_t *peer_of_chunk, int32_t *peer_chunk) {
    if (G < 1 || (G & (G - 1)) || rank < 0 || rank >= G || !peer_of_chunk || !peer_chunk) {
        set_error("qva_exchange_plan: G must be a power of two, 0 <= rank < G");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    for (int32_t t = 0; t < G; ++t) {
        peer_of_chunk[t] = t;    // chunk t (top local bits = t) goes to the shard whose rank is t
        peer_chunk[t] = rank;    // ... where it becomes chunk `rank` (top local bits = our rank)
    }
    return QVA_OK;
}

qva_status qva_x_schedule(int32_t n_local, int32_t p, int32_t *out, int32_t cap, int32_t *n_passes) {
    if (n_local < kTileBits || n_local > 40 || p < 0 || !n_passes) {
        set_error("qva_x_schedule: need 12 <= n_local <= 40");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    auto sets = make_tile_sets(n_local);
    auto passes = cut_passes(evolve_tokens(n_local, 0, p), sets, true);
    *n_passes = (int32_t)passes.size();
    for (int i = 0; i < (int)passes.size() && i < cap; ++i) {
        out[4 * i + 0] = passes[i].set;
        out[4 * i + 1] = __builtin_popcount(passes[i].r1);
        out[4 * i + 2] = passes[i].phase >= 0 ? 1 : 0;
        out[4 * i + 3] = __builtin_popcount(passes[i].r2);
    }
    return QVA_OK;
}

qva_status qva_x_schedule_permuted(int32_t n_local, int32_t p, int64_t *out, int32_t cap, int32_t *n_passes) {
    if (n_local < 21 || n_local > 40 || p < 1 || !n_passes) {
        set_error("qva_x_schedule_permuted: need 21 <= n_local <= 40 and p >= 1");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    std::vector<int> fin;
    auto passes = perm_passes(n_local, p, &fin);
    *n_passes = (int32_t)passes.size();
    for (int i = 0; i < (int)passes.size() && i < cap; ++i) {
        const PassPlan &pp = passes[i];
        int64_t l1 = 0, l2 = 0;
        for (int k = 0; k < kTileBits; ++k) {
            if ((pp.r1 >> k) & 1) l1 |= 1ll << pp.lay_in[pp.tbits[k]];
            if ((pp.r2 >> k) & 1) l2 |= 1ll << pp.lay_in[pp.tbits[k]];
        }
        int64_t *o = out + 8 * (size_t)i;
        o[0] = pp.tbits[3];
        o[1] = pp.a1;
        o[2] = pp.a2;
        o[3] = pp.phase;
        o[4] = pp.expect ? 1 : 0;
        o[5] = l1;
        o[6] = l2;
        o[7] = tile_tma_dims(pp.tbits.data(), n_local, pp.obit.data());
    }
    return QVA_OK;
}

qva_status qva_parity_schedule(int32_t n, const int32_t *seq, int32_t count, int32_t *out, int32_t cap,
                               int32_t *n_windows) {
    if (n < 1 || n > 62 || !seq || count < 2 || !n_windows) {
        set_error("qva_parity_schedule: need 1 <= n <= 62 and a sequence of >= 2 qubits");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    std::vector<int> s(seq, seq + count);
    for (int q : s)
        if (q < 0 || q >= n) {
            set_error("qva_parity_schedule: qubit outside [0, n)");
            return QVA_ERR_INVALID_ARGUMENT;
        }
    const std::vector<ParityWindow> wins = parity_windows(n, s);
    *n_windows = (int32_t)wins.size();
    // per window: [w, np, bits of the window (w entries, ascending), (a, b) physical per pair]
    int32_t pos = 0;
    for (const ParityWindow &W : wins) {
        std::vector<int> bits;
        for (int r = 0; r < W.n_in; ++r)
            for (int j = 0; j < W.in_w[r]; ++j) bits.push_back(W.in_dst[r] + j);
        const int32_t need = 2 + W.w + 2 * W.np;
        if (pos + need <= cap) {
            out[pos] = W.w;
            out[pos + 1] = W.np;
            for (int j = 0; j < W.w; ++j) out[pos + 2 + j] = bits[j];
            for (int i = 0; i < W.np; ++i) {
                out[pos + 2 + W.w + 2 * i] = bits[W.pa[i]];
                out[pos + 3 + W.w + 2 * i] = bits[W.pb[i]];
            }
        }
        pos += need;
    }
    return QVA_OK;
}

qva_status qva_circulant_plan_shape(uint64_t dim, int32_t shards, int32_t flags, int64_t *out) {
    if (!out || shards < 1) return QVA_ERR_INVALID_ARGUMENT;
    const FftShape sh = fft_plan_shape(dim, shards, (flags & 1) != 0);
    out[0] = sh.ok ? (sh.whole ? 0 : (sh.bluestein ? 2 : (sh.levels == 3 ? 3 : 1))) : -1;
    out[1] = (int64_t)sh.M;
    out[2] = sh.M1;
    out[3] = sh.levels == 3 ? (int64_t)sh.Mi1 * sh.Mi2 : sh.M2;
    out[4] = sh.cw;
    out[5] = sh.rb;
    out[6] = sh.levels;
    out[7] = sh.Mi1;
    out[8] = sh.Mi2;
    if (!sh.ok) {
        set_error("no FFT plan for dim " + std::to_string(dim));
        return QVA_ERR_UNSUPPORTED;
    }
    return QVA_OK;
}

qva_status qva_nccl_unique_id(void *id_out) {
    if (!id_out) return QVA_ERR_INVALID_ARGUMENT;
    ncclUniqueId id;
    QVA_NCCL_TRY(ncclGetUniqueId(&id));
    memcpy(id_out, &id, sizeof(id));
    return QVA_OK;
}

qva_status qva_plan_destroy(qva_plan *P) {
    if (!P) return QVA_OK;
    DeviceGuard dg(P->device);
    if (P->stream) cudaStreamSynchronize(P->stream);
    harvest(P);
    if (P->ipc_ok || P->sm.peer_ok) {
        // collective teardown: unmap the peers' buffers, then wait until every rank has unmapped
        // ours before freeing them (freeing exported memory that a peer still maps is undefined)
        close_peer_maps(P);
        if (P->sm.peer_ok) {
            for (int k = 0; k < 2; ++k)
                for (int t = 0; t < P->world; ++t)
                    if (t != P->rank && P->sm.src.peer[k][t]) cudaIpcCloseMemHandle((void *)P->sm.src.peer[k][t]);
            cudaGetLastError();
            P->sm.peer_ok = false;
        }
        if (P->created) {
            if (coll_stream_barrier(P) != QVA_OK) fprintf(stderr, "[qva] destroy: barrier failed: %s\n", qva_last_error());
            cudaStreamSynchronize(P->stream);
        }
        P->ipc_ok = false;
    }
    cudaFree(P->psi);
    cudaFree(P->psi_alt);
    cudaFree(P->xfer);
    cudaFree(P->psi0);
    cudaFree(P->q);
    cudaFree(P->qB);
    cudaFree(P->qc);
    cudaFree(P->qcB);
    cudaFree(P->d_tab);
    cudaFree(P->d_gam);
    drop_qt(P);
    for (auto &g : P->graphs) {
        cudaGraphExecDestroy(g.exec);
        cudaFreeHost(g.stage);
    }
    cudaFree(P->d_mult);
    cudaFree(P->d_edges);
    cudaFree(P->d_gen_edges);
    cudaFree(P->q_ex);
    cudaFree(P->d_ex_edges);
    for (int k = 0; k < 2; ++k)
        for (int t = 0; t < kMaxPeers; ++t)
            if (P->ipc_peer[k][t] && P->ipc_peer[k][t] != P->ipc_own[k]) cudaIpcCloseMemHandle(P->ipc_peer[k][t]);
    cudaFree(P->d_bar);
    cudaFree(P->d_ctr);
    cudaFree(P->scratch);
    cudaFree(P->small_batch);
    for (auto &e : P->pool) cudaFree(e.second);
    if (P->ring) cudaFreeHost(P->ring);
    cudaFree(P->partials);
    cudaFree(P->red);
    cudaFree(P->d_angles);
    cudaFree(P->d_thetas);
    cudaFree(P->d_flag);
    cudaFree(P->batch_psi);
    cudaFree(P->lambda_perm);
    if (P->fft) fft_plan_destroy(P->fft);
    cudaFree(P->sm.row_ptr);
    cudaFree(P->sm.col);
    cudaFree(P->sm.val);
    cudaFree(P->sm.t0);
    cudaFree(P->sm.t1);
    cudaFree(P->sm.scratch);
    cudaFree(P->sm.gather_buf);
    for (auto e : P->event_pool) cudaEventDestroy(e);
    if (P->comm) ncclCommDestroy(P->comm);
    if (P->own_stream && P->stream) cudaStreamDestroy(P->stream);
    delete P;
    return QVA_OK;
}

qva_status qva_plan_create(const qva_plan_desc *desc, qva_plan **out) { return qva_plan_create_ex(desc, nullptr, out); }

qva_status qva_plan_create_ex(const qva_plan_desc *desc, const qva_transport *transport, qva_plan **out) {
    if (!desc || !out) {
        set_error("qva_plan_create: NULL argument");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    if (transport && (!transport->allgather || !transport->allreduce_f64 || !transport->alltoall)) {
        set_error("qva_plan_create_ex: every transport function must be non-NULL");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    *out = nullptr;
    const qva_plan_desc &d = *desc;
    if (d.dim == 0 || d.world < 1 || d.rank < 0 || d.rank >= d.world || d.mixer < 0 || d.mixer > 3) {
        set_error("qva_plan_create: invalid dim/world/rank/mixer");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    int vs = d.virtual_shards > 1 ? d.virtual_shards : 1;
    bool replicated = d.reserved[0] != 0;
    if (vs > 1 && d.world > 1) {
        set_error("virtual_shards requires world == 1");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    if (d.mixer == QVA_MIXER_X || d.mixer == QVA_MIXER_PARITY) {
        if (d.n_qubits < 1 || d.n_qubits > 40 || d.dim != (1ull << d.n_qubits) ||
            (d.mixer == QVA_MIXER_PARITY && d.n_qubits < 2)) {
            set_error("X / parity mixer needs dim == 2^n_qubits (1 <= n <= 40; parity: n >= 2)");
            return QVA_ERR_UNSUPPORTED;
        }
    }
    int G = replicated ? 1 : d.world * vs;
    if (G > 1 && d.mixer == QVA_MIXER_CIRCULANT) {
        // distributed four-step FFT: needs G | M1 and G | M2 (checked on the FFT plan)
        if (d.dim % (uint64_t)G) {
            set_error("sharded circulant mixer needs dim divisible by the shard count");
            return QVA_ERR_UNSUPPORTED;
        }
    } else if (G > 1 && d.mixer == QVA_MIXER_PARITY && vs == 1) {
        // QAOAz over real ranks: windows of local bits + peer passes for rank-qubit terms
        if (!is_pow2((uint64_t)G) || d.n_qubits - ilog2(G) < kTileBits) {
            set_error("sharded QAOAz needs a power-of-two world and n_qubits - log2(world) >= 12");
            return QVA_ERR_UNSUPPORTED;
        }
    } else if (G > 1 && d.mixer == QVA_MIXER_SPARSE && vs == 1) {
        // row-partitioned W over real ranks (qva_set_sparse_mixer_rows): any dim, COMM-psi blocks
        if ((uint64_t)d.world > d.dim) {
            set_error("sharded sparse mixer needs dim >= world");
            return QVA_ERR_UNSUPPORTED;
        }
    } else if (G > 1) {
        if (d.mixer != QVA_MIXER_X) {
            set_error("sharded state (world*virtual_shards > 1) is implemented for the X and circulant mixers; "
                      "use the replicated mode (reserved[0]=1) for batches of sparse / parity evolutions");
            return QVA_ERR_UNSUPPORTED;
        }
        if (!is_pow2((uint64_t)G)) {
            set_error("X mixer sharding needs a power-of-two shard count");
            return QVA_ERR_UNSUPPORTED;
        }
        int g = ilog2(G);
        int L = d.n_qubits - g;
        if (L < kTileBits || g > L - 3 || g > 9) {
            set_error("sharded X mixer needs n_qubits - log2(shards) >= 12 local qubits");
            return QVA_ERR_UNSUPPORTED;
        }
    }
    DeviceGuard dg(d.device);
    qva_plan *P = new qva_plan();
    P->d = d;
    P->device = d.device;
    P->N = d.dim;
    P->mixer = d.mixer;
    P->world = d.world;
    P->rank = d.rank;
    P->vshards = vs;
    P->replicated = replicated;
    P->G = G;
    P->gbits = ilog2(G);
    P->max_batch = d.max_batch > 0 ? d.max_batch : 1;
    if (d.mixer == QVA_MIXER_X || d.mixer == QVA_MIXER_PARITY) {
        P->n = d.n_qubits;
        P->L = P->n - P->gbits;
    }
    if (d.mixer == QVA_MIXER_PARITY)
        for (int j = 0; j < d.n_qubits; ++j) P->parity_seq.push_back(j);
    if (replicated || d.world == 1) {
        P->local_n = P->N;
        P->offset = 0;
    } else {
        qva_partition(P->N, d.world, d.rank, &P->local_n, &P->offset);
    }
    P->arr_n = P->local_n;  // vshards: the whole vector lives here, in shard-major order
    auto fail = [&](qva_status s) {
        qva_plan_destroy(P);
        return s;
    };
    if (d.stream) {
        P->stream = (cudaStream_t)d.stream;
    } else {
        if (cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking) != cudaSuccess) {
            set_error("cudaStreamCreate failed");
            return fail(QVA_ERR_CUDA);
        }
        P->own_stream = true;
    }
    auto alloc = [&](void **ptr, size_t bytes) -> bool {
        if (cudaMalloc(ptr, bytes) != cudaSuccess) {
            cudaGetLastError();
            set_error("cudaMalloc of " + std::to_string(bytes) + " bytes failed");
            return false;
        }
        return true;
    };
    if (!alloc((void **)&P->psi, P->arr_n * sizeof(double2))) return fail(QVA_ERR_OUT_OF_MEMORY);
    if (G > 1 && d.mixer != QVA_MIXER_SPARSE && !alloc((void **)&P->psi_alt, P->arr_n * sizeof(double2)))
        return fail(QVA_ERR_OUT_OF_MEMORY);
    if (!alloc((void **)&P->red, (size_t)P->max_batch * 2 * sizeof(double))) return fail(QVA_ERR_OUT_OF_MEMORY);
    if (!alloc((void **)&P->d_flag, sizeof(int))) return fail(QVA_ERR_OUT_OF_MEMORY);
    P->thetas_cap = 256;
    if (!alloc((void **)&P->d_thetas, P->thetas_cap * sizeof(double))) return fail(QVA_ERR_OUT_OF_MEMORY);
    if (P->max_batch > 1) {
        if (!alloc((void **)&P->batch_psi, (size_t)P->max_batch * P->arr_n * sizeof(double2)))
            return fail(QVA_ERR_OUT_OF_MEMORY);
    }
    if (d.mixer == QVA_MIXER_X && P->L >= kTileBits) P->sets = make_tile_sets(P->L);
    if (d.mixer == QVA_MIXER_CIRCULANT) {
        const bool force3 = d.reserved[2] != 0;
        qva_status s = fft_plan_create(P->N, P->device, G, force3, &P->fft);
        if (s != QVA_OK) return fail(s);
        {
            const FftShape sh = fft_plan_shape(P->N, G, force3);
            P->fft_M1 = sh.M1;
            P->fft_M2 = sh.levels == 3 ? sh.Mi1 * sh.Mi2 : sh.M2;
        }
        if (G > 1 && !fft_shardable(P->fft, G)) {
            set_error("sharded circulant mixer: dim " + std::to_string(P->N) + " has no four-step split M1*M2 with " +
                      std::to_string(G) + " | M1 and M2 (prime-heavy dims need the single-GPU Bluestein path)");
            return fail(QVA_ERR_UNSUPPORTED);
        }
    }
    if (d.world > 1 && transport) {
        P->host_tp = true;
        P->tp = *transport;
    } else if (d.world > 1) {
        if (!d.nccl_unique_id) {
            set_error("world > 1 needs nccl_unique_id");
            return fail(QVA_ERR_INVALID_ARGUMENT);
        }
        ncclUniqueId id;
        memcpy(&id, d.nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&P->comm, d.world, id, d.rank);
        if (r != ncclSuccess) {
            set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
            return fail(QVA_ERR_NCCL);
        }
    }
    if (d.world > 1 && (d.mixer == QVA_MIXER_X || d.mixer == QVA_MIXER_CIRCULANT ||
                        (d.mixer == QVA_MIXER_PARITY && !replicated)))
        setup_peer_exchange(P);  // falls back to NCCL on failure (QAOAz: no fallback, see parity_sharded_run)
    if (reset_state(P) != QVA_OK) return fail(QVA_ERR_CUDA);
    if (cudaStreamSynchronize(P->stream) != cudaSuccess) {
        set_error("plan init failed");
        return fail(QVA_ERR_CUDA);
    }
    P->created = true;
    *out = P;
    return QVA_OK;
}

qva_status qva_plan_get_partition(const qva_plan *P, uint64_t *local_n, uint64_t *offset) {
    if (!P || !local_n || !offset) return QVA_ERR_INVALID_ARGUMENT;
    *local_n = P->local_n;
    *offset = P->offset;
    return QVA_OK;
}

static qva_status set_q_common(qva_plan *P, const double *src, bool device, uint64_t offset, uint64_t count) {
    uint64_t lo;
    QVA_TRY(check_range(P, offset, count, &lo));
    if (count == 0) return QVA_OK;
    QVA_TRY(ensure_q_alloc(P));
    if (P->q_graph) {  // a partial upload overwrites part of the graph's q: materialise it first
        QVA_TRY(ensure_q_dev(P));
        P->q_graph = false;
    }
    QVA_CUDA_TRY(cudaMemcpyAsync(P->q + lo, src, count * sizeof(double),
                                 device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, P->stream));
    QVA_CUDA_TRY(cudaMemsetAsync(P->d_flag, 0, sizeof(int), P->stream));
    QVA_CUDA_TRY(launch_check_finite(P->q + lo, count, P->d_flag, P->stream));
    int flag = 0;
    QVA_CUDA_TRY(cudaMemcpyAsync(&flag, P->d_flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    QVA_TRY(sync(P));
    if (flag) {
        set_error("non-finite quality value");
        return QVA_ERR_NUMERIC;
    }
    P->q_set = true;
    P->qB_valid = false;
    P->q_classified = false;
    P->q_mode = 0;
    drop_qt(P);
    return QVA_OK;
}

qva_status qva_set_qualities(qva_plan *P, const double *q, uint64_t offset, uint64_t count) {
    NvtxRange nvtx_range_("qva_set_qualities");
    if (!P || (!q && count)) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    return set_q_common(P, q, false, offset, count);
}

qva_status qva_set_qualities_device(qva_plan *P, const double *q, uint64_t offset, uint64_t count) {
    NvtxRange nvtx_range_("qva_set_qualities_device");
    if (!P || (!q && count)) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    return set_q_common(P, q, true, offset, count);
}

qva_status qva_set_qualities_maxcut(qva_plan *P, int32_t m, const int32_t *u, const int32_t *v, const double *w) {
    NvtxRange nvtx_range_("qva_set_qualities_maxcut");
    if (!P || m < 0 || (m > 0 && (!u || !v))) return QVA_ERR_INVALID_ARGUMENT;
    if (P->mixer != QVA_MIXER_X && P->mixer != QVA_MIXER_PARITY) {
        set_error("qva_set_qualities_maxcut: qubit (X / parity mixer) plans only");
        return QVA_ERR_UNSUPPORTED;
    }
    for (int e = 0; e < m; ++e) {
        if (u[e] < 0 || u[e] >= P->n || v[e] < 0 || v[e] >= P->n) {
            set_error("edge vertex out of range");
            return QVA_ERR_INVALID_ARGUMENT;
        }
        if (w && !std::isfinite(w[e])) {
            set_error("non-finite edge weight");
            return QVA_ERR_NUMERIC;
        }
    }
    DeviceGuard dg(P->device);
    // the graph is the input: q_x = -cut_w(x) is generated where it is consumed (tile passes) or
    // materialised on demand by ensure_q_dev (observables computed in parallel)
    P->g_m = m;
    P->g_unit = (w == nullptr);
    P->g_u.assign(u, u + m);
    P->g_v.assign(v, v + m);
    if (w) P->g_w.assign(w, w + m);
    else P->g_w.clear();
    P->q_graph = true;
    P->q_dev_valid = false;
    P->q_set = true;
    P->qB_valid = false;
    P->q_classified = false;
    P->q_mode = 0;
    drop_qt(P);
    return QVA_OK;
}

qva_status qva_set_qualities_permutation(qva_plan *P, int32_t m, int32_t k, const double *F, const double *D,
                                         const double *lin) {
    NvtxRange nvtx_range_("qva_set_qualities_permutation");
    if (!P || m < 1 || m > kKpermMaxMHost || k < 1 || k > m || (F && !D)) {
        set_error("qva_set_qualities_permutation: need 1 <= k <= m <= 20 (and D with F)");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    uint64_t total = 1;
    for (int a = 0; a < k; ++a) total *= (uint64_t)(m - a);  // m!/(m-k)! <= 20! < 2^64
    if (total != P->N) {
        set_error("qva_set_qualities_permutation: plan dim " + std::to_string(P->N) + " != m!/(m-k)! = " +
                  std::to_string(total));
        return QVA_ERR_SIZE_MISMATCH;
    }
    auto finite = [](const double *x, size_t n) {
        for (size_t i = 0; i < n; ++i)
            if (!std::isfinite(x[i])) return false;
        return true;
    };
    if ((F && !finite(F, (size_t)k * k)) || (D && !finite(D, (size_t)m * m)) || (lin && !finite(lin, (size_t)k * m))) {
        set_error("non-finite permutation cost data");
        return QVA_ERR_NUMERIC;
    }
    // pack: cnt[k] u64, D[m*m], lin[k*m], fv[nf] f64, frow[k+1], fab[nf] int
    std::vector<uint64_t> cnt(k);
    for (int a = 0; a < k; ++a) {
        uint64_t c = 1;
        for (int t = a + 1; t < k; ++t) c *= (uint64_t)(m - t);  // (m-a-1)!/(m-k)!
        cnt[a] = c;
    }
    std::vector<double> fv;
    std::vector<int> frow(k + 1, 0), fab;
    for (int a = 0; a < k; ++a) {
        frow[a] = (int)fv.size();
        if (F)
            for (int b = 0; b < k; ++b)
                if (F[(size_t)a * k + b] != 0.0) {
                    fv.push_back(F[(size_t)a * k + b]);
                    fab.push_back(a << 8 | b);
                }
    }
    frow[k] = (int)fv.size();
    const int nf = (int)fv.size();
    if (nf > kKpermMaxNfHost) {
        set_error("qva_set_qualities_permutation: more than 400 nonzero F entries");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    std::vector<unsigned char> pack;
    auto put = [&](const void *src, size_t n) {
        const unsigned char *c = (const unsigned char *)src;
        pack.insert(pack.end(), c, c + n);
    };
    put(cnt.data(), cnt.size() * sizeof(uint64_t));
    std::vector<double> Dv(D ? D : nullptr, D ? D + (size_t)m * m : nullptr);
    Dv.resize((size_t)m * m, 0.0);
    put(Dv.data(), Dv.size() * sizeof(double));
    if (lin) put(lin, (size_t)k * m * sizeof(double));
    put(fv.data(), fv.size() * sizeof(double));
    put(frow.data(), frow.size() * sizeof(int));
    put(fab.data(), fab.size() * sizeof(int));
    DeviceGuard dg(P->device);
    QVA_TRY(ensure_q_alloc(P));
    void *dpack = nullptr;
    QVA_CUDA_TRY(scratch_get(P, &dpack, pack.size()));
    QVA_TRY(upload(P, dpack, pack.data(), pack.size()));
    {
        ProfScope ps(P, K_OTHER, 8.0 * P->local_n);
        QVA_CUDA_TRY(launch_kperm_q(P->q, P->local_n, P->offset, m, k, dpack, nf, lin != nullptr, P->stream));
    }
    P->q_graph = false;  // the whole partition is overwritten
    P->q_dev_valid = true;
    QVA_CUDA_TRY(cudaMemsetAsync(P->d_flag, 0, sizeof(int), P->stream));
    QVA_CUDA_TRY(launch_check_finite(P->q, P->local_n, P->d_flag, P->stream));
    int flag = 0;
    QVA_CUDA_TRY(cudaMemcpyAsync(&flag, P->d_flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
    QVA_TRY(sync(P));
    P->qB_valid = false;
    P->q_classified = false;
    P->q_mode = 0;
    drop_qt(P);
    if (flag) {
        P->q_set = false;
        set_error("non-finite permutation quality (overflow)");
        return QVA_ERR_NUMERIC;
    }
    P->q_set = true;
    return QVA_OK;
}


qva_status qva_get_qualities(qva_plan *P, double *q_out, uint64_t offset, uint64_t count) {
    if (!P || (!q_out && count)) return QVA_ERR_INVALID_ARGUMENT;
    uint64_t lo;
    QVA_TRY(check_range(P, offset, count, &lo));
    DeviceGuard dg(P->device);
    QVA_TRY(ensure_q_dev(P));
    if (count)
        QVA_CUDA_TRY(cudaMemcpyAsync(q_out, P->q + lo, count * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    return sync(P);
}

qva_status qva_set_circulant_eigenvalues(qva_plan *P, const double *lambda, uint64_t offset, uint64_t count) {
    if (!P || (!lambda && count)) return QVA_ERR_INVALID_ARGUMENT;
    if (P->mixer != QVA_MIXER_CIRCULANT) {
        set_error("not a circulant-mixer plan");
        return QVA_ERR_UNSUPPORTED;
    }
    if (offset > P->N || count > P->N - offset) {
        set_error("eigenvalue range outside [0, dim)");
        return QVA_ERR_SIZE_MISMATCH;
    }
    for (uint64_t i = 0; i < count; ++i)
        if (!std::isfinite(lambda[i])) {
            set_error("non-finite eigenvalue");
            return QVA_ERR_NUMERIC;
        }
    DeviceGuard dg(P->device);
    if (P->lambda_host.size() != P->N) P->lambda_host.assign(P->N, 0.0);
    std::copy(lambda, lambda + count, P->lambda_host.begin() + offset);
    if (!P->lambda_perm) QVA_CUDA_TRY(cudaMalloc(&P->lambda_perm, P->N * sizeof(double)));
    std::vector<double> perm(P->N);
    fft_permute_spectrum(P->fft, P->lambda_host.data(), perm.data());
    QVA_CUDA_TRY(cudaMemcpyAsync(P->lambda_perm, perm.data(), P->N * sizeof(double), cudaMemcpyHostToDevice,
                                 P->stream));
    QVA_TRY(sync(P));
    P->lam_set = true;
    P->lam_const = false;
    return QVA_OK;
}

qva_status qva_set_circulant_eigenvalues_const(qva_plan *P, double lambda0, double c) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    if (P->mixer != QVA_MIXER_CIRCULANT) {
        set_error("not a circulant-mixer plan");
        return QVA_ERR_UNSUPPORTED;
    }
    if (!std::isfinite(lambda0) || !std::isfinite(c)) {
        set_error("non-finite eigenvalue");
        return QVA_ERR_NUMERIC;
    }
    P->lam_set = true;
    P->lam_const = true;
    P->lam0 = lambda0;
    P->lamc = c;
    return QVA_OK;
}

qva_status qva_set_parity_mixer(qva_plan *P, const int32_t *qubits, int32_t count) {
    if (!P || !qubits || count < 2) {
        set_error("qva_set_parity_mixer: need at least 2 qubits");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    if (P->mixer != QVA_MIXER_PARITY) {
        set_error("not a parity-mixer plan");
        return QVA_ERR_UNSUPPORTED;
    }
    std::vector<int> seen(P->n, 0), seq(count);
    for (int i = 0; i < count; ++i) {
        if (qubits[i] < 0 || qubits[i] >= P->n || seen[qubits[i]]++) {
            set_error("qva_set_parity_mixer: qubit index outside [0, n) or repeated");
            return QVA_ERR_INVALID_ARGUMENT;
        }
        seq[i] = qubits[i];
    }
    P->parity_seq = seq;
    return QVA_OK;
}

qva_status qva_set_sparse_mixer(qva_plan *P, const int64_t *row_ptr, const int32_t *col, const double *val,
                                uint64_t nnz) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    if (P->world > 1 && !P->replicated) {
        set_error("world > 1: each rank passes its own rows with qva_set_sparse_mixer_rows");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    return qva_set_sparse_mixer_rows(P, row_ptr, col, val, 0, P->N, nnz);
}

// Row-partitioned W (the paper's distributed SpMV): this rank's rows
// [row_offset, row_offset + rows) = its COMM-psi partition, global column indices.  Collective for
// world > 1: the global ||W||_1 (max-allreduce) and the IPC handles of every rank's Taylor buffers
// (the SpMV reads remote columns straight from the peers' buffers; if any rank cannot map them,
// all fall back to gathering each term vector).
qva_status qva_set_sparse_mixer_rows(qva_plan *P, const int64_t *row_ptr, const int32_t *col, const double *val,
                                     uint64_t row_offset, uint64_t rows, uint64_t nnz) {
    if (!P || !row_ptr || (nnz && !col)) return QVA_ERR_INVALID_ARGUMENT;
    if (P->mixer != QVA_MIXER_SPARSE) {
        set_error("not a sparse-mixer plan");
        return QVA_ERR_UNSUPPORTED;
    }
    if (row_offset != P->offset || rows != P->local_n) {
        set_error("qva_set_sparse_mixer_rows: rows must be this rank's partition [" + std::to_string(P->offset) + ", " +
                  std::to_string(P->offset + P->local_n) + ")");
        return QVA_ERR_SIZE_MISMATCH;
    }
    const bool sharded = P->world > 1 && !P->replicated;
    if (row_ptr[0] != 0 || (uint64_t)row_ptr[rows] != nnz) {
        set_error("row_ptr[0] must be 0 and row_ptr[rows] == nnz");
        return QVA_ERR_SIZE_MISMATCH;
    }
    // ||W||_1 = max_j sum_i |w_ij| = max row abs sum for symmetric W (reading R13); validate
    double norm1 = 0.0;
    qva_status bad = QVA_OK;
    for (uint64_t r = 0; r < rows && bad == QVA_OK; ++r) {
        if (row_ptr[r + 1] < row_ptr[r]) {
            set_error("row_ptr not monotone");
            bad = QVA_ERR_INVALID_ARGUMENT;
            break;
        }
        double sum = 0.0;
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            if (col[k] < 0 || (uint64_t)col[k] >= P->N) {
                set_error("column index out of range");
                bad = QVA_ERR_INVALID_ARGUMENT;
                break;
            }
            double v = val ? val[k] : 1.0;
            if (!std::isfinite(v)) {
                set_error("non-finite matrix entry");
                bad = QVA_ERR_NUMERIC;
                break;
            }
            sum += fabs(v);
        }
        norm1 = std::max(norm1, sum);
    }
    DeviceGuard dg(P->device);
    if (sharded) {  // every rank joins the collectives below even when its own rows were rejected
        double v[3] = {norm1, bad == QVA_OK ? 0.0 : 1.0, 0.0};
        QVA_TRY(coll_allreduce_host(P, v, 3, kCollMax));
        if (bad != QVA_OK) return bad;
        if (v[1] != 0.0) {
            set_error("another rank rejected its rows of W");
            return QVA_ERR_INVALID_ARGUMENT;
        }
        norm1 = v[0];
    } else if (bad != QVA_OK) {
        return bad;
    }
    SparseMixer &sm = P->sm;
    cudaFree(sm.row_ptr);
    cudaFree(sm.col);
    cudaFree(sm.val);
    sm.row_ptr = nullptr; sm.col = nullptr; sm.val = nullptr;
    QVA_CUDA_TRY(cudaMalloc(&sm.row_ptr, (rows + 1) * sizeof(int64_t)));
    QVA_CUDA_TRY(cudaMalloc(&sm.col, std::max<uint64_t>(nnz, 1) * sizeof(int32_t)));
    QVA_CUDA_TRY(cudaMemcpyAsync(sm.row_ptr, row_ptr, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, P->stream));
    if (nnz) QVA_CUDA_TRY(cudaMemcpyAsync(sm.col, col, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, P->stream));
    if (val) {
        QVA_CUDA_TRY(cudaMalloc(&sm.val, std::max<uint64_t>(nnz, 1) * sizeof(double)));
        if (nnz) QVA_CUDA_TRY(cudaMemcpyAsync(sm.val, val, nnz * sizeof(double), cudaMemcpyHostToDevice, P->stream));
    }
    // Taylor buffers: the largest partition's length on every rank (the gather fallback moves
    // equal slices)
    uint64_t stride = rows;
    if (sharded) {
        uint64_t n0, o0;
        qva_partition(P->N, P->world, 0, &n0, &o0);  // rank 0 holds the largest block (R16)
        stride = n0;
    }
    if (!sm.t0) QVA_CUDA_TRY(cudaMalloc(&sm.t0, std::max<uint64_t>(stride, 1) * sizeof(double2)));
    if (!sm.t1) QVA_CUDA_TRY(cudaMalloc(&sm.t1, std::max<uint64_t>(stride, 1) * sizeof(double2)));
    sm.nnz = nnz;
    sm.rows = rows;
    sm.norm1 = norm1;
    if (sharded && sm.src.G == 1) {  // first call: map the peers' Taylor buffers (collective)
        SpmvSource src;
        src.G = P->world;
        for (int r = 0; r <= P->world; ++r) {
            uint64_t n_r, o_r;
            if (r < P->world) {
                qva_partition(P->N, P->world, r, &n_r, &o_r);
                src.off[r] = o_r;
            } else {
                src.off[r] = P->N;
            }
        }
        const size_t hb = sizeof(cudaIpcMemHandle_t);
        std::vector<unsigned char> mine(2 * hb, 0), all(2 * hb * P->world, 0);
        bool ok = fuse_exchange_enabled() && P->world <= kMaxPeers &&
                  cudaIpcGetMemHandle((cudaIpcMemHandle_t *)mine.data(), sm.t0) == cudaSuccess &&
                  cudaIpcGetMemHandle((cudaIpcMemHandle_t *)(mine.data() + hb), sm.t1) == cudaSuccess;
        cudaGetLastError();
        unsigned char *stage = nullptr;
        QVA_CUDA_TRY(scratch_get(P, (void **)&stage, (P->world + 1) * 2 * hb));
        ok = (coll_allgather_host(P, mine.data(), all.data(), 2 * hb, stage) == QVA_OK) && ok;
        for (int t = 0; ok && t < P->world; ++t)
            for (int k = 0; ok && k < 2; ++k) {
                if (t == P->rank) {
                    src.peer[k][t] = k ? sm.t1 : sm.t0;
                    continue;
                }
                cudaIpcMemHandle_t h;
                memcpy(&h, all.data() + (2 * t + k) * hb, hb);
                void *ptr = nullptr;
                ok = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
                src.peer[k][t] = (const double2 *)ptr;
            }
        cudaGetLastError();
        double flag = ok ? 1.0 : 0.0;
        if (coll_allreduce_host(P, &flag, 1, kCollMin) != QVA_OK) flag = 0.0;
        if (flag == 1.0) {
            sm.peer_ok = true;
        } else {  // unmap what was mapped; gather each term instead
            for (int k = 0; k < 2; ++k)
                for (int t = 0; t < P->world; ++t)
                    if (t != P->rank && src.peer[k][t]) cudaIpcCloseMemHandle((void *)src.peer[k][t]);
            memset(src.peer, 0, sizeof(src.peer));
            cudaGetLastError();
            QVA_CUDA_TRY(cudaMalloc(&sm.gather_buf, (size_t)P->world * stride * sizeof(double2)));
            src.gathered = sm.gather_buf;
        }
        src.stride = stride;
        sm.src = src;
        if (!P->host_tp && !P->d_bar) QVA_CUDA_TRY(cudaMalloc(&P->d_bar, sizeof(int)));
    }
    QVA_TRY(sync(P));
    P->sparse_set = true;
    return QVA_OK;
}

qva_status qva_set_initial_state(qva_plan *P, const double *re_im, uint64_t offset, uint64_t count) {
    if (!P || (!re_im && count)) return QVA_ERR_INVALID_ARGUMENT;
    uint64_t lo;
    QVA_TRY(check_range(P, offset, count, &lo));
    DeviceGuard dg(P->device);
    if (!P->psi0) {
        QVA_CUDA_TRY(cudaMalloc(&P->psi0, P->arr_n * sizeof(double2)));
        QVA_CUDA_TRY(cudaMemsetAsync(P->psi0, 0, P->arr_n * sizeof(double2), P->stream));
    }
    for (uint64_t i = 0; i < 2 * count; ++i)
        if (!std::isfinite(re_im[i])) {
            set_error("non-finite initial amplitude");
            return QVA_ERR_NUMERIC;
        }
    if (count)
        QVA_CUDA_TRY(cudaMemcpyAsync(P->psi0 + lo, re_im, count * sizeof(double2), cudaMemcpyHostToDevice, P->stream));
    QVA_TRY(sync(P));
    P->has_psi0 = true;
    return QVA_OK;
}

qva_status qva_clear_initial_state(qva_plan *P) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    P->has_psi0 = false;
    return QVA_OK;
}

qva_status qva_reset_state(qva_plan *P) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    QVA_TRY(reset_state(P));
    P->expect_valid = false;
    return sync(P);
}

static const double *q_current(qva_plan *P) { return (P->layout == 1) ? P->qB : P->q; }

qva_status qva_apply_phase(qva_plan *P, double gamma) {
    NvtxRange nvtx_range_("qva_apply_phase");
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    if (!std::isfinite(gamma)) {
        set_error("non-finite gamma");
        return QVA_ERR_NUMERIC;
    }
    if (!P->q_set) {
        set_error("qualities not set");
        return QVA_ERR_NOT_READY;
    }
    DeviceGuard dg(P->device);
    QVA_TRY(to_natural_perm(P));
    QVA_TRY(ensure_q_dev(P));
    if (P->layout == 1) QVA_TRY(ensure_qB(P));
    {
        ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
        QVA_CUDA_TRY(launch_phase(P->psi, q_current(P), P->arr_n, gamma, P->stream));
    }
    P->expect_valid = false;
    return sync(P);
}

qva_status qva_apply_mixer(qva_plan *P, double beta) {
    NvtxRange nvtx_range_("qva_apply_mixer");
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    if (!std::isfinite(beta)) {
        set_error("non-finite beta");
        return QVA_ERR_NUMERIC;
    }
    DeviceGuard dg(P->device);
    P->expect_valid = false;
    QVA_TRY(to_natural_perm(P));
    QVA_TRY(apply_mixer_impl(P, beta));
    return sync(P);
}

// X-mixer evolution through the tile passes (permuted or in-place schedule); graph: allow CUDA
// graph replay of the single-shard sequence
static qva_status x_tile_evolve(qva_plan *P, const double *theta, int p, bool graph, bool *have_red) {
    P->layout = 0;
    P->perm.clear();
    if (p == 0) {
        QVA_TRY(reset_state(P));
        return QVA_OK;
    }
    if (use_permuted(P)) {
        if (!P->psi_alt && cudaMalloc(&P->psi_alt, P->arr_n * sizeof(double2)) != cudaSuccess) {
            cudaGetLastError();
            P->perm_failed = true;  // no room for the ping-pong buffer: in-place schedule
        }
    }
    if (use_permuted(P)) {
        // the schedule depends on (L, p) only: planned once per p (host planning off the step path)
        auto it = P->perm_sched.find(p);
        if (it == P->perm_sched.end()) {
            std::vector<int> fin;
            auto passes = perm_passes(P->L, p, &fin);
            if (passes.empty() || !passes.back().expect) {
                set_error("internal: permuted schedule did not complete");
                return QVA_ERR_UNSUPPORTED;
            }
            it = P->perm_sched.emplace(p, std::make_pair(std::move(passes), std::move(fin))).first;
        }
        QVA_TRY(graph ? run_passes_graph(P, it->second.first, theta, p, P->has_psi0 ? 2 : 1)
                      : run_passes(P, it->second.first, theta, p, 1, P->psi, 0, P->has_psi0 ? 2 : 1, nullptr));
        P->perm = it->second.second;
        *have_red = true;
        return QVA_OK;
    }
    auto passes = cut_passes(evolve_tokens(P->L, P->gbits, p), P->sets, true);
    QVA_TRY(run_passes(P, passes, theta, p, 1, P->psi, 0, P->has_psi0 ? 2 : 1, nullptr));
    *have_red = true;
    return QVA_OK;
}

// one full evolution of the plan's own state; on return P->red holds (f, norm) (local sums)
static qva_status evolve_impl(qva_plan *P, const double *theta, int p, bool *have_red) {
    *have_red = false;
    if (P->mixer == QVA_MIXER_X) {
        if (use_small(P)) {
            QVA_TRY(ensure_q_dev(P));
            SmallEvolveParams sp{};
            sp.psi = P->psi;
            sp.psi0 = P->has_psi0 ? P->psi0 : nullptr;
            sp.q = P->q;
            sp.n = P->n;
            sp.p = p;
            sp.mode = 0;
            sp.out = P->red;
            QVA_TRY(upload(P, P->d_thetas, theta, 2 * p * sizeof(double)));
            sp.thetas = P->d_thetas;
            {
                ProfScope ps(P, K_SMALL, 24.0 * P->arr_n);
                QVA_CUDA_TRY(launch_small_evolve(sp, 1, P->stream));
            }
            P->layout = 0;
            *have_red = true;
            return QVA_OK;
        }
        QVA_TRY(x_tile_evolve(P, theta, p, true, have_red));
        return QVA_OK;
    }
    if (P->mixer == QVA_MIXER_CIRCULANT) {
        if (!P->lam_set) {
            set_error("circulant spectrum not set");
            return QVA_ERR_NOT_READY;
        }
        FftRun r;
        r.psi = P->psi;
        r.q = P->q;
        r.lambda_perm = P->lam_const ? nullptr : P->lambda_perm;
        r.lam0 = P->lam0;
        r.lamc = P->lamc;
        r.theta = theta;
        r.p = p;
        r.mode = 0;
        if (P->has_psi0 || p == 0) {
            QVA_TRY(reset_state(P));
            r.init = 0;
        } else {
            r.init = 1;
            r.amp0 = 1.0 / sqrt((double)P->N);
        }
        r.expect = p > 0;
        r.red_out = P->red;
        PlanObserver obs(P);
        if (use_complete_closed_form(P)) {
            double *scr = nullptr;
            QVA_CUDA_TRY(scratch_get(P, (void **)&scr, complete_scratch_doubles(P->arr_n) * sizeof(double)));
            PlanCompleteComm cc(P);
            QVA_TRY(complete_run(r, P->arr_n, P->N, scr, P->stream, &obs, P->world > 1 ? &cc : nullptr));
        } else if (P->G > 1) {
            PlanShardIO io(P);
            QVA_TRY(circ_shard_setup(P, io));
            QVA_TRY(fft_run_sharded(P->fft, r, io, P->stream, &obs));
        } else {
            QVA_TRY(fft_run(P->fft, r, P->stream, &obs));
        }
        *have_red = p > 0;
        return QVA_OK;
    }
    if (P->mixer == QVA_MIXER_PARITY) {
        if (p == 0) return reset_state(P);
        P->layout = 0;
        P->perm.clear();
        if (P->world > 1 && !P->replicated) {
            if (!use_qgen(P)) QVA_TRY(ensure_q_dev(P));
            return parity_sharded_run(P, theta, p, have_red, nullptr);
        }
        // tile passes (TMA pipeline, pair terms on register groups; QVA_PARITY_TILE=0: window kernel)
        static int tile_env = [] {
            const char *e = getenv("QVA_PARITY_TILE");
            return e ? atoi(e) : 1;
        }();
        if (tile_env) {
            auto it = P->parity_tile_sched.find(p);
            if (it == P->parity_tile_sched.end() || P->parity_tile_seq != P->parity_seq) {
                if (P->parity_tile_seq != P->parity_seq) P->parity_tile_sched.clear();
                P->parity_tile_seq = P->parity_seq;
                std::vector<PassPlan> passes;
                if (!parity_tile_passes(P->n, P->L, P->G, P->parity_seq, p, passes)) passes.clear();
                it = P->parity_tile_sched.emplace(p, std::move(passes)).first;
            }
            P->parity_tile_ran = !it->second.empty();
            if (!it->second.empty()) {
                if (!use_qgen(P)) QVA_TRY(ensure_q_dev(P));
                QVA_TRY(run_passes(P, it->second, theta, p, 1, P->psi, 0, P->has_psi0 ? 2 : 1, nullptr));
                *have_red = true;
                return QVA_OK;
            }
        }
        QVA_TRY(ensure_q_dev(P));
        for (int k = 0; k < p; ++k) QVA_TRY(parity_mix(P, theta[2 * k + 1], P->q, theta[2 * k], k == 0));
        return QVA_OK;
    }
    // sparse
    if (!P->sparse_set) {
        set_error("sparse mixer not set");
        return QVA_ERR_NOT_READY;
    }
    QVA_TRY(reset_state(P));
    for (int k = 0; k < p; ++k) {
        {
            ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
            QVA_CUDA_TRY(launch_phase(P->psi, P->q, P->arr_n, theta[2 * k], P->stream));
        }
        int terms = 0;
        PlanObserver obs(P);
        PlanSparseComm comm(P);
        QVA_TRY(sparse_apply_mixer(P->sm, P->psi, theta[2 * k + 1], P->stream, &obs, &terms,
                                   (P->world > 1 && !P->replicated) ? &comm : nullptr));
    }
    return QVA_OK;
}

qva_status qva_evolve(qva_plan *P, const double *theta, int32_t p) {
    NvtxRange nvtx_range_("qva_evolve");
    if (!P || p < 0 || (p > 0 && !theta)) return QVA_ERR_INVALID_ARGUMENT;
    QVA_TRY(check_theta(theta, 2 * (size_t)p));
    if (!P->q_set) {
        set_error("qualities not set (PAPER.md:649: set_qualities is required)");
        return QVA_ERR_NOT_READY;
    }
    if ((size_t)2 * p > P->thetas_cap) {
        set_error("p too large");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    DeviceGuard dg(P->device);
    P->expect_valid = false;
    bool have = false;
    QVA_TRY(evolve_impl(P, theta, p, &have));
    if (have) {
        double pair[2];
        QVA_CUDA_TRY(cudaMemcpyAsync(pair, P->red, sizeof(pair), cudaMemcpyDeviceToHost, P->stream));
        QVA_TRY(sync(P));
        if (!P->replicated) QVA_TRY(allreduce_host(P, pair, 2));
        P->expect_val = pair[0];
        P->norm_val = pair[1];
        P->expect_valid = true;
        return QVA_OK;
    }
    return sync(P);
}

// ---- ex-QAOA (Eqs. phase_shift_qaoa_ex / qaoa_ex; reading R25) -------------
// theta = per layer [gamma_{i,1..m}, t_i].  Layer i's phase prod_e exp(-i gamma_{i,e} Sigma_e) with
// Sigma_e = -w_e [x_u != x_v] is exp(+i cut_{w'}) for the per-layer weights w'_e = gamma_{i,e} w_e,
// i.e. the generated max-cut phase with gamma = 1: the tile passes build per-layer records of w'
// (the <Q> pass keeps the plan's w).  Other plans (small, parity mixer, shards whose phase and <Q>
// share a pass) take the step path: generate -cut_{w'} per layer, phase with gamma = 1, mixer.
static qva_status ex_impl(qva_plan *P, const double *theta, int p, bool *have_red) {
    *have_red = false;
    const int m = P->g_m;
    std::vector<double> wx((size_t)p * m), th2(2 * (size_t)p);
    for (int i = 0; i < p; ++i) {
        const double *t = theta + (size_t)i * (m + 1);
        for (int e = 0; e < m; ++e) wx[(size_t)i * m + e] = t[e] * (P->g_unit ? 1.0 : P->g_w[e]);
        th2[2 * i] = 1.0;
        th2[2 * i + 1] = t[m];
    }
    bool tile = P->mixer == QVA_MIXER_X && !use_small(P) && use_qgen(P) && p > 0;
    if (tile && !use_permuted(P)) {
        auto passes = cut_passes(evolve_tokens(P->L, P->gbits, p), P->sets, true);
        for (auto &pp : passes)
            if (pp.phase >= 0 && pp.expect) tile = false;
    }
    if (tile) {
        P->ex_w = wx.data();
        qva_status st = x_tile_evolve(P, th2.data(), p, false, have_red);
        P->ex_w = nullptr;
        return st;
    }
    QVA_TRY(reset_state(P));
    if (p == 0) return QVA_OK;
    const size_t need = (size_t)std::max(m, 1) * 2 * sizeof(int32_t) + wx.size() * sizeof(double) + 16;
    if (P->ex_edge_cap < need) {
        plan_free(P, P->d_ex_edges);
        P->d_ex_edges = nullptr;
        QVA_CUDA_TRY(cudaMalloc(&P->d_ex_edges, need));
        P->ex_edge_cap = need;
    }
    if (!P->q_ex) QVA_CUDA_TRY(cudaMalloc(&P->q_ex, P->arr_n * sizeof(double)));
    int32_t *du = (int32_t *)P->d_ex_edges, *dv = du + std::max(m, 1);
    double *dw = (double *)((unsigned char *)P->d_ex_edges + (((size_t)std::max(m, 1) * 2 * sizeof(int32_t) + 15) & ~15ull));
    if (m) {
        QVA_TRY(upload(P, du, P->g_u.data(), m * sizeof(int32_t)));
        QVA_TRY(upload(P, dv, P->g_v.data(), m * sizeof(int32_t)));
        QVA_TRY(upload(P, dw, wx.data(), wx.size() * sizeof(double)));
    }
    for (int i = 0; i < p; ++i) {
        QVA_TRY(to_layout_A(P));  // the generated term sum is in natural (partition) order
        {
            ProfScope ps(P, K_OTHER, 8.0 * P->arr_n);
            QVA_CUDA_TRY(launch_maxcut_q(P->q_ex, P->arr_n, P->offset, m, du, dv, dw + (size_t)i * m, P->stream));
        }
        {
            ProfScope ps(P, K_OTHER, 40.0 * P->arr_n);
            QVA_CUDA_TRY(launch_phase(P->psi, P->q_ex, P->arr_n, 1.0, P->stream));
        }
        QVA_TRY(apply_mixer_impl(P, th2[2 * i + 1]));
    }
    return QVA_OK;
}

static qva_status ex_check(qva_plan *P, const double *theta, size_t n_theta) {
    if (!P->q_set || !P->q_graph) {
        set_error("ex-QAOA needs the max-cut graph (qva_set_qualities_maxcut): its terms are the edges");
        return QVA_ERR_NOT_READY;
    }
    if (P->mixer != QVA_MIXER_X && P->mixer != QVA_MIXER_PARITY) {
        set_error("ex-QAOA: qubit (X / parity mixer) plans only");
        return QVA_ERR_UNSUPPORTED;
    }
    return check_theta(theta, n_theta);
}

static qva_status expect_now(qva_plan *P) {
    if (P->expect_valid) return QVA_OK;
    if (!P->q_set) {
        set_error("qualities not set");
        return QVA_ERR_NOT_READY;
    }
    QVA_TRY(to_natural_perm(P));
    QVA_TRY(ensure_q_dev(P));
    if (P->layout == 1) QVA_TRY(ensure_qB(P));
    double pair[2];
    QVA_TRY(expect_generic(P, P->psi, P->arr_n, q_current(P), pair));
    if (!P->replicated) QVA_TRY(allreduce_host(P, pair, 2));
    P->expect_val = pair[0];
    P->norm_val = pair[1];
    P->expect_valid = true;
    return QVA_OK;
}

qva_status qva_expectation(qva_plan *P, double *out) {
    NvtxRange nvtx_range_("qva_expectation");
    if (!P || !out) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    QVA_TRY(expect_now(P));
    *out = P->expect_val;
    return QVA_OK;
}

qva_status qva_norm2(qva_plan *P, double *out) {
    if (!P || !out) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    if (!P->q_set && !P->expect_valid) {
        // norm does not need q: use zeros already in P->q
        double pair[2];
        QVA_TRY(expect_generic(P, P->psi, P->arr_n, P->q, pair));
        if (!P->replicated) QVA_TRY(allreduce_host(P, pair, 2));
        *out = pair[1];
        return QVA_OK;
    }
    QVA_TRY(expect_now(P));
    *out = P->norm_val;
    return QVA_OK;
}

qva_status qva_get_state(qva_plan *P, double *re_im, uint64_t offset, uint64_t count) {
    if (!P || (!re_im && count)) return QVA_ERR_INVALID_ARGUMENT;
    uint64_t lo;
    QVA_TRY(check_range(P, offset, count, &lo));
    DeviceGuard dg(P->device);
    if (P->layout == 1 || !P->perm.empty()) {
        bool ev = P->expect_valid;
        QVA_TRY(to_layout_A(P));
        P->expect_valid = ev;
    }
    if (count)
        QVA_CUDA_TRY(cudaMemcpyAsync(re_im, P->psi + lo, count * sizeof(double2), cudaMemcpyDeviceToHost, P->stream));
    return sync(P);
}

qva_status qva_get_probabilities(qva_plan *P, double *out, uint64_t offset, uint64_t count) {
    if (!P || (!out && count)) return QVA_ERR_INVALID_ARGUMENT;
    uint64_t lo;
    QVA_TRY(check_range(P, offset, count, &lo));
    if (!count) return QVA_OK;
    DeviceGuard dg(P->device);
    if (P->layout == 1 || !P->perm.empty()) {
        bool ev = P->expect_valid;
        QVA_TRY(to_layout_A(P));
        P->expect_valid = ev;
    }
    double *d;
    QVA_CUDA_TRY(scratch_get(P, (void **)&d, count * sizeof(double)));
    {
        ProfScope ps(P, K_OTHER, 24.0 * count);
        QVA_CUDA_TRY(launch_probabilities(P->psi + lo, d, count, P->stream));
    }
    QVA_CUDA_TRY(cudaMemcpyAsync(out, d, count * sizeof(double), cudaMemcpyDeviceToHost, P->stream));
    return sync(P);
}

// batch members [first, first+count) -> vals[2*i] (local sums; not reduced over COMM-psi)
static qva_status batch_local(qva_plan *P, const double *thetas, int first, int count, int p, double *f_out) {
    if (count <= 0) return QVA_OK;
    const double *th = thetas + (size_t)first * 2 * p;
    if (P->mixer == QVA_MIXER_X && P->G == 1 && (use_small(P) || P->batch_psi)) {
        int chunk = use_small(P) ? count : std::min(std::min(count, P->max_batch), kMaxBatchSmem);
        for (int b0 = 0; b0 < count; b0 += chunk) {
            int nb = std::min(chunk, count - b0);
            std::vector<double> pairs(2 * (size_t)nb);
            if (use_small(P)) {
                QVA_TRY(ensure_q_dev(P));
                size_t need = (size_t)nb * 2 * p;
                if (need > P->thetas_cap) {
                    plan_free(P, P->d_thetas);
                    P->d_thetas = nullptr;
                    QVA_CUDA_TRY(cudaMalloc(&P->d_thetas, need * sizeof(double)));
                    P->thetas_cap = need;
                }
                if ((size_t)nb > (size_t)P->max_batch) {
                    plan_free(P, P->red);
                    P->red = nullptr;
                    QVA_CUDA_TRY(cudaMalloc(&P->red, (size_t)nb * 2 * sizeof(double)));
                    P->max_batch = nb;
                }
                if (P->small_batch_cap < (size_t)nb * P->arr_n) {
                    plan_free(P, P->small_batch);
                    P->small_batch = nullptr;
                    QVA_CUDA_TRY(cudaMalloc(&P->small_batch, (size_t)nb * P->arr_n * sizeof(double2)));
                    P->small_batch_cap = (size_t)nb * P->arr_n;
                }
                double2 *bpsi = P->small_batch;
                QVA_CUDA_TRY(cudaMemcpyAsync(P->d_thetas, th + (size_t)b0 * 2 * p, need * sizeof(double),
                                             cudaMemcpyHostToDevice, P->stream));
                SmallEvolveParams sp{};
                sp.psi = bpsi;
                sp.psi0 = P->has_psi0 ? P->psi0 : nullptr;
                sp.q = P->q;
                sp.thetas = P->d_thetas;
                sp.out = P->red;
                sp.n = P->n;
                sp.p = p;
                sp.mode = 0;
                {
                    ProfScope ps(P, K_SMALL, 24.0 * P->arr_n * nb);
                    QVA_CUDA_TRY(launch_small_evolve(sp, nb, P->stream));
                }
                QVA_CUDA_TRY(cudaMemcpyAsync(pairs.data(), P->red, pairs.size() * sizeof(double),
                                             cudaMemcpyDeviceToHost, P->stream));
                QVA_TRY(sync(P));
            } else {
                auto passes = cut_passes(evolve_tokens(P->L, 0, p), P->sets, true);
                QVA_TRY(run_passes(P, passes, th + (size_t)b0 * 2 * p, p, nb, P->batch_psi, P->arr_n,
                                   P->has_psi0 ? 2 : 1, pairs.data()));
                QVA_TRY(sync(P));
            }
            for (int i = 0; i < nb; ++i) f_out[b0 + i] = pairs[2 * i];
        }
        return QVA_OK;
    }
    // generic: sequential members on the plan's own state
    for (int i = 0; i < count; ++i) {
        bool have = false;
        QVA_TRY(evolve_impl(P, th + (size_t)i * 2 * p, p, &have));
        double pair[2];
        if (have) {
            QVA_CUDA_TRY(cudaMemcpyAsync(pair, P->red, sizeof(pair), cudaMemcpyDeviceToHost, P->stream));
            QVA_TRY(sync(P));
        } else {
            QVA_TRY(ensure_q_dev(P));
            if (P->layout == 1) QVA_TRY(ensure_qB(P));
            QVA_TRY(expect_generic(P, P->psi, P->arr_n, q_current(P), pair));
        }
        f_out[i] = pair[0];
    }
    return QVA_OK;
}

qva_status qva_evolve_ex(qva_plan *P, const double *theta, int32_t p) {
    NvtxRange nvtx_range_("qva_evolve_ex");
    if (!P || p < 0 || (p > 0 && !theta)) return QVA_ERR_INVALID_ARGUMENT;
    QVA_TRY(ex_check(P, theta, (size_t)p * (P->g_m + 1)));
    DeviceGuard dg(P->device);
    P->expect_valid = false;
    bool have = false;
    QVA_TRY(ex_impl(P, theta, p, &have));
    if (have) {
        double pair[2];
        QVA_CUDA_TRY(cudaMemcpyAsync(pair, P->red, sizeof(pair), cudaMemcpyDeviceToHost, P->stream));
        QVA_TRY(sync(P));
        if (!P->replicated) QVA_TRY(allreduce_host(P, pair, 2));
        P->expect_val = pair[0];
        P->norm_val = pair[1];
        P->expect_valid = true;
        return QVA_OK;
    }
    return sync(P);
}

qva_status qva_evolve_ex_batch(qva_plan *P, const double *thetas, int32_t B, int32_t p, double *f_out) {
    NvtxRange nvtx_range_("qva_evolve_ex_batch");
    if (!P || B < 0 || p < 0 || (B > 0 && (!thetas || !f_out))) return QVA_ERR_INVALID_ARGUMENT;
    const size_t per = (size_t)p * (P->g_m + 1);
    QVA_TRY(ex_check(P, thetas, (size_t)B * per));
    DeviceGuard dg(P->device);
    P->expect_valid = false;
    std::vector<double> f((size_t)B, 0.0);
    int32_t first = 0, cnt = B;
    if (P->replicated && P->world > 1) QVA_TRY(qva_batch_partition(B, P->world, P->rank, &first, &cnt));
    for (int i = first; i < first + cnt; ++i) {  // members one after another on the plan's state
        bool have = false;
        QVA_TRY(ex_impl(P, thetas + (size_t)i * per, p, &have));
        double pair[2];
        if (have) {
            QVA_CUDA_TRY(cudaMemcpyAsync(pair, P->red, sizeof(pair), cudaMemcpyDeviceToHost, P->stream));
            QVA_TRY(sync(P));
        } else {
            QVA_TRY(to_natural_perm(P));
            QVA_TRY(ensure_q_dev(P));
            if (P->layout == 1) QVA_TRY(ensure_qB(P));
            QVA_TRY(expect_generic(P, P->psi, P->arr_n, q_current(P), pair));
        }
        f[i] = pair[0];
    }
    if (P->world > 1) QVA_TRY(allreduce_host(P, f.data(), B));  // replicated: disjoint members; sharded: partial sums
    std::copy(f.begin(), f.end(), f_out);
    return QVA_OK;
}

qva_status qva_evolve_batch(qva_plan *P, const double *thetas, int32_t B, int32_t p, double *f_out) {
    NvtxRange nvtx_range_("qva_evolve_batch");
    if (!P || B < 0 || p < 0 || (B > 0 && (!thetas || !f_out))) return QVA_ERR_INVALID_ARGUMENT;
    QVA_TRY(check_theta(thetas, (size_t)B * 2 * p));
    if (!P->q_set) {
        set_error("qualities not set");
        return QVA_ERR_NOT_READY;
    }
    if ((size_t)2 * p > P->thetas_cap && !use_small(P)) {
        set_error("p too large");
        return QVA_ERR_INVALID_ARGUMENT;
    }
    DeviceGuard dg(P->device);
    P->expect_valid = false;
    std::vector<double> f((size_t)B, 0.0);
    if (P->replicated && P->world > 1) {
        // COMM-grad_f analogue: split the B sets over ranks, then all-reduce
        int32_t first, cnt;
        QVA_TRY(qva_batch_partition(B, P->world, P->rank, &first, &cnt));
        std::vector<double> part(cnt > 0 ? cnt : 1);
        QVA_TRY(batch_local(P, thetas, first, cnt, p, part.data()));
        for (int i = 0; i < cnt; ++i) f[first + i] = part[i];
        QVA_TRY(allreduce_host(P, f.data(), B));
    } else {
        QVA_TRY(batch_local(P, thetas, 0, B, p, f.data()));
        if (!P->replicated && P->world > 1) QVA_TRY(allreduce_host(P, f.data(), B));
    }
    std::copy(f.begin(), f.end(), f_out);
    return QVA_OK;
}

qva_status qva_set_profiling(qva_plan *P, int32_t enable) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    P->prof = enable != 0;
    return QVA_OK;
}

qva_status qva_kernel_stats(qva_plan *P, int32_t which, double *ms, int64_t *launches, double *bytes) {
    if (!P || which < 0 || which >= kKernelClasses) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    QVA_TRY(sync(P));
    if (ms) *ms = P->stats[which].ms;
    if (launches) *launches = P->stats[which].launches;
    if (bytes) *bytes = P->stats[which].bytes;
    return QVA_OK;
}

qva_status qva_reset_kernel_stats(qva_plan *P) {
    if (!P) return QVA_ERR_INVALID_ARGUMENT;
    DeviceGuard dg(P->device);
    QVA_TRY(sync(P));
    for (auto &s : P->stats) s = KernelStat();
    P->launches = 0;
    P->xfer_bytes = 0.0;
    return QVA_OK;
}

qva_status qva_launch_count(qva_plan *P, int64_t *launches) {
    if (!P || !launches) return QVA_ERR_INVALID_ARGUMENT;
    *launches = P->launches;
    return QVA_OK;
}

qva_status qva_plan_query(const qva_plan *P, int32_t what, int64_t *out) {
    if (!P || !out) return QVA_ERR_INVALID_ARGUMENT;
    switch (what) {
        case 0:
            *out = P->world > 1 ? (P->ipc_ok ? 1 : 0)
                                : ((P->G > 1 && fuse_exchange_enabled() && P->d.reserved[3] != 0) ? 1 : 0);
            return QVA_OK;
        case 1: *out = P->G; return QVA_OK;
        case 2: *out = P->host_tp ? 1 : 0; return QVA_OK;
        case 3: *out = P->world; return QVA_OK;
        case 4: *out = P->rank; return QVA_OK;
        case 5: *out = (int64_t)P->xfer_bytes; return QVA_OK;
        case 6: *out = P->parity_tile_ran ? 1 : 0; return QVA_OK;
        case 7: *out = P->sm.peer_ok ? 1 : 0; return QVA_OK;
        default: set_error("qva_plan_query: unknown query"); return QVA_ERR_INVALID_ARGUMENT;
    }
}

}  // extern "C"
