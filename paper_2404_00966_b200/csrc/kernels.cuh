// kernels.cuh -- sm_100a device code of the GTS batch search path.
//
// Device layout (all in HBM, built once per index by gts_index_create):
//   node table   NodeRec[nodes+1] {min f32 (rounded down), max f32 (rounded
//                up), size i32, pivot table-position i32}  16 B, one load
//   node pos     i32[nodes+1]  first table entry of the node's segment
//   object table dis f32[n] (entry -> own leaf pivot), ids i64[n],
//                alive bitmask u32[n/32]   (all in table = leaf order)
//   payloads     vectors: f32 [n][Dp] in table order (Dp = D rounded to 4),
//                optional f64 [n][D] when the data is not fp32-exact;
//                strings: dense u8 symbols in table order + i64 offsets.
// Reference semantics being restated: search.py:28-57 (predicates),
// 405-477 (_expand), 507-538 (_verify_range), metrics.py:54-133 (metrics).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gts {

constexpr int kWarp = 32;
constexpr unsigned kFull = 0xffffffffu;
constexpr int kMetricEdit = 0, kMetricL1 = 1, kMetricL2 = 2, kMetricAngular = 3;
constexpr int kMetricSq = 4;   // pw_sum64 term x*x (norms; the second operand is not read for its value)
constexpr int kMaxWords = 128;      // edit patterns up to 4096 symbols
constexpr uint8_t kNoSym = 0xff;    // query symbol absent from the index alphabet

struct NodeRec {
    float mn, mx;
    int32_t size, piv;
};

struct Row {            // one (query, node, d(q, node pivot)) frontier row
    int32_t q, node;
    float dqp;
    int32_t pad;
};

struct IndexView {
    const NodeRec *node;
    const int32_t *npos;
    const float *dis;
    const uint32_t *alive;
    const float *vec32;
    const double *vec64;   // may be null (fp32-exact data: widen vec32)
    const uint32_t *str;     // dense symbols, 4 per word, each object 4-byte aligned
    const uint32_t *sword;   // [n] first word of each entry's symbols
    const int32_t *slen;     // [n] symbols per entry
    const int32_t *row;      // [n] dataset row of each entry (row order = id order)
    const uint4 *erec;       // [n] edit scan records {dis f32 bits, len, first text word, 0}
    const uint4 *ehist;      // [2n] 32 byte-buckets of symbol counts (symbol % 32), or null
    const uint4 *esig;       // [2n] 256-bit q-gram signature per entry (qgram_sig), or null
    int sig_q;               // q of the signature (4 for alphabets <= 4, else 2); 0: none
    const uint4 *vcent;      // [n][Dk/8] bf16 vectors centred on their leaf pivot (tensor-core L2 path), or null
    const uint4 *vtile;      // the same per leaf, in the MMA's shared-memory image (k_vtile), or null
    const float *vnorm32;    // angular: |o| per entry (fp32 screen), or null
    const double *vnorm64;   // angular: |o| per entry, numpy's pairwise sum of squares
    const float *vse;        // [n] c . vcent_e (pivot . centred bf16 entry), tensor-core path
    int Dk;                  // D rounded up to 64 (one 128-byte bf16 row per K-block)
    int D, Dp, nc, levels;
    int leaf_first, leaf_count, max_leaf;
    float rel, abs_eps;    // fp32 slack model (vectors); 0 for edit
};

struct QueryView {
    const float *vec32;    // [nq][Dp]
    const double *vec64;   // [nq][D]
    const int64_t *soff;   // [nq+1] symbol offsets
    const uint8_t *str;    // dense symbols
    const uint32_t *peq;   // Myers match masks, [A][W] per query
    const int64_t *peq_off;
    const uint4 *qhist;    // [2nq] query symbol histograms (same buckets as ehist)
    const uint4 *qsig;     // [2nq] query q-gram signatures (same mapping as esig)
    const uint4 *qbf;      // [nq][Dk/8] bf16 query rows (tensor-core L2 path)
    const float *qnorm32;  // angular: |q| (fp32 screen)
    const double *qnorm64; // angular: |q|, pairwise sum of squares
    const float *qn;       // [nq] |q| rounded up
    int A;
};

// Symbol-histogram lower bound of the edit distance: every edit changes the
// multiset difference by at most one, so ED >= (SAD(hist_q, hist_o) + |lq - lo|) / 2
// (buckets merge symbols, saturating byte counts only shrink SAD: still a
// lower bound).  Eight byte-SIMD absolute-difference sums.
__device__ __forceinline__ int hist_lb(const uint4 &a0, const uint4 &a1, const uint4 &b0, const uint4 &b1, int dl)
{
    unsigned sad = __vsadu4(a0.x, b0.x) + __vsadu4(a0.y, b0.y) + __vsadu4(a0.z, b0.z) + __vsadu4(a0.w, b0.w) +
                   __vsadu4(a1.x, b1.x) + __vsadu4(a1.y, b1.y) + __vsadu4(a1.z, b1.z) + __vsadu4(a1.w, b1.w);
    return (int)((sad + (unsigned)abs(dl)) >> 1);
}

// ---------------------------------------------------------------------------
// q-gram signature lower bound for edit distance.  A string's signature is a
// 256-bit set: bit bucket(g) for every q-gram g (q consecutive dense
// symbols); bucket = the exact index for q = 4 over an alphabet of <= 4
// symbols or q = 2 over <= 16, else a hash.  If bucket b is set for x and
// clear for y, every q-gram of x in b is absent from y, and each edit
// operation touches at most q q-gram windows of x, so
//     ed(x, y) >= ceil(popc(Sx & ~Sy) / q)        (and symmetrically).
// Collisions only weaken the bound.  Query symbols absent from the index
// alphabet hash like any other: their grams cannot occur in an object.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int qgram_q(int A) { return A <= 4 ? 4 : 2; }

__host__ __device__ __forceinline__ uint32_t qgram_bucket(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, int A)
{
    if (A <= 4) return (((c0 & 3u) * 4u + (c1 & 3u)) * 4u + (c2 & 3u)) * 4u + (c3 & 3u);
    if (A <= 16) return (c0 & 15u) * 16u + (c1 & 15u);
    return ((c0 * 29u) ^ (c1 * 113u) ^ (c1 >> 3)) & 255u;
}

// sym(i) -> dense symbol of position i, for i < n
template <class Sym>
__host__ __device__ __forceinline__ void qgram_sig(Sym sym, int n, int A, uint32_t (&w)[8])
{
    for (int k = 0; k < 8; k++) w[k] = 0u;
    const int Q = qgram_q(A);
    if (n < Q) return;
    uint32_t c0 = 0, c1 = sym(0), c2 = Q == 4 ? sym(1) : 0u, c3 = Q == 4 ? sym(2) : 0u;
    for (int i = Q - 1; i < n; i++) {
        uint32_t b;
        if (Q == 4) {
            c0 = c1; c1 = c2; c2 = c3; c3 = sym(i);
            b = qgram_bucket(c0, c1, c2, c3, A);
        } else {
            c0 = c1; c1 = sym(i);
            b = qgram_bucket(c0, c1, 0u, 0u, A);
        }
        w[b >> 5] |= 1u << (b & 31);
    }
}

__device__ __forceinline__ int qgram_lb(const uint4 &a0, const uint4 &a1, const uint4 &b0, const uint4 &b1, int Q)
{
    const int x = __popc(a0.x & ~b0.x) + __popc(a0.y & ~b0.y) + __popc(a0.z & ~b0.z) + __popc(a0.w & ~b0.w) +
                  __popc(a1.x & ~b1.x) + __popc(a1.y & ~b1.y) + __popc(a1.z & ~b1.z) + __popc(a1.w & ~b1.w);
    const int y = __popc(b0.x & ~a0.x) + __popc(b0.y & ~a0.y) + __popc(b0.z & ~a0.z) + __popc(b0.w & ~a0.w) +
                  __popc(b1.x & ~a1.x) + __popc(b1.y & ~a1.y) + __popc(b1.z & ~a1.z) + __popc(b1.w & ~a1.w);
    const int m = max(x, y);
    return Q == 4 ? (m + 3) >> 2 : (m + 1) >> 1;
}

struct HitBuf {
    int32_t *q;
    int32_t *e;
    double *d;
    unsigned long long cap;
    unsigned long long *counter;
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ bool is_alive(const uint32_t *alive, int e)
{
    return (__ldg(alive + (e >> 5)) >> (e & 31)) & 1u;
}

// ---------------------------------------------------------------------------
// edit distance: Myers/Hyyro block bit-vector recurrence, pattern = query
// (match masks Peq[A][W] precomputed per query), text = stored object
// (dense symbols, 4 per 32-bit word, 4-byte aligned).  The horizontal carry
// between 32-bit blocks travels as two bits (hp: +1, hm: -1); the score is
// read off the final column, D[m][n] = n + popc(Pv) - popc(Mv), so the loop
// carries no per-column score.  Same integer as the reference DP
// (metrics.py:54-84).
// ---------------------------------------------------------------------------
// The constant 2 from the constant bank: ptxas cannot fold a __constant__
// value, so x * kTwo + 1 (the +1-boundary shift) and sym * kTwo * kTwo + base
// (the mask address) stay IMADs on the fma pipe instead of LEA / SHF+LOP on
// the ALU pipe, which is the binding pipe of the DP (7 LOP3 per step).
__constant__ uint32_t kTwo = 2u;

__device__ __forceinline__ void myers_step1(uint32_t Eq, uint32_t &Pv, uint32_t &Mv)
{
    // single block, top boundary row +1 per column.  Hyyro's form: with
    // X = Eq | Mv, D0 = (((X & Pv) + Pv) ^ Pv) | X (Pv & Mv == 0 makes it
    // the textbook Xh | Mv), 10 integer ops per text symbol.
    const uint32_t X = Eq | Mv;
    const uint32_t D0 = (((X & Pv) + Pv) ^ Pv) | X;
    const uint32_t HN = Pv & D0;
    const uint32_t HP = Mv | ~(Pv | D0);
    const uint32_t Xs = HP * kTwo + 1u;
    Mv = Xs & D0;
    Pv = (HN * kTwo) | ~(Xs | D0);
}

// One 32-row block of the multi-block recurrence with the horizontal carry
// (hp: +1, hm: -1) in and out.  (Moving the shifts to IMAD / IMAD.HI on the
// fma pipe measured slower on DNA-108: 5.13 vs 4.86 s per step.)
__device__ __forceinline__ void myers_stepb(uint32_t Eq, uint32_t &Pv, uint32_t &Mv, uint32_t &hp, uint32_t &hm)
{
    const uint32_t Xv = Eq | Mv;
    Eq |= hm;
    const uint32_t Xh = (((Eq & Pv) + Pv) ^ Pv) | Eq;
    uint32_t Ph = Mv | ~(Xh | Pv);
    uint32_t Mh = Pv & Xh;
    const uint32_t op = Ph >> 31, om = Mh >> 31;
    Ph = (Ph << 1) | hp;
    Mh = (Mh << 1) | hm;
    Pv = Mh | ~(Xv | Ph);
    Mv = Ph & Xv;
    hp = op;
    hm = om;
}

template <int W>
__device__ __forceinline__ void myers_char(const uint32_t *peq, uint32_t c, uint32_t (&P)[W], uint32_t (&M)[W])
{
    if (W == 1) {
        myers_step1(*reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(peq) + c * (kTwo * kTwo)),
                    P[0], M[0]);
    } else {
        uint32_t hp = 1u, hm = 0u;
#pragma unroll
        for (int b = 0; b < W; b++) myers_stepb(peq[c * W + b], P[b], M[b], hp, hm);
    }
}

// peq: [A][W] masks of the query (shared or global); t4: text (storage is
// padded, so reading one word past the end is safe).  Four symbols per
// 32-bit word, unrolled; the next word is loaded while this one computes.
template <int W>
__device__ __forceinline__ void myers_word(const uint32_t *peq, uint32_t w, uint32_t (&P)[W], uint32_t (&M)[W])
{
    // one ALU op per symbol: LOP (byte 0), PRMT (bytes 1, 2), SHF (byte 3)
    myers_char<W>(peq, w & 0xffu, P, M);
    myers_char<W>(peq, __byte_perm(w, 0u, 0x4441), P, M);
    myers_char<W>(peq, __byte_perm(w, 0u, 0x4442), P, M);
    myers_char<W>(peq, w >> 24, P, M);
}

// text loads: global (read-only path) or shared (leaf staged by the block)
template <bool SMEM>
__device__ __forceinline__ uint32_t tload(const uint32_t *p)
{
    if (SMEM) return *p;
    return __ldg(p);
}

template <int W, bool SMEM = false>
__device__ __forceinline__ int myers_fixed(const uint32_t *peq, int m, const uint32_t *__restrict__ t4, int n)
{
    uint32_t P[W], M[W];
#pragma unroll
    for (int b = 0; b < W; b++) { P[b] = ~0u; M[b] = 0u; }
    const int nfull = n >> 2;
    uint32_t w = tload<SMEM>(t4);
    for (int jw = 0; jw < nfull; jw++) {
        const uint32_t nxt = tload<SMEM>(t4 + jw + 1);
        myers_word<W>(peq, w, P, M);
        w = nxt;
    }
    const int rem = n & 3;
    if (rem) {
        myers_char<W>(peq, w & 0xffu, P, M);
        if (rem > 1) myers_char<W>(peq, (w >> 8) & 0xffu, P, M);
        if (rem > 2) myers_char<W>(peq, (w >> 16) & 0xffu, P, M);
    }
    // blocks past the pattern's last word (a batch runs its widest lane's W)
    // only see rows below row m; they never feed back into rows <= m
    const int wl = (m + 31) >> 5;
    const uint32_t lastmask = (m & 31) ? ((1u << (m & 31)) - 1u) : ~0u;
    int score = n;
#pragma unroll
    for (int b = 0; b < W; b++) {
        const uint32_t mk = b < wl - 1 ? ~0u : (b == wl - 1 ? lastmask : 0u);
        score += __popc(P[b] & mk) - __popc(M[b] & mk);
    }
    return score;
}

// Text in shared memory, one symbol per byte load (LDS.U8 with immediate
// offsets): no ALU-pipe symbol extraction per step.  `two` is the runtime
// constant 2 (a kernel argument ptxas cannot fold), so the +1-boundary shift
// (HP * 2 + 1) and the mask address (peq + sym * 4 * W) are IMADs on the
// fma pipe and the ALU pipe carries only the 7 LOP3 of the recurrence.
// Blocks past the pattern's last word behave as in myers_fixed.
template <int W>
__device__ __forceinline__ void myers_char_s(const uint32_t *peq, uint32_t c, uint32_t two, int A, uint32_t (&P)[W],
                                             uint32_t (&M)[W])
{
    // masks block-major [W][A]: block b of symbol c at peq[b * A + c]
    const uint32_t *pe = reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(peq) + c * (two * two));
    if (W == 1) {
        const uint32_t X = pe[0] | M[0];
        const uint32_t D0 = (((X & P[0]) + P[0]) ^ P[0]) | X;
        const uint32_t HN = P[0] & D0;
        const uint32_t HP = M[0] | ~(P[0] | D0);
        const uint32_t Xs = HP * two + 1u;
        M[0] = Xs & D0;
        P[0] = HN * two | ~(Xs | D0);
    } else {
        uint32_t hp = 1u, hm = 0u;
#pragma unroll
        for (int b = 0; b < W; b++) myers_stepb(pe[b * A], P[b], M[b], hp, hm);
    }
}

template <int W>
__device__ __forceinline__ int myers_smem(const uint32_t *peq, int m, const uint8_t *t, int n, uint32_t two, int A)
{
    uint32_t P[W], M[W];
#pragma unroll
    for (int b = 0; b < W; b++) { P[b] = ~0u; M[b] = 0u; }
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        const uint32_t c0 = t[j], c1 = t[j + 1], c2 = t[j + 2], c3 = t[j + 3];
        myers_char_s<W>(peq, c0, two, A, P, M);
        myers_char_s<W>(peq, c1, two, A, P, M);
        myers_char_s<W>(peq, c2, two, A, P, M);
        myers_char_s<W>(peq, c3, two, A, P, M);
    }
    for (; j < n; j++) myers_char_s<W>(peq, t[j], two, A, P, M);
    const int wl = (m + 31) >> 5;
    const uint32_t lastmask = (m & 31) ? ((1u << (m & 31)) - 1u) : ~0u;
    int score = n;
#pragma unroll
    for (int b = 0; b < W; b++) {
        const uint32_t mk = b < wl - 1 ? ~0u : (b == wl - 1 ? lastmask : 0u);
        score += __popc(P[b] & mk) - __popc(M[b] & mk);
    }
    return score;
}

// Text in shared memory (one byte per symbol, LDS.U8), masks in the
// per-query [A][W] layout of the row-wise kernel (block b of symbol c at
// peq[c * W + b]); the address is an IMAD through kTwo.
template <int W>
__device__ __forceinline__ int myers_smem_aw(const uint32_t *peq, int m, const uint8_t *t, int n)
{
    uint32_t P[W], M[W];
#pragma unroll
    for (int b = 0; b < W; b++) { P[b] = ~0u; M[b] = 0u; }
    const uint32_t scale = kTwo * kTwo * W;
    auto step = [&](uint32_t c) {
        const uint32_t *pe = reinterpret_cast<const uint32_t *>(reinterpret_cast<const char *>(peq) + c * scale);
        if (W == 1) {
            myers_step1(pe[0], P[0], M[0]);
        } else {
            uint32_t hp = 1u, hm = 0u;
#pragma unroll
            for (int b = 0; b < W; b++) myers_stepb(pe[b], P[b], M[b], hp, hm);
        }
    };
    int j = 0;
    for (; j + 4 <= n; j += 4) {
        const uint32_t c0 = t[j], c1 = t[j + 1], c2 = t[j + 2], c3 = t[j + 3];
        step(c0);
        step(c1);
        step(c2);
        step(c3);
    }
    for (; j < n; j++) step(t[j]);
    const uint32_t lastmask = (m & 31) ? ((1u << (m & 31)) - 1u) : ~0u;
    int score = n;
#pragma unroll
    for (int b = 0; b < W; b++) {
        const uint32_t mk = (b == W - 1) ? lastmask : ~0u;
        score += __popc(P[b] & mk) - __popc(M[b] & mk);
    }
    return score;
}

// Patterns longer than 32 * kMaxWords symbols (texts of at most that many):
// the same recurrence in row-band order.  Band b (pattern rows 32b..32b+31)
// sweeps the whole text; the horizontal carry (hp: +1, hm: -1) of every text
// column passes from band b to band b+1 through two bit arrays of n bits
// (band 0 sees the top boundary row D[0][j] = j: hp = 1, hm = 0).  The score
// is n plus the vertical deltas of the last column, summed band by band.
__device__ __noinline__ int myers_banded(const uint32_t *peq, int W, int m, const uint32_t *__restrict__ t4, int n)
{
    uint32_t cp[kMaxWords], cm[kMaxWords];   // per text column: carry of the band above
    const int nw = (n + 31) >> 5;
    for (int k = 0; k < nw; k++) { cp[k] = ~0u; cm[k] = 0u; }
    const uint32_t lastmask = (m & 31) ? ((1u << (m & 31)) - 1u) : ~0u;
    int score = n;
    for (int b = 0; b < W; b++) {
        uint32_t P = ~0u, M = 0u;
        for (int k = 0; k < nw; k++) {
            uint32_t op = 0u, om = 0u;
            const int jn = min(32, n - 32 * k);
            for (int t = 0; t < jn; t++) {
                const int j = 32 * k + t;
                const uint32_t c = (__ldg(t4 + (j >> 2)) >> (8 * (j & 3))) & 0xffu;
                uint32_t hp = (cp[k] >> t) & 1u, hm = (cm[k] >> t) & 1u;
                myers_stepb(peq[c * W + b], P, M, hp, hm);
                op |= hp << t;
                om |= hm << t;
            }
            cp[k] = op;
            cm[k] = om;
        }
        const uint32_t mk = (b == W - 1) ? lastmask : ~0u;
        score += __popc(P & mk) - __popc(M & mk);
    }
    return score;
}

__device__ __noinline__ int myers_generic(const uint32_t *peq, int W, int m, const uint32_t *__restrict__ t4, int n)
{
    if (W > kMaxWords) return n <= 32 * kMaxWords ? myers_banded(peq, W, m, t4, n) : -1;
    uint32_t P[kMaxWords], M[kMaxWords];
    for (int b = 0; b < W; b++) { P[b] = ~0u; M[b] = 0u; }
    for (int j = 0; j < n; j++) {
        const uint32_t c = (__ldg(t4 + (j >> 2)) >> (8 * (j & 3))) & 0xffu;
        uint32_t hp = 1u, hm = 0u;
        for (int b = 0; b < W; b++) myers_stepb(peq[c * W + b], P[b], M[b], hp, hm);
    }
    const uint32_t lastmask = (m & 31) ? ((1u << (m & 31)) - 1u) : ~0u;
    int score = n;
    for (int b = 0; b < W; b++) {
        const uint32_t mk = (b == W - 1) ? lastmask : ~0u;
        score += __popc(P[b] & mk) - __popc(M[b] & mk);
    }
    return score;
}

// edit distance between pattern (m symbols, masks peq) and text (n symbols)
__device__ __forceinline__ int edit_peq(const uint32_t *peq, int m, const uint32_t *t4, int n)
{
    if (m == 0) return n;
    if (n == 0) return m;
    switch ((m + 31) >> 5) {
    case 1: return myers_fixed<1>(peq, m, t4, n);
    case 2: return myers_fixed<2>(peq, m, t4, n);
    case 3: return myers_fixed<3>(peq, m, t4, n);
    case 4: return myers_fixed<4>(peq, m, t4, n);
    default: return myers_generic(peq, (m + 31) >> 5, m, t4, n);
    }
}

__device__ __forceinline__ int qlen(const QueryView &qv, int q) { return (int)(qv.soff[q + 1] - qv.soff[q]); }

// ---------------------------------------------------------------------------
// vectors: fp32 screening distance (float4 loads) and the exact float64
// distance in numpy's pairwise row-sum order (bit-identical to the
// reference's l1/l2_one_to_many, metrics.py:127-133).
// ---------------------------------------------------------------------------
template <int MET>
__device__ __forceinline__ float vdist32(const float *__restrict__ a, const float *__restrict__ b, int Dp)
{
    float acc = 0.f;
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    for (int i = 0; i < (Dp >> 2); i++) {
        float4 x = __ldg(a4 + i), y = __ldg(b4 + i);
        float d0 = x.x - y.x, d1 = x.y - y.y, d2 = x.z - y.z, d3 = x.w - y.w;
        if (MET == kMetricL1) acc += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
        else acc += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
    return MET == kMetricL1 ? acc : sqrtf(acc);
}

template <int MET>
__device__ __forceinline__ double term64(double x, double y)
{
    if (MET == kMetricAngular) return __dmul_rn(x, y);   // dot-product terms
    if (MET == kMetricSq) return __dmul_rn(x, x);        // squared-norm terms
    double d = __dadd_rn(x, -y);
    return MET == kMetricL1 ? fabs(d) : __dmul_rn(d, d);
}

template <int MET>
__device__ double pw_sum64(const float *o32, const double *o64, const double *q, int s, int n)
{
#define GTS_X(i) (o64 ? o64[(i)] : (double)o32[(i)])
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; i++) r = __dadd_rn(r, term64<MET>(GTS_X(s + i), q[s + i]));
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = term64<MET>(GTS_X(s + j), q[s + j]);
        int i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], term64<MET>(GTS_X(s + i + j), q[s + i + j]));
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, term64<MET>(GTS_X(s + i), q[s + i]));
        return res;
    }
#undef GTS_X
    int n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sum64<MET>(o32, o64, q, s, n2), pw_sum64<MET>(o32, o64, q, s + n2, n - n2));
}

// angular_one_to_many (metrics.py:136-163) from the dot product and the two
// norms: zero vectors at pi from non-zero vectors and 0 from each other,
// arccos(clip(dot / (|o| |q|))), and identical vectors forced to 0.
__device__ __forceinline__ double angular_finish(double dot, double no, double nq, const float *o32,
                                                 const double *o64, const double *qv64, int D)
{
    if (nq == 0.0) return no == 0.0 ? 0.0 : 3.141592653589793;
    if (no == 0.0) return 3.141592653589793;
    double c = __ddiv_rn(dot, __dmul_rn(no, nq));
    c = fmin(1.0, fmax(-1.0, c));
    double r = acos(c);
    if (r < 1e-6) {
        bool eq = true;
        for (int i = 0; i < D && eq; i++) eq = (o64 ? o64[i] : (double)o32[i]) == qv64[i];
        if (eq) r = 0.0;
    }
    return r;
}

template <int MET>
__device__ __forceinline__ double vdist64(const IndexView &ix, const QueryView &qv, int q, int e)
{
    const float *o32 = ix.vec64 ? nullptr : ix.vec32 + (size_t)e * ix.Dp;
    const double *o64 = ix.vec64 ? ix.vec64 + (size_t)e * ix.D : nullptr;
    const double *q64 = qv.vec64 + (size_t)q * ix.D;
    double s = pw_sum64<MET>(o32, o64, q64, 0, ix.D);
    if (MET == kMetricAngular) return angular_finish(s, ix.vnorm64[e], qv.qnorm64[q], o32, o64, q64, ix.D);
    return MET == kMetricL1 ? s : __dsqrt_rn(s);
}

// |x| in numpy's order: sqrt of the pairwise sum of squares (data.py:81-84)
__device__ __forceinline__ double norm64(const double *x, int D)
{
    return __dsqrt_rn(pw_sum64<kMetricSq>(nullptr, x, x, 0, D));
}

// fp32 angular screen: arccos of the fp32 cosine (error bound: ix.abs_eps)
__device__ __forceinline__ float angular32(const float *__restrict__ a, const float *__restrict__ b, int Dp, float na,
                                           float nb)
{
    if (nb == 0.f) return na == 0.f ? 0.f : 3.14159265f;
    if (na == 0.f) return 3.14159265f;
    float acc = 0.f;
    const float4 *a4 = reinterpret_cast<const float4 *>(a);
    const float4 *b4 = reinterpret_cast<const float4 *>(b);
    for (int i = 0; i < (Dp >> 2); i++) {
        const float4 x = __ldg(a4 + i), y = __ldg(b4 + i);
        acc += (x.x * y.x + x.y * y.y) + (x.z * y.z + x.w * y.w);
    }
    return acosf(fminf(1.f, fmaxf(-1.f, acc / (na * nb))));
}

// screening distance query q -> table entry e (exact integer for edit)
template <int MET>
__device__ __forceinline__ float dist32(const IndexView &ix, const QueryView &qv, int q, int e)
{
    if (MET == kMetricEdit) {
        return (float)edit_peq(qv.peq + qv.peq_off[q], qlen(qv, q), ix.str + ix.sword[e], ix.slen[e]);
    } else if (MET == kMetricAngular) {
        return angular32(ix.vec32 + (size_t)e * ix.Dp, qv.vec32 + (size_t)q * ix.Dp, ix.Dp, ix.vnorm32[e], qv.qnorm32[q]);
    } else {
        return vdist32<MET>(ix.vec32 + (size_t)e * ix.Dp, qv.vec32 + (size_t)q * ix.Dp, ix.Dp);
    }
}

// fp32 error slack for comparisons involving magnitudes a, b (and c);
// exact metrics (rel == 0) never touch the magnitudes, so an infinite
// radius cannot turn the slack into NaN.
__device__ __forceinline__ float slack(const IndexView &ix, float a, float b, float c = 0.f)
{
    return ix.rel > 0.f ? ix.rel * (fabsf(a) + fabsf(b) + fabsf(c)) + ix.abs_eps : ix.abs_eps;
}

// Lemma-1 entry test for float metrics (search.py:523, 559) as a window on
// the entry's pivot distance: |dis - dqp| <= r + rel*(dis + dqp + r) + eps
// solved for dis (no divisions: 1/(1+rel) >= 1-rel, 1/(1-rel) <= 1+2rel),
//   lo = (dqp - r - s)(1 - rel)(1 - 2^-21)   (or -inf when that is <= 0),
//   hi = (dqp + r + s)(1 + 2 rel)(1 + 2^-21),   s = rel (dqp + r) + eps,
// a superset of the fp32-slack test, which is itself a superset of the
// reference's float64 test.  Two comparisons per entry; every float kernel
// counts the same "verified" entries.  NaN (tombstoned / padding) fails.
__device__ __forceinline__ float2 lemma1_range(const IndexView &ix, float dqp, float r)
{
    const float s = ix.rel * (dqp + r) + ix.abs_eps;
    const float num = dqp - r - s;
    const float lo = num > 0.f ? num * (1.f - ix.rel) * (1.f - 0x1p-21f) : -INFINITY;
    const float hi = (dqp + r + s) * (1.f + 2.f * ix.rel) * (1.f + 0x1p-21f);
    return make_float2(lo, hi);
}
__device__ __forceinline__ bool lemma1_in(float dis, float2 rg) { return dis >= rg.x && dis <= rg.y; }

}  // namespace gts
