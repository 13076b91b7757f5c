// engine.cu -- device index, batch range / kNN search driver and the C ABI.
//
// Pipeline per batch (reference BatchSearcher, search.py:273-296):
//   root table   k_root       d(q, root pivot)                (search.py:316-334)
//   per layer    k_expand     Eq.1 children, parent-range pre-screen,
//                             child pivot distance, own-range post-screen,
//                             block-aggregated compaction     (search.py:405-477)
//   leaves       k_verify     lemma-1 entry filter, exact distance, hits
//                                                              (search.py:507-538)
//   collect      3 stable CUB radix sorts -> (q, d, id) CSR   (search.py:298-314)
// The host driver walks layers depth-first in chunks of level_size_limit
// parent rows, so no child table exceeds memory_units rows
// (search.py:359-403, runtime.py:56-88).
// kNN = k_probe (radius estimate from the query's nearest sibling leaves)
// + the same range pipeline with that radius (tie-inclusive) + per-query
// truncation to the k smallest (distance, id) (oracle.py:30-36).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <thread>
#include <tuple>
#include <string>
#include <vector>

#include <cub/cub.cuh>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "../../include/gts.h"
#include "common.h"
#include "kernels.cuh"
#include "tcgen05.cuh"

namespace gts {

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local char g_err[2048] = "";

int set_error(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

struct Error {
    int code;
};

[[noreturn]] static void fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    throw Error{code};
}

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess)                                                                  \
            fail(e_ == cudaErrorMemoryAllocation ? GTS_EOOM : GTS_ECUDA, "%s: %s (%s:%d)", #x, \
                 cudaGetErrorString(e_), __FILE__, __LINE__);                                   \
    } while (0)

static std::atomic<int64_t> g_launches{0};
static std::atomic<double> g_hits_per_query[2] = {{0.0}, {0.0}};   // largest hits / query seen (range, kNN)

// Optional per-kernel timing (CUDA events on the launching stream) and
// algorithmic work counters, read by bench.py for the roofline figures.
static std::atomic<int> g_profile{0};
struct ProfRec {
    double ms = 0;
    int64_t count = 0;
};
static std::mutex g_prof_mu;
static std::vector<std::pair<std::string, ProfRec>> g_prof;
static unsigned long long g_work[4] = {0, 0, 0, 0};   // pairs, word-steps, entries, rows
static unsigned long long *g_phase_dev = nullptr;       // GTS_PHASES: per-phase clocks of k_leafgroup_mma
enum { kWorkPairs = 0, kWorkSteps = 1, kWorkEntries = 2, kWorkRows = 3 };
static double g_expand[4] = {0, 0, 0, 0};   // traversal: algorithmic bytes, parent rows in, child rows out, distances

static void prof_add(const char *name, double ms)
{
    std::lock_guard<std::mutex> g(g_prof_mu);
    for (auto &kv : g_prof)
        if (kv.first == name) { kv.second.ms += ms; kv.second.count++; return; }
    g_prof.push_back({name, ProfRec{ms, 1}});
}

#define LAUNCH_CHECK() \
    do {               \
        g_launches++;  \
        CK(cudaGetLastError()); \
    } while (0)

// stream-ordered device buffer
template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    cudaStream_t s = 0;
    DBuf() = default;
    DBuf(size_t cnt, cudaStream_t st) { alloc(cnt, st); }
    DBuf(const DBuf &) = delete;
    DBuf &operator=(const DBuf &) = delete;
    DBuf(DBuf &&o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DBuf &operator=(DBuf &&o) noexcept
    {
        if (this != &o) { release(); p = o.p; n = o.n; s = o.s; o.p = nullptr; o.n = 0; }
        return *this;
    }
    void alloc(size_t cnt, cudaStream_t st)
    {
        release();
        s = st;
        static const bool trace = std::getenv("GTS_TRACE_ALLOC") != nullptr;
        const auto t0 = trace ? std::chrono::steady_clock::now() : std::chrono::steady_clock::time_point{};
        if (cnt) CK(cudaMallocAsync((void **)&p, cnt * sizeof(T), st));
        if (trace) {
            const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
            if (ms > 0.5) fprintf(stderr, "[gts] slow cudaMallocAsync: %.2f ms for %zu bytes\n", ms, cnt * sizeof(T));
        }
        n = cnt;
    }
    void release()
    {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { release(); }
};

template <class T>
static void h2d(T *dst, const T *src, size_t cnt, cudaStream_t s)
{
    if (cnt) CK(cudaMemcpyAsync(dst, src, cnt * sizeof(T), cudaMemcpyHostToDevice, s));
}

static inline unsigned grid_for(int64_t threads, int block, unsigned cap = 1u << 30)
{
    int64_t g = (threads + block - 1) / block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

// Dynamic shared-memory opt-in.  cudaFuncSetAttribute applies per device
// context, so the granted size is recorded per (device, kernel); a mutex
// makes it safe for the per-shard host threads of a multi-device index.
static void smem_optin(const void *fn, size_t bytes)
{
    static std::mutex mu;
    static std::vector<std::tuple<int, const void *, size_t>> granted;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    for (auto &t : granted)
        if (std::get<0>(t) == dev && std::get<1>(t) == fn) {
            if (std::get<2>(t) >= bytes) return;
            CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
            std::get<2>(t) = bytes;
            return;
        }
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    granted.emplace_back(dev, fn, bytes);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

// Root table: d(q, root pivot) for every query (search.py:316-334).
template <int MET>
__global__ void k_root(IndexView ix, QueryView qv, int nq, Row *out)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const int piv = ix.node[1].piv;
    out[q] = Row{q, 1, dist32<MET>(ix, qv, q, piv), 0};
}

// Block-aggregated compaction: returns this thread's output slot (or -1).
__device__ __forceinline__ long long block_append(bool keep, unsigned long long *counter, int *sh_warp,
                                                  unsigned long long *sh_base)
{
    const int lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned b = __ballot_sync(kFull, keep);
    if (lane == 0) sh_warp[warp] = __popc(b);
    __syncthreads();
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < nwarps; w++) { int c = sh_warp[w]; sh_warp[w] = tot; tot += c; }
        *sh_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    long long slot = -1;
    if (keep) slot = (long long)(*sh_base) + sh_warp[warp] + __popc(b & ((1u << lane) - 1u));
    __syncthreads();
    return slot;
}

// Warp-aggregated per-query counter add (all 32 lanes call; val 0 = no-op).
__device__ __forceinline__ void warp_add_q(unsigned long long *arr, int q, unsigned val)
{
    unsigned peers = __match_any_sync(kFull, q);
    unsigned s = __reduce_add_sync(peers, val);
    if (s && lane_id() == __ffs(peers) - 1) atomicAdd(arr + q, (unsigned long long)s);
}

// One level of the descent (search.py:405-477).  Thread per (row, child).
template <int MET>
__global__ void __launch_bounds__(256) k_expand(IndexView ix, QueryView qv, const Row *__restrict__ in,
                                                int64_t m, int own, int pruning, const float *__restrict__ r32,
                                                Row *out, unsigned long long *counter,
                                                unsigned long long *pruned_stat)
{
    __shared__ int sh_warp[32];
    __shared__ unsigned long long sh_base;
    const int nc = ix.nc;
    const int64_t total = m * nc;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < total; base += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = base + threadIdx.x;
        bool valid = i < total;
        bool keep = false, nonempty = false;
        int q = -1, child = 0;
        float cd = 0.f;
        if (valid) {
            const int64_t row = i / nc;
            const int j = (int)(i - row * nc);
            const Row pr = in[row];
            q = pr.q;
            child = (pr.node - 1) * nc + 2 + j;
            const NodeRec c = ix.node[child];
            nonempty = c.size > 0;
            keep = nonempty;
            const float r = r32[q];
            if (keep && !own && pruning) {
                // internal children carry ranges to the parent pivot:
                // keep iff dq + r >= min and dq - r <= max (search.py:425-433)
                const float e = slack(ix, pr.dqp, r);
                keep = (pr.dqp + r + e >= c.mn) && (pr.dqp - r - e <= c.mx);
            }
            if (keep) {
                cd = dist32<MET>(ix, qv, q, c.piv);
                if (own && pruning) {
                    // leaves carry ranges to their own pivot (search.py:467-471)
                    const float e = slack(ix, cd, r);
                    keep = (cd + r + e >= c.mn) && (cd - r - e <= c.mx);
                }
            }
        }
        warp_add_q(pruned_stat, valid ? q : -1, (valid && nonempty && !keep) ? 1u : 0u);
        long long slot = block_append(keep, counter, sh_warp, &sh_base);
        if (keep) out[slot] = Row{q, child, cd, 0};
    }
}

// Leaf verification (search.py:507-538), one warp per leaf row; emits
// (query, entry, exact float64 distance) for every live entry with d <= r.
template <int MET>
__global__ void __launch_bounds__(256) k_verify(IndexView ix, QueryView qv, const Row *__restrict__ rows,
                                                int64_t m, int pruning, const float *__restrict__ r32,
                                                const double *__restrict__ r64, HitBuf out,
                                                unsigned long long *verified_stat, int stats_on,
                                                unsigned long long *work)
{
    const int lane = lane_id();
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < m; w += warps) {
        const Row lr = rows[w];
        const int q = lr.q;
        const NodeRec leaf = ix.node[lr.node];
        const int pos = ix.npos[lr.node];
        const float r = r32[q];
        const double rr = r64[q];
        unsigned ver = 0;
        unsigned long long steps = 0;
        for (int b = 0; b < leaf.size; b += kWarp) {
            const int k = b + lane;
            bool pass = false;
            int e = pos + k;
            if (k < leaf.size && is_alive(ix.alive, e)) {
                if (!pruning) pass = true;
                else {
                    const float de = __ldg(ix.dis + e);
                    pass = lemma1_in(de, lemma1_range(ix, lr.dqp, r));
                }
            }
            ver += __popc(__ballot_sync(kFull, pass));
            bool hit = false;
            double d64 = 0.0;
            if (pass) {
                const float d = dist32<MET>(ix, qv, q, e);
                if (MET == kMetricEdit) {
                    hit = d <= r;
                    d64 = (double)d;
                } else if (d - slack(ix, d, 0.f) <= r) {
                    d64 = vdist64<MET>(ix, qv, q, e);
                    hit = d64 <= rr;
                }
            }
            unsigned hb = __ballot_sync(kFull, hit);
            if (hb) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(out.counter, (unsigned long long)__popc(hb));
                base = __shfl_sync(kFull, base, 0);
                if (hit) {
                    unsigned long long slot = base + __popc(hb & ((1u << lane) - 1u));
                    if (slot < out.cap) { out.q[slot] = q; out.e[slot] = e; out.d[slot] = d64; }
                }
            }
        }
        if (stats_on && lane == 0 && ver) atomicAdd(verified_stat + q, (unsigned long long)ver);
        if (work) {
            for (int o = 16; o > 0; o >>= 1) steps += __shfl_down_sync(kFull, steps, o);
            if (lane == 0) {
                atomicAdd(work + kWorkPairs, (unsigned long long)ver);
                atomicAdd(work + kWorkSteps, steps);
                atomicAdd(work + kWorkEntries, (unsigned long long)leaf.size);
                atomicAdd(work + kWorkRows, 1ull);
            }
        }
    }
}

constexpr int kLeafWarps = 8;          // warps per block of k_leaf_edit
constexpr int kRowChunk = 16;          // rows a warp claims per cursor bump

// match masks too large to stage (A*W > kWarpPeqWords): read from global
__device__ __noinline__ int edit_peq_global(const uint32_t *peq, int m, const uint32_t *t4, int n)
{
    return edit_peq(peq, m, t4, n);
}
constexpr int kWarpPeqWords = 1024;     // per-warp staged match masks (A*W <= 1024)

// Fused leaf scan + verification for edit distance (search.py:507-570).
// Each warp owns a contiguous run of leaf rows.  Per row, live entries
// passing the lemma-1 pivot test count as "verified" (the reference's
// counter) and those whose length also fits the radius (|len q - len o|
// lower-bounds the edit distance) are pushed onto a warp-private queue in
// shared memory; every 32 queued entries run as one batch of bit-parallel
// DPs (one per lane) against the row query's match masks staged in shared
// memory.  Leaves are length-sorted, so a batch has similar DP lengths.
constexpr int kHistBins = 256;   // kNN shrinking-bound histogram: exact distances 0..255

// SIG: q-gram signatures; PRUNE: lemma-1 test (pruning on); EHIST: symbol
// histograms (compile-time, so the entry loop carries no runtime flags)
template <bool SIG, bool PRUNE, bool EHIST>
__global__ void __launch_bounds__(256, 4) k_leaf_edit(IndexView ix, QueryView qv, const Row *__restrict__ rows,
                                                      int64_t m, int pruning, float *r32,
                                                      HitBuf out, unsigned long long *verified_stat, int stats_on,
                                                      unsigned long long *work, unsigned long long *cursor,
                                                      unsigned *hist, const int32_t *__restrict__ ks, int claim,
                                                      int tstride)
{
    extern __shared__ uint32_t le_text[];   // [kLeafWarps][32][tstride] when tstride > 0
    __shared__ uint32_t peq_s[kLeafWarps][kWarpPeqWords];
    __shared__ int32_t queue[kLeafWarps][3][64];   // entry, first text word, length
    __shared__ uint4 qsig_s[kLeafWarps][2];        // the current query's q-gram signature
    const int lane = lane_id(), wib = threadIdx.x >> 5;
    uint32_t *peq_w = peq_s[wib];
    int32_t *qu = queue[wib][0];
    int32_t *qw = queue[wib][1];
    int32_t *ql = queue[wib][2];
    int cur_q = -1, mq = 0, qn = 0;
    int qsig_reach = 0;   // ceil(distinct query q-gram buckets / q)
    unsigned long long nrows = 0;
    uint4 qh0 = make_uint4(0u, 0u, 0u, 0u), qh1 = qh0;
    float r = 0.f;
    bool staged = false;
    const uint32_t *peq_g = nullptr;
    unsigned long long steps = 0, pairs = 0, entries = 0;

    // kNN shrinking bound (hist != null): count every emitted candidate's
    // exact distance per query; the k-th smallest found so far is an upper
    // bound on the query's k-th distance, so the radius only ever shrinks
    // to values that still admit every true answer (and its ties).
    auto shrink = [&](bool ha, int dA, bool hb2, int dB) {
        const unsigned any = __ballot_sync(kFull, ha || hb2);
        if (!hist || !any) return;
        unsigned *hq_ = hist + (size_t)cur_q * kHistBins;
        if (ha && dA < kHistBins) atomicAdd(hq_ + dA, 1u);
        if (hb2 && dB < kHistBins) atomicAdd(hq_ + dB, 1u);
        // the k-th bound can only drop below r through a hit strictly below r
        // (hits at d == r, the common case once r has converged, leave it)
        if (!__any_sync(kFull, (ha && (float)dA < r) || (hb2 && (float)dB < r))) return;
        __syncwarp();
        __threadfence_block();
        // warp prefix over the 256 bins (8 per lane) -> smallest t with count(d <= t) >= k
        const int kq = ks[cur_q];
        unsigned c[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) { c[i] = __ldcg(hq_ + lane * 8 + i); tot += c[i]; }
        unsigned inc = tot;
        for (int o = 1; o < 32; o <<= 1) {
            unsigned v = __shfl_up_sync(kFull, inc, o);
            if (lane >= o) inc += v;
        }
        const unsigned before = inc - tot;
        int t = kHistBins;
        if (before < (unsigned)kq && inc >= (unsigned)kq) {
            unsigned run = before;
#pragma unroll
            for (int i = 0; i < 8; i++) {
                run += c[i];
                if (run >= (unsigned)kq) { t = lane * 8 + i; break; }
            }
        }
        for (int o = 16; o > 0; o >>= 1) t = min(t, __shfl_xor_sync(kFull, t, o));
        if (t < kHistBins && (float)t < r) {
            r = (float)t;
            if (lane == 0) atomicMin(reinterpret_cast<int *>(r32 + cur_q), __float_as_int((float)t));
        }
    };
    // emit one hit per lane (warp-aggregated slot claim)
    auto emit = [&](bool hit, int e, int d) {
        const unsigned hb = __ballot_sync(kFull, hit);
        if (hb) {
            unsigned long long hbase = 0;
            if (lane == 0) hbase = atomicAdd(out.counter, (unsigned long long)__popc(hb));
            hbase = __shfl_sync(kFull, hbase, 0);
            if (hit) {
                const unsigned long long sl = hbase + __popc(hb & ((1u << lane) - 1u));
                if (sl < out.cap) { out.q[sl] = cur_q; out.e[sl] = e; out.d[sl] = (double)d; }
            }
        }
    };
    // run DPs for queue slots [0, cnt) (cnt <= 32), one per lane
    auto run_batch = [&](int cnt) {
        const bool va = lane < cnt;
        int ea = -1, da = 0;
        const int wq = (mq + 31) >> 5;
        if (tstride && staged && wq <= 2 && mq > 0) {
            // stage each lane's text in shared memory (odd word stride: the
            // per-symbol byte loads of 32 lanes hit distinct banks), then run
            // the DP with LDS.U8 symbols -- no ALU-pipe symbol extraction
            uint32_t *tx = le_text + (size_t)wib * kWarp * tstride + (size_t)lane * tstride;
            int na = 0;
            if (va) {
                ea = qu[lane];
                na = ql[lane];
                const uint32_t *tA = ix.str + (uint32_t)qw[lane];
                for (int w = 0; w < ((na + 3) >> 2); w++) tx[w] = __ldg(tA + w);
            }
            __syncwarp();
            if (va) {
                const uint8_t *t1 = reinterpret_cast<const uint8_t *>(tx);
                da = na == 0 ? mq : (wq == 1 ? myers_smem_aw<1>(peq_w, mq, t1, na) : myers_smem_aw<2>(peq_w, mq, t1, na));
                steps += (unsigned long long)wq * (unsigned long long)na;
            }
        } else if (va) {
            ea = qu[lane];
            const int na = ql[lane];
            const uint32_t *tA = ix.str + (uint32_t)qw[lane];
            da = staged ? edit_peq(peq_w, mq, tA, na) : edit_peq_global(peq_g, mq, tA, na);
            steps += (unsigned long long)wq * (unsigned long long)na;
        }
        const bool ha = va && (float)da <= r;
        emit(ha, ea, da);
        shrink(ha, da, false, 0);
        __syncwarp();
    };

    // a warp claims `claim` consecutive rows (rows are in query order): with
    // a large claim one warp walks most of a query's leaves in sequence, so
    // the kNN radius shrunk by its own early hits filters the later leaves
    for (;;) {
        unsigned long long cstart = 0;
        if (lane == 0) cstart = atomicAdd(cursor, (unsigned long long)claim);
        cstart = __shfl_sync(kFull, cstart, 0);
        if ((int64_t)cstart >= m) break;
        const int64_t cstop = min(m, (int64_t)cstart + claim);
    for (int64_t start = (int64_t)cstart; start < cstop; start += kRowChunk) {
        const int64_t stop = min(cstop, start + kRowChunk);
        nrows += (unsigned long long)(stop - (int64_t)start);
        // lanes fetch the chunk's row and leaf records in one parallel batch
        Row pr{0, 0, 0.f, 0};
        NodeRec pn{0.f, 0.f, 0, 0};
        int ppos = 0;
        if ((int64_t)start + lane < stop) {
            pr = rows[start + lane];
            pn = ix.node[pr.node];
            ppos = ix.npos[pr.node];
        }
    for (int64_t w = (int64_t)start; w < stop; w++) {
        const int src = (int)(w - (int64_t)start);
        Row lr;
        lr.q = __shfl_sync(kFull, pr.q, src);
        lr.node = __shfl_sync(kFull, pr.node, src);
        lr.dqp = __shfl_sync(kFull, pr.dqp, src);
        if (lr.q != cur_q) {
            if (qn) { run_batch(qn); qn = 0; }
            cur_q = lr.q;
            mq = qlen(qv, cur_q);
            r = __ldcg(r32 + cur_q);
            if (EHIST) { qh0 = qv.qhist[2 * cur_q]; qh1 = qv.qhist[2 * cur_q + 1]; }
            if (SIG) {
                uint4 sg = make_uint4(0u, 0u, 0u, 0u);
                if (lane < 2) qsig_s[wib][lane] = sg = qv.qsig[2 * cur_q + lane];
                // the query's distinct q-gram buckets bound how far the
                // signature bound can reach from its side: ceil(popc / q)
                int pc = lane < 2 ? __popc(sg.x) + __popc(sg.y) + __popc(sg.z) + __popc(sg.w) : 0;
                pc += __shfl_xor_sync(kFull, pc, 1);
                pc = __shfl_sync(kFull, pc, 0);
                qsig_reach = (pc + ix.sig_q - 1) / max(ix.sig_q, 1);
            }
            peq_g = qv.peq + qv.peq_off[cur_q];
            const int words = qv.A * ((mq + 31) >> 5);
            staged = words <= kWarpPeqWords;
            if (staged) {
                for (int t = lane; t < words; t += kWarp) peq_w[t] = __ldg(peq_g + t);
            }
            __syncwarp();
        }
        if (hist) r = fminf(r, __ldcg(r32 + cur_q));   // another warp may have shrunk it
        NodeRec leaf;
        leaf.size = __shfl_sync(kFull, pn.size, src);
        const int pos = __shfl_sync(kFull, ppos, src);
        unsigned ver = 0;
        // the chunk's records are loaded one chunk ahead.  erec = {dis (NaN
        // when tombstoned, k_erec_alive), len, first text word, float(len)}:
        // the tombstone, lemma-1 and length tests are FP compares (fma pipe),
        // leaving the ALU pipe to the DP
        uint4 nrec = make_uint4(0u, 0u, 0u, 0u);
        if (lane < leaf.size) nrec = __ldg(ix.erec + pos + lane);
        const float mqf = (float)mq;
        const int ri = r < 1e9f ? (int)r : (1 << 30);   // edit distances are integers
        for (int b = 0; b < leaf.size; b += kWarp) {
            const int k = b + lane;
            const int e = pos + k;
            const uint4 rec = nrec;
            if (b + kWarp + lane < leaf.size) nrec = __ldg(ix.erec + e + kWarp);
            const float dis = __uint_as_float(rec.x), lenf = __uint_as_float(rec.w);
            bool pass = false;
            if (k < leaf.size) pass = PRUNE ? fabsf(dis - lr.dqp) <= r : dis == dis;
            ver += __popc(__ballot_sync(kFull, pass));
            bool cand = pass && fabsf(mqf - lenf) <= r;
            // the histogram bound never exceeds max(|q|, |o|): skip it when that
            // fits.  (Issuing these loads before the lemma-1 work, for every
            // length-passing entry, measured slower: 86.8 vs 84 ms on words.)
            if (EHIST && cand && fmaxf(mqf, lenf) > r) {
                const uint4 h0 = __ldg(ix.ehist + 2 * e), h1 = __ldg(ix.ehist + 2 * e + 1);
                cand = hist_lb(qh0, qh1, h0, h1, mq - (int)rec.y) <= ri;
            }
            // q-gram signature bound (qgram_lb), for the candidates still left,
            // when the query's side of it can exceed the radius (words kNN:
            // never, ~20% slower if tested anyway; DNA range r = 8: prunes
            // nearly every pair, 1.9x faster)
            if (SIG && cand && qsig_reach > ri) {
                const uint4 s0 = __ldg(ix.esig + 2 * e), s1 = __ldg(ix.esig + 2 * e + 1);
                cand = qgram_lb(qsig_s[wib][0], qsig_s[wib][1], s0, s1, ix.sig_q) <= ri;
            }
            const unsigned cb = __ballot_sync(kFull, cand);
            if (cand) {
                const int slot = qn + __popc(cb & ((1u << lane) - 1u));
                qu[slot] = e;
                qw[slot] = (int32_t)rec.z;
                ql[slot] = (int)rec.y;
            }
            qn += __popc(cb);
            __syncwarp();
            if (qn >= kWarp) {
                run_batch(kWarp);
                qn -= kWarp;
                if (lane < qn) { qu[lane] = qu[kWarp + lane]; qw[lane] = qw[kWarp + lane]; ql[lane] = ql[kWarp + lane]; }
                __syncwarp();
            }
        }
        if (lane == 0 && stats_on && ver) atomicAdd(verified_stat + lr.q, (unsigned long long)ver);
        pairs += ver;
        entries += leaf.size;
    }
    }
    }
    if (qn) run_batch(qn);
    if (work) {
        for (int o = 16; o > 0; o >>= 1) steps += __shfl_down_sync(kFull, steps, o);
        if (lane == 0) {
            atomicAdd(work + kWorkSteps, steps);
            atomicAdd(work + kWorkPairs, pairs);
            atomicAdd(work + kWorkEntries, entries);
            atomicAdd(work + kWorkRows, nrows);
        }
    }
}

// kNN: drop the hits already outside their query's (shrunk) radius.  The
// radius only shrinks to values that keep k objects (and their ties) at or
// below it, so such a hit can never be among the final k.  Output order is
// free (collect sorts).
__global__ void k_compact_hits(const int32_t *__restrict__ q, const int32_t *__restrict__ e,
                               const double *__restrict__ d, int64_t n, const float *__restrict__ r32,
                               const double *__restrict__ r64, int32_t *oq, int32_t *oe, double *od,
                               unsigned long long *cnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool keep = false;
    int32_t qi = 0;
    if (i < n) {
        qi = q[i];
        keep = d[i] <= (r64 ? __ldcg(r64 + qi) : (double)__ldcg(r32 + qi));
    }
    const unsigned b = __ballot_sync(kFull, keep);
    if (!b) return;
    unsigned long long base = 0;
    const int lane = lane_id();
    if (lane == __ffs(b) - 1) base = atomicAdd(cnt, (unsigned long long)__popc(b));
    base = __shfl_sync(kFull, base, __ffs(b) - 1);
    if (keep) {
        const unsigned long long o = base + __popc(b & ((1u << lane) - 1u));
        oq[o] = qi;
        oe[o] = e[i];
        od[o] = d[i];
    }
}

// erec.x = dis of live entries, NaN of tombstoned ones (every test fails)
__global__ void k_erec_alive(uint4 *erec, const float *dis, const uint32_t *alive, int64_t n)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const bool al = (alive[e >> 5] >> (e & 31)) & 1u;
    erec[e].x = al ? __float_as_uint(dis[e]) : 0x7fc00000u;
}

// Packed sort key for exact small-integer distances: query | distance |
// dataset row (row order == id order, data.py:149-153).
__global__ void k_pack_keys(const int32_t *hq, const int32_t *he, const double *hd, const int32_t *row, int64_t n,
                            int dshift, int qshift, unsigned long long *key, int32_t *perm)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = ((unsigned long long)hq[i] << qshift) | ((unsigned long long)hd[i] << dshift) |
             (unsigned long long)row[he[i]];
    perm[i] = (int32_t)i;
}

// counts[q] from sorted packed keys (two binary searches per query)
__global__ void k_seg_counts(const unsigned long long *key, int64_t n, int qshift, int nq, long long *counts)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    auto lb = [&](unsigned long long v) {
        int64_t lo = 0, hi = n;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (key[mid] < v) lo = mid + 1; else hi = mid;
        }
        return lo;
    };
    counts[q] = lb((unsigned long long)(q + 1) << qshift) - lb((unsigned long long)q << qshift);
}

// ---------------------------------------------------------------------------
// Leaf-grouped verification for vectors.  The chunk's leaf rows are counting-
// sorted by leaf; a work item is (leaf, up to kItemQueries queries).  A block
// stages the leaf's vectors in shared memory once and every query visiting
// the leaf reads them from there: one HBM/L2 read of a leaf per item instead
// of one per (query, entry) pair.  Same filter / screen / float64 recheck as
// k_verify (search.py:507-570).
// ---------------------------------------------------------------------------
struct Item {                      // 32 B: a leaf (node) and a run of its grouped rows
    int32_t leaf, start, count, size;   // size / pos: the node's, for kernels that stage it
    int32_t pos, pad0, pad1, pad2;
};
constexpr int kItemQueries = 128;

// Counting sort of frontier rows by node.  Warp-aggregated: lanes holding the
// same node elect one atomic (upper layers have only 1-20 distinct nodes, so
// per-row atomics would serialise on a handful of counters).
__global__ void k_leaf_hist(const Row *rows, int64_t m, int leaf_first, int *cnt)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int key = i < m ? rows[i].node - leaf_first : -1;
    const unsigned peers = __match_any_sync(kFull, key);
    if (key >= 0 && lane_id() == __ffs(peers) - 1) atomicAdd(cnt + key, __popc(peers));
}

__global__ void k_leaf_scatter(const Row *rows, int64_t m, int leaf_first, int *cursor, Row *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    Row r{0, 0, 0.f, 0};
    int key = -1;
    if (i < m) {
        r = rows[i];
        key = r.node - leaf_first;
    }
    const unsigned peers = __match_any_sync(kFull, key);
    const int leader = __ffs(peers) - 1, lane = lane_id();
    int base = 0;
    if (key >= 0 && lane == leader) base = atomicAdd(cursor + key, __popc(peers));
    base = __shfl_sync(kFull, base, leader);
    if (key >= 0) out[base + __popc(peers & ((1u << lane) - 1u))] = r;
}

// The same counting sort with block-private shared-memory counters (indexes
// of <= kPrivLeaves leaves): a block counts a contiguous slice of rows with
// shared atomics, then claims its per-leaf bases with one global atomic per
// non-empty leaf (bbase[block][leaf]); the scatter re-walks the same slice
// and places rows through shared cursors.  Two global atomics per (block,
// leaf) instead of one per row on a few thousand hot counters.
constexpr int kPrivLeaves = 40 * 1024;   // 160 KB of counters
constexpr int kPrivThreads = 1024;

__global__ void __launch_bounds__(kPrivThreads) k_leaf_hist_priv(const Row *__restrict__ rows, int64_t m,
                                                                 int leaf_first, int nleaf, int *cnt, int *bbase)
{
    extern __shared__ int hcount[];
    for (int l = threadIdx.x; l < nleaf; l += blockDim.x) hcount[l] = 0;
    __syncthreads();
    const int64_t per = (m + gridDim.x - 1) / gridDim.x;
    const int64_t a = (int64_t)blockIdx.x * per, b = min(m, a + per);
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        const int key = rows[i].node - leaf_first;
        if ((unsigned)key < (unsigned)nleaf) atomicAdd(&hcount[key], 1);
    }
    __syncthreads();
    int *bb = bbase + (size_t)blockIdx.x * nleaf;
    for (int l = threadIdx.x; l < nleaf; l += blockDim.x) {
        const int c = hcount[l];
        bb[l] = c ? atomicAdd(cnt + l, c) : 0;
    }
}

__global__ void __launch_bounds__(kPrivThreads) k_leaf_scatter_priv(const Row *__restrict__ rows, int64_t m,
                                                                    int leaf_first, int nleaf,
                                                                    const int *__restrict__ off,
                                                                    const int *__restrict__ bbase, Row *out)
{
    extern __shared__ int hcur[];
    const int *bb = bbase + (size_t)blockIdx.x * nleaf;
    for (int l = threadIdx.x; l < nleaf; l += blockDim.x) hcur[l] = off[l] + bb[l];
    __syncthreads();
    const int64_t per = (m + gridDim.x - 1) / gridDim.x;
    const int64_t a = (int64_t)blockIdx.x * per, b = min(m, a + per);
    for (int64_t i = a + threadIdx.x; i < b; i += blockDim.x) {
        const Row r = rows[i];
        const int key = r.node - leaf_first;
        if ((unsigned)key < (unsigned)nleaf) out[atomicAdd(&hcur[key], 1)] = r;
    }
}

__global__ void k_item_counts(const int *cnt, int nleaf, int per, int *nitem)
{
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l < nleaf) nitem[l] = (cnt[l] + per - 1) / per;
}

// one thread per item: its leaf is the last l with item_off[l] <= item
// (leaves without rows have item_off[l] == item_off[l + 1])
__global__ void k_make_items(const int *cnt, const int *off, const int *item_off, int nleaf, int nitems,
                             int leaf_first, int per, const NodeRec *node, const int32_t *npos, Item *items,
                             const int32_t *vt_off, const int32_t *vt_rows)
{
    const int it = blockIdx.x * blockDim.x + threadIdx.x;
    if (it >= nitems) return;
    int lo = 0, hi = nleaf;   // upper_bound(it) over item_off[0..nleaf) - 1
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (item_off[mid] <= it) lo = mid + 1; else hi = mid;
    }
    const int l = lo - 1;
    const int c = cnt[l], nd = leaf_first + l;
    const int s = (it - item_off[l]) * per;
    // pad0: the leaf's image in vtile, (offset / 2 KB) << 8 | rows / 16
    const int tr = vt_off ? (int)(((uint32_t)(vt_off[l] >> 4) << 8) | (uint32_t)(vt_rows[l] >> 4)) : 0;
    items[it] = Item{nd, off[l] + s, min(per, c - s), node[nd].size, npos[nd], tr, 0, 0};
}

// ---------------------------------------------------------------------------
// Leaf-grouped edit verification (the words / DNA hot kernel).  Rows are
// grouped by leaf into items of <= kItemQueries rows (k_leaf_hist /
// k_leaf_scatter above).  A block stages one leaf -- pivot distances,
// lengths, alive bits, symbol histograms and the packed text -- in shared
// memory ONCE, and every query row of the item scans it from there: a leaf
// costs one L2 read per item instead of one per (query, entry) pair (kNN
// over 1M words visits ~all 8,000 leaves from every query).  Each warp takes
// kLgSlots rows at a time, stages their match masks, and feeds the
// candidates of all of them into one warp queue, so 32-lane DP batches stay
// full even when a row has only a few candidates.  Filters and counters are
// those of k_leaf_edit (search.py:507-570): the lemma-1 pivot test is the
// reference's "verified", then the |len q - len o| and symbol-histogram
// lower bounds, then the exact bit-parallel DP with the text read from
// shared memory.
// ---------------------------------------------------------------------------
constexpr int kLgSlots = 4;        // rows (queries) a warp has in flight
constexpr int kLgWarps = 8;
constexpr int kLgItemRows = 512;   // rows per item: leaf staging amortised over 512 rows

struct LgEditLayout {              // shared-memory carve-up in bytes (host-computed)
    int cap_e, cap_w;              // staged entries / text words per leaf
    int tstride;                   // text words per staged entry (odd; fits the longest stored string)
    int wmax, slot_words;          // pattern words (<= 4); words per staged slot (wmax * A, padded)
    int use_hist;
    int off_meta, off_h0, off_h1, off_text, off_peq, off_queue, off_slot, total;
    uint32_t two;                  // the constant 2, opaque to ptxas (see myers_smem)
};

// Shared-memory layouts are chosen for conflict-free LDS:
//   text    entry k at word k * tstride (tstride odd), so the byte loads of
//           32 lanes on 32 different entries spread over the banks;
//   hist    two uint4 arrays (16-byte stride) instead of one 32-byte record;
//   masks   per slot block-major [W][A], slots padded to an odd multiple
//           of 8 words apart.
__global__ void __launch_bounds__(32 * kLgWarps, 4)
k_leafgroup_edit(IndexView ix, QueryView qv, const Row *__restrict__ srows, const Item *__restrict__ items, int nitems,
                 unsigned long long *item_cursor, LgEditLayout L, int pruning, float *r32, HitBuf out,
                 unsigned long long *verified_stat, int stats_on, unsigned long long *work, unsigned *hist,
                 const int32_t *__restrict__ ks)
{
    extern __shared__ uint4 lg_smem4[];
    char *sm = reinterpret_cast<char *>(lg_smem4);
    float *dis_s = reinterpret_cast<float *>(sm);
    uint32_t *meta_s = reinterpret_cast<uint32_t *>(sm + L.off_meta);   // len | alive << 31
    uint4 *h0_s = reinterpret_cast<uint4 *>(sm + L.off_h0);
    uint4 *h1_s = reinterpret_cast<uint4 *>(sm + L.off_h1);
    uint32_t *text_s = reinterpret_cast<uint32_t *>(sm + L.off_text);
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t *peq_w = reinterpret_cast<uint32_t *>(sm + L.off_peq) + (size_t)warp * kLgSlots * L.slot_words;
    int32_t *qk = reinterpret_cast<int32_t *>(sm + L.off_queue) + warp * 64;        // slot << 16 | entry
    int32_t *slot_q = reinterpret_cast<int32_t *>(sm + L.off_slot) + warp * 4 * kLgSlots;
    int32_t *slot_m = slot_q + kLgSlots;
    int32_t *slot_w = slot_m + kLgSlots;
    float *slot_r = reinterpret_cast<float *>(slot_w + kLgSlots);
    __shared__ int item_s, group_s, tstride_s;
    const int A = qv.A;
    unsigned long long steps = 0, pairs = 0, entries = 0, nrows = 0;

    for (;;) {
        __syncthreads();   // the previous leaf is no longer read
        if (threadIdx.x == 0) {
            item_s = (int)atomicAdd(item_cursor, 1ull);
            group_s = kLgWarps;
        }
        __syncthreads();
        const int it = item_s;
        if (it >= nitems) break;
        const Item item = items[it];
        const int size = ix.node[item.leaf].size;
        const int pos = ix.npos[item.leaf];
        if (size == 0) continue;
        // one stride for every leaf: entries inserted in place (leaf slack)
        // break the in-leaf length order, so the last entry need not be the longest
        const int tstride = L.tstride;
        for (int k = threadIdx.x; k < size; k += blockDim.x) {
            const int e = pos + k;
            const uint4 rec = __ldg(ix.erec + e);
            const uint32_t al = (__ldg(ix.alive + (e >> 5)) >> (e & 31)) & 1u;
            dis_s[k] = __uint_as_float(rec.x);
            meta_s[k] = rec.y | (al << 31);
            if (L.use_hist) {
                h0_s[k] = __ldg(ix.ehist + 2 * e);
                h1_s[k] = __ldg(ix.ehist + 2 * e + 1);
            }
        }
        for (int t = threadIdx.x; t < size * tstride; t += blockDim.x) {
            const int k = t / tstride, w = t - k * tstride;
            const int e = pos + k;
            if (w < ((__ldg(ix.slen + e) + 3) >> 2)) text_s[t] = __ldg(ix.str + __ldg(ix.sword + e) + w);
        }
        __syncthreads();

        const int ngroups = (item.count + kLgSlots - 1) / kLgSlots;
        // row groups: warp w starts with group w, then claims the next free one
        for (int g = warp; g < ngroups;) {
            const int rbase = item.start + g * kLgSlots;
            const int ns = min(kLgSlots, item.count - g * kLgSlots);
            float dqp_l = 0.f;
            if (lane < ns) {
                const Row rw = srows[rbase + lane];
                const int m = qlen(qv, rw.q);
                dqp_l = rw.dqp;
                slot_q[lane] = rw.q;
                slot_m[lane] = m;
                slot_w[lane] = max(1, (m + 31) >> 5);
                slot_r[lane] = __ldcg(r32 + rw.q);
            }
            __syncwarp();
            // stage masks: slot s block-major [W][A] (blocks past its own W zeroed)
            for (int s = 0; s < ns; s++) {
                const int qs = slot_q[s], ws = (slot_m[s] + 31) >> 5;
                const uint32_t *src = qv.peq + qv.peq_off[qs];
                uint32_t *dst = peq_w + s * L.slot_words;
                for (int t = lane; t < L.wmax * A; t += kWarp) {
                    const int b = t / A, c = t - b * A;
                    dst[t] = b < ws ? __ldg(src + c * ws + b) : 0u;
                }
            }
            __syncwarp();
            nrows += (unsigned long long)ns;

            // run queued DPs [0, cnt), one per lane; emit hits; shrink kNN radii
            auto run_batch = [&](int cnt) {
                const bool va = lane < cnt;
                int d = 0, k = 0, sl = 0, wl = 1;
                if (va) {
                    const int v = qk[lane];
                    sl = v >> 16;
                    k = v & 0xffff;
                    wl = slot_w[sl];
                }
                const int Wb = (int)__reduce_max_sync(kFull, (unsigned)wl);   // widest pattern in the batch
                if (va) {
                    const int n = (int)(meta_s[k] & 0xffffu);
                    const uint8_t *t1 = reinterpret_cast<const uint8_t *>(text_s + k * tstride);
                    const uint32_t *pq = peq_w + sl * L.slot_words;
                    const int ms = slot_m[sl];
                    switch (Wb) {
                    case 1: d = myers_smem<1>(pq, ms, t1, n, L.two, A); break;
                    case 2: d = myers_smem<2>(pq, ms, t1, n, L.two, A); break;
                    case 3: d = myers_smem<3>(pq, ms, t1, n, L.two, A); break;
                    default: d = myers_smem<4>(pq, ms, t1, n, L.two, A); break;
                    }
                    steps += (unsigned long long)wl * (unsigned long long)n;
                }
                const bool hit = va && (float)d <= slot_r[sl];
                const unsigned hb = __ballot_sync(kFull, hit);
                if (hb) {
                    unsigned long long hbase = 0;
                    if (lane == 0) hbase = atomicAdd(out.counter, (unsigned long long)__popc(hb));
                    hbase = __shfl_sync(kFull, hbase, 0);
                    if (hit) {
                        const unsigned long long o = hbase + __popc(hb & ((1u << lane) - 1u));
                        if (o < out.cap) { out.q[o] = slot_q[sl]; out.e[o] = pos + k; out.d[o] = (double)d; }
                        if (hist && d < kHistBins) atomicAdd(hist + (size_t)slot_q[sl] * kHistBins + d, 1u);
                    }
                    if (hist) {
                        __syncwarp();
                        __threadfence_block();
                        for (int s = 0; s < ns; s++) {
                            if (!__any_sync(kFull, hit && sl == s)) continue;
                            const int qs = slot_q[s];
                            const unsigned *hq_ = hist + (size_t)qs * kHistBins;
                            const unsigned kq = (unsigned)ks[qs];
                            unsigned c[8], tot = 0;
#pragma unroll
                            for (int i = 0; i < 8; i++) { c[i] = __ldcg(hq_ + lane * 8 + i); tot += c[i]; }
                            unsigned inc = tot;
                            for (int o = 1; o < 32; o <<= 1) {
                                const unsigned v = __shfl_up_sync(kFull, inc, o);
                                if (lane >= o) inc += v;
                            }
                            const unsigned before = inc - tot;
                            int t = kHistBins;
                            if (before < kq && inc >= kq) {
                                unsigned run = before;
#pragma unroll
                                for (int i = 0; i < 8; i++) {
                                    run += c[i];
                                    if (run >= kq) { t = lane * 8 + i; break; }
                                }
                            }
                            t = (int)__reduce_min_sync(kFull, (unsigned)t);
                            __syncwarp();
                            if (t < kHistBins && (float)t < slot_r[s] && lane == 0) {
                                slot_r[s] = (float)t;
                                atomicMin(reinterpret_cast<int *>(r32 + qs), __float_as_int((float)t));
                            }
                            __syncwarp();
                        }
                    }
                }
                __syncwarp();
            };

            int qn = 0;
            for (int s = 0; s < ns; s++) {
                const int qs = slot_q[s];
                const int ms = slot_m[s];
                const float dq = __shfl_sync(kFull, dqp_l, s);
                if (hist && lane == 0) slot_r[s] = fminf(slot_r[s], __ldcg(r32 + qs));   // other blocks shrink it
                __syncwarp();
                uint4 qh0 = make_uint4(0u, 0u, 0u, 0u), qh1 = qh0;
                if (L.use_hist) { qh0 = qv.qhist[2 * qs]; qh1 = qv.qhist[2 * qs + 1]; }
                unsigned ver = 0;
                for (int b = 0; b < size; b += kWarp) {
                    const float rs = slot_r[s];
                    const int k = b + lane;
                    bool pass = false;
                    uint32_t mt = 0;
                    if (k < size) {
                        mt = meta_s[k];
                        if (mt >> 31) pass = !pruning || fabsf(dis_s[k] - dq) <= rs;
                    }
                    ver += __popc(__ballot_sync(kFull, pass));
                    const int len = (int)(mt & 0xffffu);
                    bool cand = pass && (float)abs(ms - len) <= rs;
                    if (cand && L.use_hist) cand = (float)hist_lb(qh0, qh1, h0_s[k], h1_s[k], ms - len) <= rs;
                    const unsigned cb = __ballot_sync(kFull, cand);
                    if (cand) qk[qn + __popc(cb & ((1u << lane) - 1u))] = (s << 16) | k;
                    qn += __popc(cb);
                    __syncwarp();
                    if (qn >= kWarp) {
                        run_batch(kWarp);
                        qn -= kWarp;
                        if (lane < qn) qk[lane] = qk[kWarp + lane];
                        __syncwarp();
                    }
                }
                if (lane == 0 && stats_on && ver) atomicAdd(verified_stat + qs, (unsigned long long)ver);
                pairs += ver;
                entries += (unsigned long long)size;
            }
            if (qn) run_batch(qn);
            __syncwarp();
            int nx = 0;
            if (lane == 0) nx = atomicAdd(&group_s, 1);
            g = __shfl_sync(kFull, nx, 0);
        }
    }
    if (work) {
        for (int o = 16; o > 0; o >>= 1) steps += __shfl_down_sync(kFull, steps, o);
        if (lane == 0) {
            atomicAdd(work + kWorkSteps, steps);
            atomicAdd(work + kWorkPairs, pairs);
            atomicAdd(work + kWorkEntries, entries);
            atomicAdd(work + kWorkRows, nrows);
        }
    }
}

template <int MET>
__device__ __forceinline__ float vdist32_smem(const float *a, const float *b, int Dp)
{
    float acc = 0.f;
    for (int i = 0; i < Dp; i += 4) {
        const float4 x = *reinterpret_cast<const float4 *>(a + i);
        const float4 y = *reinterpret_cast<const float4 *>(b + i);
        const float d0 = x.x - y.x, d1 = x.y - y.y, d2 = x.z - y.z, d3 = x.w - y.w;
        if (MET == kMetricL1) acc += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
        else acc += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
    }
    return MET == kMetricL1 ? acc : sqrtf(acc);
}

// One level of the descent for vectors, rows grouped by parent node
// (same predicates and outputs as k_expand).  A block stages the node's
// child records and child pivot vectors in shared memory once per item of
// <= kItemQueries rows; thread per (row, child) then reads only its query
// (broadcast across the row's nc consecutive lanes) from global memory.
template <int MET>
__global__ void __launch_bounds__(256) k_expand_grouped(IndexView ix, QueryView qv, const Row *__restrict__ srows,
                                                        const Item *__restrict__ items, int nitems, int own,
                                                        int pruning, const float *__restrict__ r32, Row *out,
                                                        unsigned long long *counter, unsigned long long *pruned_stat)
{
    extern __shared__ float4 ex_smem4[];
    // [nc][Dp + 4]: the 16-byte row skew puts the nc children of one row on
    // different banks (a 512-byte stride would make them a 20-way conflict)
    const int ps = ix.Dp + 4;
    float *piv_s = reinterpret_cast<float *>(ex_smem4);
    NodeRec *rec_s = reinterpret_cast<NodeRec *>(piv_s + (size_t)ix.nc * ps);
    __shared__ int sh_warp[32];
    __shared__ unsigned long long sh_base;
    const int nc = ix.nc, d4 = ix.Dp >> 2;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item item = items[it];
        const int child0 = (item.leaf - 1) * nc + 2;   // Eq. 1: children of node p are (p-1)*nc+2 ...
        __syncthreads();
        for (int t = threadIdx.x; t < nc; t += blockDim.x) rec_s[t] = ix.node[child0 + t];
        __syncthreads();
        for (int t = threadIdx.x; t < nc * d4; t += blockDim.x) {
            const int j = t / d4, c = t - j * d4;
            reinterpret_cast<float4 *>(piv_s + (size_t)j * ps)[c] =
                __ldg(reinterpret_cast<const float4 *>(ix.vec32 + (size_t)rec_s[j].piv * ix.Dp) + c);
        }
        __syncthreads();
        const int total = item.count * nc;
        for (int base = 0; base < total; base += blockDim.x) {
            const int i = base + threadIdx.x;
            const bool valid = i < total;
            bool keep = false, nonempty = false;
            int q = -1, child = 0;
            float cd = 0.f;
            if (valid) {
                const int row = i / nc, j = i - row * nc;
                const Row pr = srows[item.start + row];
                q = pr.q;
                child = child0 + j;
                const NodeRec c = rec_s[j];
                nonempty = c.size > 0;
                keep = nonempty;
                const float r = r32[q];
                if (keep && !own && pruning) {
                    const float e = slack(ix, pr.dqp, r);
                    keep = (pr.dqp + r + e >= c.mn) && (pr.dqp - r - e <= c.mx);
                }
                if (keep) {
                    float acc = 0.f;
                    const float4 *qp = reinterpret_cast<const float4 *>(qv.vec32 + (size_t)q * ix.Dp);
                    const float4 *pp = reinterpret_cast<const float4 *>(piv_s + (size_t)j * ps);
                    for (int k = 0; k < d4; k++) {
                        const float4 x = pp[k], y = __ldg(qp + k);
                        const float d0 = x.x - y.x, d1 = x.y - y.y, d2 = x.z - y.z, d3 = x.w - y.w;
                        if (MET == kMetricL1) acc += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
                        else acc += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
                    }
                    cd = MET == kMetricL1 ? acc : sqrtf(acc);
                    if (own && pruning) {
                        const float e = slack(ix, cd, r);
                        keep = (cd + r + e >= c.mn) && (cd - r - e <= c.mx);
                    }
                }
            }
            warp_add_q(pruned_stat, valid ? q : -1, (valid && nonempty && !keep) ? 1u : 0u);
            long long slot = block_append(keep, counter, sh_warp, &sh_base);
            if (keep) out[slot] = Row{q, child, cd, 0};
        }
    }
}

// Register-tiled variant of k_expand_grouped (vectors, the default for
// D >= 16): the item's <= 128 query vectors are staged in shared memory next
// to the node's child pivots, and a thread computes a 2-row x CPG-child tile
// (rows a and a + 64, children CPG g .. CPG g + CPG - 1 for child group
// g = threadIdx / 64), so one float4 step issues 2 + CPG shared loads for
// 2 CPG distances instead of 2 loads per distance.  Same per-float4
// accumulation order as k_expand_grouped (identical child distances), same
// keep tests (search.py:425-433, 467-471), pruned counts summed per row in
// shared memory, one block-wide compaction per item.
constexpr int kXtRows = 128;
template <int MET, int CPG>
__global__ void __launch_bounds__(256, 2) k_expand_tile(IndexView ix, QueryView qv, const Row *__restrict__ srows,
                                                        const Item *__restrict__ items, int nitems, int own,
                                                        int pruning, const float *__restrict__ r32, Row *out,
                                                        unsigned long long *counter, unsigned long long *pruned_stat)
{
    extern __shared__ float4 xt_smem4[];
    const int ps = ix.Dp + 4;   // 16-byte skew: consecutive rows on different banks
    float *piv_s = reinterpret_cast<float *>(xt_smem4);
    float *qs_s = piv_s + (size_t)4 * CPG * ps;
    NodeRec *rec_s = reinterpret_cast<NodeRec *>(qs_s + (size_t)kXtRows * ps);
    __shared__ int s_q[kXtRows];
    __shared__ float s_dqp[kXtRows], s_r[kXtRows];
    __shared__ unsigned s_pruned[kXtRows];
    __shared__ int sh_warp[8];
    __shared__ unsigned long long sh_base;
    const int nc = ix.nc, d4 = ix.Dp >> 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int ra = tid & 63, g = tid >> 6;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item item = items[it];
        const int child0 = (item.leaf - 1) * nc + 2;   // Eq. 1
        __syncthreads();   // the previous item's smem is no longer read
        if (tid < 4 * CPG) {
            NodeRec c{0.f, 0.f, 0, 0};
            if (tid < nc) c = ix.node[child0 + tid];
            rec_s[tid] = c;
        }
        if (tid < kXtRows) {
            int q = -1;
            float dqp = 0.f, r = 0.f;
            if (tid < item.count) {
                const Row pr = srows[item.start + tid];
                q = pr.q;
                dqp = pr.dqp;
                r = r32[q];
            }
            s_q[tid] = q;
            s_dqp[tid] = dqp;
            s_r[tid] = r;
            s_pruned[tid] = 0u;
        }
        __syncthreads();
        // staging by cp.async (many 16-byte copies in flight per thread;
        // absent rows / children zero-filled)
        for (int t = tid; t < 4 * CPG * d4; t += blockDim.x) {
            const int j = t / d4, c = t - j * d4;
            const float *src = ix.vec32 + (size_t)(j < nc ? rec_s[j].piv : 0) * ix.Dp + 4 * c;
            tc::cp_async16(tc::smem_u32(piv_s + (size_t)j * ps + 4 * c), src, j < nc ? 16u : 0u);
        }
        for (int t = tid; t < kXtRows * d4; t += blockDim.x) {
            const int a = t / d4, c = t - a * d4;
            const int q = s_q[a];
            const float *src = qv.vec32 + (size_t)max(q, 0) * ix.Dp + 4 * c;
            tc::cp_async16(tc::smem_u32(qs_s + (size_t)a * ps + 4 * c), src, q >= 0 ? 16u : 0u);
        }
        tc::cp_async_commit();
        tc::cp_async_wait_all();
        __syncthreads();
        float acc[2][CPG];
#pragma unroll
        for (int u = 0; u < 2; u++)
#pragma unroll
            for (int k = 0; k < CPG; k++) acc[u][k] = 0.f;
        const float4 *xa = reinterpret_cast<const float4 *>(qs_s + (size_t)ra * ps);
        const float4 *xb = reinterpret_cast<const float4 *>(qs_s + (size_t)(ra + 64) * ps);
        const float4 *py = reinterpret_cast<const float4 *>(piv_s + (size_t)g * CPG * ps);
        for (int c = 0; c < d4; c++) {
            const float4 x0 = xa[c], x1 = xb[c];
#pragma unroll
            for (int k = 0; k < CPG; k++) {
                const float4 y = py[(size_t)k * (ps >> 2) + c];   // warp-uniform: broadcast
                {
                    const float d0 = y.x - x0.x, d1 = y.y - x0.y, d2 = y.z - x0.z, d3 = y.w - x0.w;
                    if (MET == kMetricL1) acc[0][k] += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
                    else acc[0][k] += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
                }
                {
                    const float d0 = y.x - x1.x, d1 = y.y - x1.y, d2 = y.z - x1.z, d3 = y.w - x1.w;
                    if (MET == kMetricL1) acc[1][k] += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
                    else acc[1][k] += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
                }
            }
        }
        // keep tests, pruned counts, this thread's kept rows
        uint32_t keepm = 0;   // bit u * CPG + k
#pragma unroll
        for (int u = 0; u < 2; u++) {
            const int a = ra + 64 * u;
            const int q = s_q[a];
            if (q < 0) continue;
            const float dqp = s_dqp[a], r = s_r[a];
            unsigned pr = 0;
#pragma unroll
            for (int k = 0; k < CPG; k++) {
                const int j = g * CPG + k;
                if (j >= nc) continue;
                const NodeRec c = rec_s[j];
                if (c.size <= 0) continue;
                bool keep = true;
                if (!own && pruning) {
                    const float e = slack(ix, dqp, r);
                    keep = (dqp + r + e >= c.mn) && (dqp - r - e <= c.mx);
                }
                const float cd = MET == kMetricL1 ? acc[u][k] : sqrtf(acc[u][k]);
                acc[u][k] = cd;
                if (keep && own && pruning) {
                    const float e = slack(ix, cd, r);
                    keep = (cd + r + e >= c.mn) && (cd - r - e <= c.mx);
                }
                if (keep) keepm |= 1u << (u * CPG + k);
                else pr++;
            }
            if (pr) atomicAdd(&s_pruned[a], pr);
        }
        // block-wide compaction: warp scan of the per-thread counts
        const unsigned nk = __popc(keepm);
        unsigned incl = nk;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(kFull, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) sh_warp[warp] = (int)incl;
        __syncthreads();
        if (tid == 0) {
            int tot = 0;
            for (int w = 0; w < 8; w++) { const int c = sh_warp[w]; sh_warp[w] = tot; tot += c; }
            sh_base = tot ? atomicAdd(counter, (unsigned long long)tot) : 0ull;
        }
        __syncthreads();
        unsigned long long slot = sh_base + (unsigned long long)sh_warp[warp] + (incl - nk);
#pragma unroll
        for (int u = 0; u < 2; u++)
#pragma unroll
            for (int k = 0; k < CPG; k++)
                if ((keepm >> (u * CPG + k)) & 1u) {
                    const int a = ra + 64 * u;
                    out[slot++] = Row{s_q[a], child0 + g * CPG + k, acc[u][k], 0};
                }
        if (tid < kXtRows && s_pruned[tid] && s_q[tid] >= 0)
            atomicAdd(pruned_stat + s_q[tid], (unsigned long long)s_pruned[tid]);
    }
}

__device__ __forceinline__ void fhist_add(unsigned *hist, const float *r0, int q, double d);
__device__ __forceinline__ void fhist_shrink(unsigned *hist, const float *r0, const int32_t *ks, float *r32,
                                             double *r64, int q);

template <int MET>
__global__ void __launch_bounds__(256) k_leafgroup_vec(IndexView ix, QueryView qv, const Row *__restrict__ srows,
                                                       const Item *__restrict__ items, int nitems, int pruning,
                                                       float *r32, double *r64,
                                                       HitBuf out, unsigned long long *verified_stat, int stats_on,
                                                       unsigned long long *work, unsigned *fhist, const float *r0,
                                                       const int32_t *ks)
{
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    const int lane = lane_id(), warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int stride = ix.Dp + 4;                      // padded: conflict-free LDS.128 per quarter warp
    float *ent = smem;
    float *qslot = smem + (size_t)ix.max_leaf * stride + (size_t)warp * ix.Dp;
    const int d4 = ix.Dp >> 2;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item item = items[it];
        const NodeRec leaf = ix.node[item.leaf];
        const int pos = ix.npos[item.leaf];
        for (int t = threadIdx.x; t < leaf.size * d4; t += blockDim.x) {
            const int e = t / d4, c = t - e * d4;
            *reinterpret_cast<float4 *>(ent + e * stride + 4 * c) =
                __ldg(reinterpret_cast<const float4 *>(ix.vec32 + (size_t)(pos + e) * ix.Dp) + c);
        }
        __syncthreads();
        unsigned long long pairs = 0;
        for (int qi = warp; qi < item.count; qi += nwarps) {
            const Row lr = srows[item.start + qi];
            const int q = lr.q;
            const float r = __ldcg(r32 + q);
            const double rr = __ldcg(r64 + q);
            unsigned nh = 0;
            for (int c = lane; c < d4; c += kWarp)
                *reinterpret_cast<float4 *>(qslot + 4 * c) =
                    __ldg(reinterpret_cast<const float4 *>(qv.vec32 + (size_t)q * ix.Dp) + c);
            __syncwarp();
            unsigned ver = 0;
            for (int b = 0; b < leaf.size; b += kWarp) {
                const int k = b + lane;
                const int e = pos + k;
                bool pass = false;
                if (k < leaf.size && is_alive(ix.alive, e)) {
                    if (!pruning) pass = true;
                    else {
                        const float de = __ldg(ix.dis + e);
                        pass = lemma1_in(de, lemma1_range(ix, lr.dqp, r));
                    }
                }
                ver += __popc(__ballot_sync(kFull, pass));
                bool hit = false;
                double d64 = 0.0;
                if (pass) {
                    const float d = vdist32_smem<MET>(ent + k * stride, qslot, ix.Dp);
                    if (d - slack(ix, d, 0.f) <= r) {
                        d64 = vdist64<MET>(ix, qv, q, e);
                        hit = d64 <= rr;
                    }
                }
                const unsigned hb = __ballot_sync(kFull, hit);
                if (hb) {
                    unsigned long long base = 0;
                    if (lane == 0) base = atomicAdd(out.counter, (unsigned long long)__popc(hb));
                    base = __shfl_sync(kFull, base, 0);
                    if (hit) {
                        const unsigned long long slot = base + __popc(hb & ((1u << lane) - 1u));
                        if (slot < out.cap) { out.q[slot] = q; out.e[slot] = e; out.d[slot] = d64; }
                        if (fhist) fhist_add(fhist, r0, q, d64);
                    }
                    nh += __popc(hb);
                }
            }
            if (fhist && nh) {
                __threadfence();
                if (lane == 0) fhist_shrink(fhist, r0, ks, r32, r64, q);
            }
            if (lane == 0 && stats_on && ver) atomicAdd(verified_stat + q, (unsigned long long)ver);
            pairs += ver;
            __syncwarp();
        }
        if (work && lane == 0) {
            atomicAdd(work + kWorkPairs, pairs);
            atomicAdd(work + kWorkRows, 0ull);
        }
        if (work && threadIdx.x == 0) {
            atomicAdd(work + kWorkEntries, (unsigned long long)leaf.size * item.count);
            atomicAdd(work + kWorkRows, (unsigned long long)item.count);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Register-tiled CUDA-core verification (L1, and L2 off the tensor-core
// path).  Item = (leaf, <= 128 query rows); the block stages the leaf's
// entries AND the item's query vectors in shared memory (rows padded by 16
// bytes: conflict-free LDS.128), then every thread computes a 4 x 4 tile of
// (query, entry) fp32 distances: lane -> query rows lane + 32a, warp -> entry
// chunks of 4.  Per 4 dimensions that is 8 LDS.128 (4 per-lane query rows, 4
// broadcast entry rows) for 64 pair-dimensions, so the FP32 pipes, not
// shared memory, bound it.  Filters and outputs are those of
// k_leafgroup_vec: lemma 1 (the verified count), fp32 screen with slack,
// exact float64 recheck in numpy order, kNN histogram shrink.
// ---------------------------------------------------------------------------
// screened (query, entry) candidates awaiting the exact float64 recheck
struct CandBuf {
    int32_t *q, *e;
    float *lb;                 // lower bound of the compared quantity (d^2 for L2, d for L1)
    unsigned long long cap;
    unsigned long long *counter;
};

template <int MET>
__global__ void __launch_bounds__(256, 4) k_leafgroup_tile(IndexView ix, QueryView qv, const Row *__restrict__ srows,
                                                        const Item *__restrict__ items, int nitems, int pruning,
                                                        float *r32, double *r64, CandBuf cb,
                                                        unsigned long long *verified_stat, int stats_on,
                                                        unsigned long long *work, unsigned *fhist, const float *r0,
                                                        const int32_t *ks)
{
    extern __shared__ float4 tile_smem4[];
    const int stride = ix.Dp + 4;
    float *ent = reinterpret_cast<float *>(tile_smem4);                 // [max_leaf][stride]
    float *qs = ent + (size_t)ix.max_leaf * stride;                       // [128][stride]
    float *s_dis = qs + (size_t)128 * stride;                             // [max_leaf] (NaN: tombstoned)
    float *s_lo = s_dis + ix.max_leaf;                                    // [128] lemma-1 window, per row
    float *s_r = s_lo + 128;                                              // [128]
    int *s_q = reinterpret_cast<int *>(s_r + 128);                        // [128]
    unsigned *s_ver = reinterpret_cast<unsigned *>(s_q + 128);            // [128]
    float *s_hi = reinterpret_cast<float *>(s_ver + 128);                 // [128]
    const int lane = lane_id(), warp = threadIdx.x >> 5;
    const int d4 = ix.Dp >> 2;
    unsigned long long w_entries = 0, w_rows = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item item = items[it];
        const int size = ix.node[item.leaf].size;
        const int pos = ix.npos[item.leaf];
        __syncthreads();
        if (threadIdx.x < 128) {
            const int a = threadIdx.x;
            int q = -1;
            float dqp = 0.f, r = -1.f;
            if (a < item.count) {
                const Row lr = srows[item.start + a];
                q = lr.q;
                dqp = lr.dqp;
                r = __ldcg(r32 + q);
            }
            // the window is fixed for the item (a kNN shrink narrows only the
            // screen; the wider window is conservative)
            const float2 rg = lemma1_range(ix, dqp, r);
            s_q[a] = q;
            s_lo[a] = rg.x;
            s_hi[a] = rg.y;
            s_r[a] = r;
            s_ver[a] = 0;
        }
        for (int j = threadIdx.x; j < size; j += blockDim.x) {
            const bool al = is_alive(ix.alive, pos + j);
            s_dis[j] = al ? __ldg(ix.dis + pos + j) : __int_as_float(0x7fc00000);
        }
        for (int t = threadIdx.x; t < size * d4; t += blockDim.x) {
            const int e = t / d4, c = t - e * d4;
            *reinterpret_cast<float4 *>(ent + e * stride + 4 * c) =
                __ldg(reinterpret_cast<const float4 *>(ix.vec32 + (size_t)(pos + e) * ix.Dp) + c);
        }
        __syncthreads();
        for (int t = threadIdx.x; t < 128 * d4; t += blockDim.x) {
            const int a = t / d4, c = t - a * d4;
            const int q = s_q[a];
            *reinterpret_cast<float4 *>(qs + a * stride + 4 * c) =
                q >= 0 ? __ldg(reinterpret_cast<const float4 *>(qv.vec32 + (size_t)q * ix.Dp) + c)
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        __syncthreads();
        // tasks = (4-entry chunk, half of the 128 rows): a lane computes a
        // 2-row x 4-entry tile.  Small leaves (the 12.5M shard's ~78 entries:
        // 20 chunks) then split evenly over the 8 warps (40 tasks) instead of
        // 3 / 2 chunks per warp waiting at the item barrier.
        const int nchunks = (size + 3) >> 2;
        for (int task = warp; task < 2 * nchunks; task += 8) {
            const int ch = task >> 1, half = task & 1;
            const int e0 = ch * 4;
            const int rbase = lane + 64 * half;   // rows rbase, rbase + 32
            float acc[2][4];
#pragma unroll
            for (int a = 0; a < 2; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = 0.f;
            const float *qrow = qs + rbase * stride;
            const float *erow = ent + e0 * stride;
            for (int c = 0; c < d4; c++) {
                float4 x[2], y[4];
#pragma unroll
                for (int a = 0; a < 2; a++) x[a] = *reinterpret_cast<const float4 *>(qrow + a * 32 * stride + 4 * c);
#pragma unroll
                for (int b = 0; b < 4; b++) y[b] = *reinterpret_cast<const float4 *>(erow + b * stride + 4 * c);
#pragma unroll
                for (int a = 0; a < 2; a++)
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        const float d0 = x[a].x - y[b].x, d1 = x[a].y - y[b].y;
                        const float d2 = x[a].z - y[b].z, d3 = x[a].w - y[b].w;
                        if (MET == kMetricL1)
                            acc[a][b] += (fabsf(d0) + fabsf(d1)) + (fabsf(d2) + fabsf(d3));
                        else
                            acc[a][b] += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
                    }
            }
#pragma unroll
            for (int a = 0; a < 2; a++) {
                const int row = rbase + 32 * a;
                const int q = s_q[row];
                const float r = s_r[row];
                const float2 rg = make_float2(s_lo[row], s_hi[row]);
                bool any_ub = false;
                unsigned ver = 0;
                uint32_t cmask = 0;   // candidates of this row among the 4 entries
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int j = e0 + b;
                    if (q < 0 || j >= size) continue;
                    const float dis = s_dis[j];
                    if (!(dis == dis)) continue;   // tombstoned
                    if (pruning && !lemma1_in(dis, rg)) continue;
                    ver++;
                    const float d = MET == kMetricL1 ? acc[a][b] : sqrtf(acc[a][b]);
                    const float sl = slack(ix, d, 0.f);
                    if (!(d - sl <= r)) continue;
                    // candidate: exact float64 check later (k_recheck) against the final radius
                    cmask |= 1u << b;
                    if (fhist && d + sl <= r) {
                        // the true distance is <= d + slack: a valid upper bound for the shrink
                        fhist_add(fhist, r0, q, (double)(d + sl) * (1.0 + 1e-6));
                        any_ub = true;
                    }
                }
                if (ver) atomicAdd(s_ver + row, ver);
                // warp-aggregated append (one atomic per warp instead of per candidate)
                if (__any_sync(kFull, cmask)) {
                    const unsigned nc = __popc(cmask);
                    unsigned incl = nc;
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned v = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const unsigned wtot = __shfl_sync(kFull, incl, 31);
                    unsigned long long base = 0;
                    if (lane == 31) base = atomicAdd(cb.counter, (unsigned long long)wtot);
                    base = __shfl_sync(kFull, base, 31) + (incl - nc);
#pragma unroll
                    for (int b = 0; b < 4; b++) {
                        if (!((cmask >> b) & 1u)) continue;
                        if (base < cb.cap) {
                            const float d = MET == kMetricL1 ? acc[a][b] : sqrtf(acc[a][b]);
                            const float lb = fmaxf(d - slack(ix, d, 0.f), 0.f) * (1.f - 1e-6f);
                            cb.q[base] = q;
                            cb.e[base] = pos + e0 + b;
                            cb.lb[base] = MET == kMetricL2 ? lb * lb : lb;
                        }
                        base++;
                    }
                }
                if (any_ub) {
                    // shrink once per tile row; later tiles of this block see it via s_r
                    __threadfence();
                    fhist_shrink(fhist, r0, ks, r32, r64, q);
                    atomicMin(reinterpret_cast<int *>(s_r + row), __float_as_int(__ldcg(r32 + q)));
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < 128) {
            const int q = s_q[threadIdx.x];
            const unsigned v = q >= 0 ? s_ver[threadIdx.x] : 0u;
            if (stats_on && v) atomicAdd(verified_stat + q, (unsigned long long)v);
            if (work) {
                // one work-counter atomic per warp (a per-row atomic on one
                // address serialises the profiling pass)
                const unsigned wsum = __reduce_add_sync(kFull, v);
                if (lane == 0 && wsum) atomicAdd(work + kWorkPairs, (unsigned long long)wsum);
            }
        }
        if (threadIdx.x == 0) {
            w_entries += (unsigned long long)size * item.count;
            w_rows += (unsigned long long)item.count;
        }
    }
    if (work && threadIdx.x == 0) {
        atomicAdd(work + kWorkEntries, w_entries);
        atomicAdd(work + kWorkRows, w_rows);
    }
}

// ---------------------------------------------------------------------------
// Tensor-core verification for dense L2 (north_star: "norm-expansion MMA with
// an exact recheck").  One work item = (leaf, up to 128 queries): a
// kind::f16 (bf16 in, fp32 accumulate) tcgen05 MMA of M=128 queries x
// N=leaf entries x K=D into TMEM.  Both operands are centred on the leaf's
// pivot c, so
//     d^2(q,o) = dqp^2 + dis^2 - 2 (q-c).(o-c)
// reuses the pivot distances the tree already holds and keeps operand norms
// small.  bf16 rounding (2^-9 per operand) bounds the dot error by
// 2^-8 ||q-c|| ||o-c||, i.e. d^2 by 2^-7 dqp dis; the screen uses twice that.
// Every entry passing lemma 1 whose approximate d^2 is within the band of r^2
// is recomputed exactly in float64 (numpy order), so answers are exact.
// ~64 KB of shared memory per CTA: three CTAs per SM overlap each other's
// staging, MMA and epilogue.
// ---------------------------------------------------------------------------
// kNN shrinking bound for float metrics: per-query 64-bin histogram of the
// exact distances found so far over [0, r0] (r0 = the probe radius).  The
// upper edge of the bin where the count reaches k bounds the k-th distance
// from above (k distinct real objects lie at or below it), so the radius can
// only shrink to values that still admit every true answer and its ties.
constexpr int kFHist = 64;   // bins per query (256 bins: a 4x longer scan per shrink, 12% slower on 128-d)
// Bins split [0, r0] evenly; the upper edge of bin t is (t + 1) r0 / 64.
// (Bins focused on [0.75 r0, r0] measured worse: the probe radius is often
// well above the k-th distance, so the bound stuck at 0.75 r0 -- 98M instead
// of 63M tie-inclusive kNN hits on 128-d, 22.6k vs 28.2k q/s on the L1 shard.)
__device__ __forceinline__ int fhist_bin(double d, double R0)
{
    return min(max((int)(d / R0 * kFHist), 0), kFHist - 1);
}

__device__ __forceinline__ double fhist_edge(int t, double R0)
{
    return (double)(t + 1) / kFHist * R0 * (1.0 + 1.0 / (1 << 20));
}

__device__ __forceinline__ void fhist_add(unsigned *hist, const float *r0, int q, double d)
{
    const double R0 = (double)r0[q];
    if (!(d <= R0) || !(R0 > 0.0) || isinf(R0)) return;
    atomicAdd(hist + (size_t)q * kFHist + fhist_bin(d, R0), 1u);
}

__device__ __forceinline__ void fhist_shrink(unsigned *hist, const float *r0, const int32_t *ks, float *r32,
                                             double *r64, int q)
{
    const double R0 = (double)r0[q];
    if (!(R0 > 0.0) || isinf(R0)) return;
    const uint4 *h4 = reinterpret_cast<const uint4 *>(hist + (size_t)q * kFHist);
    const unsigned k = (unsigned)ks[q];
    unsigned run = 0;
    int t = -1;
    // 16 bins per batch: four independent L2 loads in flight instead of one
    // dependent load per 4 bins (a shrink sits on the kernel's critical path)
    for (int b = 0; b < kFHist / 16 && t < 0; b++) {
        uint4 v[4];
#pragma unroll
        for (int i = 0; i < 4; i++) v[i] = __ldcg(h4 + 4 * b + i);
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const unsigned c[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int j = 0; j < 4; j++) {
                run += c[j];
                if (t < 0 && run >= k) t = 16 * b + 4 * i + j;
            }
        }
    }
    if (t < 0) return;
    const double R = fhist_edge(t, R0);
    if (R < r64[q]) {
        atomicMin(reinterpret_cast<unsigned long long *>(r64 + q), (unsigned long long)__double_as_longlong(R));
        float Rf = (float)R;
        if ((double)Rf < R) Rf = nextafterf(Rf, INFINITY);
        atomicMin(reinterpret_cast<int *>(r32 + q), __float_as_int(Rf));
    }
}

constexpr int kMmaThreads = 256;  // 8 warps: warps w and w+4 share TMEM lane quadrant w%4
// TMEM columns per CTA: power of two >= the largest leaf (N <= 256); the
// host launches at most 512 / cols CTAs per SM so allocation never waits.

__global__ void __launch_bounds__(kMmaThreads, 3) k_leafgroup_mma(IndexView ix, QueryView qv, const Row *__restrict__ srows,
                                                                   const Item *__restrict__ items, int nitems,
                                                                   float *r32, double *r64, HitBuf out,
                                                                   unsigned long long *verified_stat, int stats_on,
                                                                   unsigned long long *work, uint32_t tmem_cols,
                                                                   unsigned long long *phase_clk, unsigned *fhist,
                                                                   const float *r0, const int32_t *ks)
{
    long long t_stage = 0, t_wait = 0, t_epi = 0;
    extern __shared__ __align__(1024) uint8_t smraw[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_slot;
    __shared__ float s_dis[256];
    __shared__ uint8_t s_al[256];
    __shared__ int s_q[128];
    // 1024-byte alignment for the 128-byte swizzle, kept as an index into the
    // shared array so the compiler emits STS (not generic stores)
    const uint32_t pad = (1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u;
    uint8_t *sm = smraw + pad;
    const int tid = threadIdx.x, warp = tid >> 5;
    const int nkb = ix.Dk >> 6;           // 64 bf16 (128 bytes) per K-block row
    uint8_t *A = sm;
    uint8_t *B = sm + (size_t)nkb * 128 * 128;
    if (warp == 0) tc::tmem_alloc(&tmem_slot, tmem_cols);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_slot;
    uint32_t phase = 0;
    const int c16 = ix.Dk >> 3;           // 16-byte chunks (8 bf16) per row
    const int dp4 = ix.Dp >> 2;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const Item item = items[it];
        const NodeRec leaf = ix.node[item.leaf];
        const int pos = ix.npos[item.leaf];
        const int N = max(16, (leaf.size + 15) & ~15);
        const float4 *pv = reinterpret_cast<const float4 *>(ix.vec32 + (size_t)leaf.piv * ix.Dp);
        const long long c_a = clock64();
        if (tid < 128) s_q[tid] = tid < item.count ? srows[item.start + tid].q : -1;
        for (int j = tid; j < leaf.size; j += blockDim.x) {
            s_dis[j] = __ldg(ix.dis + pos + j);
            s_al[j] = is_alive(ix.alive, pos + j) ? 1 : 0;
        }
        __syncthreads();
        // A: query rows centred on the leaf pivot, rounded to bf16 (zero pad)
        constexpr int kBatch = 4;
        for (int t0 = tid; t0 < 128 * c16; t0 += kBatch * kMmaThreads) {
            uint4 pk[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; u++) {
                const int t = t0 + u * kMmaThreads;
                const int row = t / c16, c = t - row * c16;
                pk[u] = make_uint4(0u, 0u, 0u, 0u);
                const int q = (t < 128 * c16) ? s_q[row] : -1;
                if (q >= 0 && 2 * c < dp4) {
                    const float4 *qp = reinterpret_cast<const float4 *>(qv.vec32 + (size_t)q * ix.Dp);
                    const float4 x0 = __ldg(qp + 2 * c), y0 = __ldg(pv + 2 * c);
                    float4 x1 = make_float4(0.f, 0.f, 0.f, 0.f), y1 = x1;
                    if (2 * c + 1 < dp4) { x1 = __ldg(qp + 2 * c + 1); y1 = __ldg(pv + 2 * c + 1); }
                    __nv_bfloat162 b0 = __floats2bfloat162_rn(x0.x - y0.x, x0.y - y0.y);
                    __nv_bfloat162 b1 = __floats2bfloat162_rn(x0.z - y0.z, x0.w - y0.w);
                    __nv_bfloat162 b2 = __floats2bfloat162_rn(x1.x - y1.x, x1.y - y1.y);
                    __nv_bfloat162 b3 = __floats2bfloat162_rn(x1.z - y1.z, x1.w - y1.w);
                    pk[u] = make_uint4(*reinterpret_cast<uint32_t *>(&b0), *reinterpret_cast<uint32_t *>(&b1),
                                       *reinterpret_cast<uint32_t *>(&b2), *reinterpret_cast<uint32_t *>(&b3));
                }
            }
#pragma unroll
            for (int u = 0; u < kBatch; u++) {
                const int t = t0 + u * kMmaThreads;
                if (t < 128 * c16) {
                    const int row = t / c16, c = t - row * c16;
                    *reinterpret_cast<uint4 *>(A + (c >> 3) * 16384 + tc::sw128_offset(row, c & 7)) = pk[u];
                }
            }
        }
        // B: the leaf's centred bf16 entries (contiguous rows)
        for (int t0 = tid; t0 < N * c16; t0 += kBatch * kMmaThreads) {
            uint4 pk[kBatch];
#pragma unroll
            for (int u = 0; u < kBatch; u++) {
                const int t = t0 + u * kMmaThreads;
                const int row = t / c16, c = t - row * c16;
                pk[u] = make_uint4(0u, 0u, 0u, 0u);
                if (t < N * c16 && row < leaf.size) pk[u] = __ldg(ix.vcent + (size_t)(pos + row) * c16 + c);
            }
#pragma unroll
            for (int u = 0; u < kBatch; u++) {
                const int t = t0 + u * kMmaThreads;
                if (t < N * c16) {
                    const int row = t / c16, c = t - row * c16;
                    *reinterpret_cast<uint4 *>(B + (size_t)(c >> 3) * N * 128 + tc::sw128_offset(row, c & 7)) = pk[u];
                }
            }
        }
        tc::fence_async_smem();
        __syncthreads();
        const long long c_b = clock64();
        if (tid == 0) {
            tc::fence_after_sync();
            const uint32_t idesc = tc::idesc_bf16(128, N);
            const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
            for (int kb = 0; kb < nkb; kb++) {
#pragma unroll
                for (int ks = 0; ks < 4; ks++) {   // K = 16 bf16 = 32 bytes per MMA
                    const uint64_t ad = tc::desc_k_sw128(a0 + kb * 16384 + ks * 32);
                    const uint64_t bd = tc::desc_k_sw128(b0 + kb * N * 128 + ks * 32);
                    tc::mma_bf16(tmem, ad, bd, idesc, (kb | ks) ? 1u : 0u);
                }
            }
            tc::mma_commit(&mbar);
        }
        tc::mbar_wait(&mbar, phase);
        phase ^= 1u;
        tc::fence_after_sync();
        const long long c_c = clock64();
        // epilogue: query row = TMEM lane 32*(warp%4)+lane; warps w and w+4
        // split the N columns in halves
        const int qrow = 32 * (warp & 3) + (tid & 31);
        const int half = warp >> 2;
        const int cbeg = half ? ((N >> 5) << 4) : 0;            // multiple of 16
        const int cend = half ? N : ((N >> 5) << 4);
        const bool valid = qrow < item.count;
        int q = 0;
        float dqp = 0.f, r = 0.f;
        double rr = 0.0;
        if (valid) {
            const Row lr = srows[item.start + qrow];
            q = lr.q;
            dqp = lr.dqp;
            r = __ldcg(r32 + q);
            rr = __ldcg(r64 + q);
        }
        const bool inf_r = isinf(r);
        const float R2 = r * r * (1.f + 1e-6f);
        unsigned nhits = 0;
        const float kd = ldexpf(dqp, -6);
        const float kq = 8.f * ix.rel * dqp * dqp + 4.f * ix.abs_eps * (dqp + ix.abs_eps);
        unsigned ver = 0;
        const uint32_t lane_base = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        for (int c0 = cbeg; c0 < cend; c0 += 16) {
            float acc[16];
            tc::tmem_ld16(lane_base + (uint32_t)c0, acc);   // warp-collective: every thread runs it
            if (!valid) continue;
#pragma unroll
            for (int jj = 0; jj < 16; jj++) {
                const int j = c0 + jj;
                if (j >= leaf.size || !s_al[j]) continue;
                const float dis = s_dis[j];
                if (!lemma1_in(dis, lemma1_range(ix, dqp, r))) continue;   // lemma 1
                ver++;
                bool cand = inf_r;
                if (!cand) {
                    const float d2a = dqp * dqp + dis * dis - 2.f * acc[jj];
                    const float err = kd * dis + kq + 8.f * ix.rel * dis * dis + 4.f * ix.abs_eps * dis;
                    cand = d2a <= R2 + err;
                }
                if (cand) {
                    const double d64 = vdist64<kMetricL2>(ix, qv, q, pos + j);
                    if (d64 <= rr) {
                        const unsigned long long sl = atomicAdd(out.counter, 1ull);
                        if (sl < out.cap) { out.q[sl] = q; out.e[sl] = pos + j; out.d[sl] = d64; }
                        if (fhist) fhist_add(fhist, r0, q, d64);
                        nhits++;
                    }
                }
            }
        }
        if (fhist && valid && nhits) fhist_shrink(fhist, r0, ks, r32, r64, q);
        if (valid && stats_on && ver) atomicAdd(verified_stat + q, (unsigned long long)ver);
        if (work && valid) atomicAdd(work + kWorkPairs, (unsigned long long)ver);
        if (work && tid == 0) {
            atomicAdd(work + kWorkEntries, (unsigned long long)leaf.size * item.count);
            atomicAdd(work + kWorkRows, (unsigned long long)item.count);
            atomicAdd(work + kWorkSteps, (unsigned long long)128 * N * ix.Dk);   // MMA MACs issued
        }
        tc::fence_before_sync();
        __syncthreads();
        const long long c_d = clock64();
        t_stage += c_b - c_a;
        t_wait += c_c - c_b;
        t_epi += c_d - c_c;
    }
    if (phase_clk && tid == 0) {
        atomicAdd(phase_clk + 0, (unsigned long long)t_stage);
        atomicAdd(phase_clk + 1, (unsigned long long)t_wait);
        atomicAdd(phase_clk + 2, (unsigned long long)t_epi);
    }
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, tmem_cols);
}

// ---------------------------------------------------------------------------
// Pending-insert cache (StreamingIndex, updates.py:109-215): a small set of
// objects not yet in the tree, scanned exactly for every query of the batch
// (one extra leaf with no pivot filter).  Hits carry entry id -(slot+1).
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// Tensor-core L2 verification, pipelined (k_leafgroup_mma2, the default).
// Differences from k_leafgroup_mma:
//  * A = the item's 128 query rows in bf16 exactly as uploaded (no per-item
//    centring / conversion): cp.async gathers them straight into the 128-byte
//    swizzled layout.  The pivot term is folded in per entry:
//        (q - c).(o - c)  ~=  q_bf16 . v_e  -  c . v_e,   v_e = bf16(o_e - c)
//    with se_e = c . v_e precomputed at index build, so
//        d^2 ~= dqp^2 + dis^2 - 2 (acc - se_e).
//    Error: |eps . v| + |(q - c) . delta| <= 2^-9 (|q| + dqp) dis per dot
//    (bf16 rounding of q and of o - c); the screen uses 2^-8, i.e. 2x margin.
//  * two smem stages and two TMEM accumulators: item i+1's operands are in
//    flight (cp.async) while item i's epilogue runs.
//  * the epilogue only screens; pairs whose approximate d^2 is within the
//    error band of r^2 go to a candidate list, and k_recheck recomputes
//    them exactly in float64 (numpy order) against the FINAL radius, so no
//    thread of an item stalls the block on a float64 recompute.
//  * kNN: candidates whose d^2 UPPER bound is inside the radius feed the
//    per-query histogram (their true distance is at most that bound), so the
//    radius shrinks as the pass goes, exactly as with exact hits.
// ---------------------------------------------------------------------------
// Two shapes (template NT threads, NSTAGE operand stages / accumulators):
//  * NT = 512, NSTAGE = 2 (default): one CTA per SM; MMA i+1 overlaps the
//    epilogue of item i inside the CTA;
//  * NT = 256, NSTAGE = 1 (GTS_MMA_SHAPE=256): two CTAs per SM (91 KB of
//    shared memory, 128 TMEM columns each), MMA i+1 issued after the item-i
//    barrier, in the hope that the other CTA covers barrier waits (ncu: the
//    barrier is the top stall of the one-CTA shape).  Measured slower on
//    B200 (443 vs 343 ms of this kernel per vec128 step).
template <int NT, int NSTAGE>
__global__ void __launch_bounds__(NT, NT == 512 ? 1 : 2)
k_leafgroup_mma2(IndexView ix, QueryView qv, const Row *__restrict__ srows, const Item *__restrict__ items, int nitems,
                 unsigned long long *item_cursor, float *r32, double *r64, CandBuf cb,
                 unsigned long long *verified_stat, int stats_on, unsigned long long *work, uint32_t acc_cols,
                 int nmax, unsigned *fhist, const float *r0, const int32_t *ks)
{
    // Software pipeline over this CTA's items (static order it_i = bid + i*G).
    //   NSTAGE 2, iteration i: wait MMA i | issue MMA i+1 (its operands landed
    //   last iteration) | cp.async operands of item i+2 into the stage MMA i
    //   just released | global loads of item i+3's row/column metadata and
    //   item i+4's descriptor (registers) | epilogue of item i (TMEM
    //   accumulator i & 1) | store the loaded metadata | barrier.
    //   NSTAGE 1: wait MMA i | cp.async operands of item i+1 into the stage
    //   MMA i released | metadata / descriptor loads | epilogue of item i |
    //   stores | barrier | MMA i+1.
    // Every global-load latency is hidden behind an epilogue; one block
    // barrier per item.
    constexpr int LA = NSTAGE == 2 ? 1 : 0;   // extra lookahead of the two-stage order
    extern __shared__ __align__(1024) uint8_t smraw[];
    __shared__ uint64_t mbar[NSTAGE];
    __shared__ uint32_t tmem_slot;
    __shared__ int4 s_item[8];           // {leaf, start, count, size}, ring by i % 8
    __shared__ int4 s_itemraw[8][2];     // raw Item copies (cp.async) before they become s_item
    __shared__ int s_pos[8];
    __shared__ float4 s_col[4][256];     // ring by i % 4 (see meta_store)
    __shared__ int s_rq[4][128];         // query ids (-1: no row)
    __shared__ float4 s_rf[4][128];      // {dqp, r at load time (radii only shrink), |q|, probe radius}
    (void)item_cursor;
    const uint32_t pad = (1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u;
    uint8_t *sm = smraw + pad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nkb = ix.Dk >> 6;
    const int c16 = ix.Dk >> 3;
    const size_t a_bytes = (size_t)nkb * 16384;
    const size_t stage_bytes = a_bytes + (size_t)nkb * nmax * 128;
    const int G = gridDim.x;
    auto idx = [&](int i) { return (int)blockIdx.x + i * G; };
    if (warp == 0) tc::tmem_alloc(&tmem_slot, NSTAGE * acc_cols);
    if (tid == 0) {
        for (int k = 0; k < NSTAGE; k++) tc::mbar_init(&mbar[k], 1);
        tc::fence_mbar_init();
    }
    // descriptors of items 0..3 ({leaf, start, count, size}, pos)
    if (tid < 4) {
        int4 d = make_int4(0, 0, 0, 0);
        int p0 = 0;
        if (idx(tid) < nitems) {
            const Item it = items[idx(tid)];
            d = make_int4(it.leaf, it.start, it.count, it.size);
            p0 = it.pos;
        }
        s_item[tid] = d;
        s_pos[tid] = p0;
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_slot;

    // metadata loads of item i (registers), then the store into ring slot i % 4.
    // Threads 0..127 load row i's {q, dqp, r, |q|, r0}; the others the
    // columns j = tid - 128 (+ NT - 128) {dis, se, alive}; packed floats, so
    // few registers stay live across the epilogue.
    constexpr int CPT = NT == 512 ? 1 : 2;   // columns per thread (<= 256 columns)
    struct Meta {
        float4 a;
        float b;
        float4 c2;   // second column (CPT 2)
    };
    auto meta_load = [&](int i, Meta &m) {
        const int4 d = s_item[i & 7];
        const int pos = s_pos[i & 7];
        m.a = make_float4(0.f, -1.f, 0.f, 0.f);
        m.b = __int_as_float(-1);
        m.c2 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (idx(i) >= nitems) return;
        if (tid < 128) {
            if (tid < d.z) {
                const Row lr = srows[d.y + tid];
                m.b = __int_as_float(lr.q);
                m.a = make_float4(lr.dqp, __ldcg(r32 + lr.q), qv.qn[lr.q], r0 ? r0[lr.q] : 0.f);
            }
        } else {
            const int j = tid - 128;
            if (j < d.w) {
                m.a.x = __ldg(ix.dis + pos + j);
                m.a.y = __ldg(ix.vse + pos + j);
                m.a.z = is_alive(ix.alive, pos + j) ? 1.f : 0.f;
            }
            if (CPT == 2 && j + (NT - 128) < d.w) {
                const int j2 = j + (NT - 128);
                m.c2.x = __ldg(ix.dis + pos + j2);
                m.c2.y = __ldg(ix.vse + pos + j2);
                m.c2.z = is_alive(ix.alive, pos + j2) ? 1.f : 0.f;
            }
        }
    };
    auto meta_store = [&](int i, const Meta &m) {
        const int sl = i & 3;
        const int4 d = s_item[i & 7];
        const int N = max(16, (d.w + 15) & ~15);
        // {dis | NaN, y - z | NaN, y + z, dis}: NaN (tombstone / padding)
        // fails the lemma-1 window and the screen
        auto put = [&](int j, const float4 &mc) {
            const float nan = __int_as_float(0x7fc00000);
            float4 col = make_float4(nan, nan, 0.f, INFINITY);
            if (j < d.w) {
                const float dis = mc.x, se = mc.y;
                const float y = fmaf(dis, dis, 2.f * se), z = 8.f * ix.rel * dis * dis;
                if (mc.z != 0.f) {
                    col.x = dis;
                    col.y = y - z;
                }
                col.z = y + z;
                col.w = dis;
            }
            s_col[sl][j] = col;
        };
        if (tid < 128) {
            s_rq[sl][tid] = __float_as_int(m.b);
            s_rf[sl][tid] = m.a;
        } else {
            if (tid - 128 < N) put(tid - 128, m.a);
            if (CPT == 2 && tid - 128 + (NT - 128) < N) put(tid - 128 + (NT - 128), m.c2);
        }
    };
    // operands of item i into smem stage i % NSTAGE (async)
    auto stage = [&](int i) {
        const int st = NSTAGE == 2 ? (i & 1) : 0;
        const int4 d = s_item[i & 7];
        const int pos = s_pos[i & 7];
        const int N = max(16, (d.w + 15) & ~15);
        const uint32_t A = tc::smem_u32(sm + st * stage_bytes);
        const uint32_t B = A + (uint32_t)a_bytes;
        const int lc = c16 == 16 ? 4 : 3;
        const int c = tid & (c16 - 1), row0 = tid >> lc, rstep = NT >> lc;
        // rstep is a multiple of 8, so every row this thread copies has the
        // same (row & 7) and the same SW128 chunk permutation: the smem
        // address advances by rstep rows, the source by rstep (B) or by a
        // 32-bit row index (A) -- a few instructions per 16-byte copy.
        const uint32_t sw = tc::sw128_offset(row0, c & 7);
        const uint32_t dstep = (uint32_t)rstep * 128u;
        const int *rq = s_rq[i & 3];
        const char *qsrc = reinterpret_cast<const char *>(qv.qbf + c);
        const uint32_t qstride = (uint32_t)c16 * 16u;
        uint32_t adst = A + (uint32_t)(c >> 3) * 16384u + sw;
#pragma unroll 4
        for (int row = row0; row < 128; row += rstep, adst += dstep) {
            const int q = rq[row];
            tc::cp_async16(adst, qsrc + (size_t)((uint32_t)max(q, 0) * (uint64_t)qstride), q >= 0 ? 16u : 0u);
        }
        // rows size..N-1 (padding) are zero-filled (src-size 0); their source
        // addresses stay inside vcent's 16-row zero tail
        const uint4 *bsrc = ix.vcent + (size_t)(pos + row0) * c16 + c;
        const size_t sstep = (size_t)rstep * c16;
        uint32_t bdst = B + (uint32_t)(c >> 3) * (uint32_t)N * 128u + sw;
        for (int row = row0; row < N; row += rstep, bdst += dstep, bsrc += sstep)
            tc::cp_async16(bdst, bsrc, row < d.w ? 16u : 0u);
        tc::cp_async_commit();
    };
    auto mma = [&](int i) {
        if (tid != 0) return;
        tc::fence_after_sync();
        const int st = NSTAGE == 2 ? (i & 1) : 0;
        const int N = max(16, (s_item[i & 7].w + 15) & ~15);
        const uint32_t idesc = tc::idesc_bf16(128, N);
        const uint32_t a0 = tc::smem_u32(sm + st * stage_bytes), b0 = a0 + (uint32_t)a_bytes;
        for (int kb = 0; kb < nkb; kb++) {
#pragma unroll
            for (int k4 = 0; k4 < 4; k4++) {
                const uint64_t ad = tc::desc_k_sw128(a0 + kb * 16384 + k4 * 32);
                const uint64_t bd = tc::desc_k_sw128(b0 + kb * N * 128 + k4 * 32);
                tc::mma_bf16(tmem + st * acc_cols, ad, bd, idesc, (kb | k4) ? 1u : 0u);
            }
        }
        tc::mma_commit(&mbar[st]);
    };

    // prologue: metadata of items 0..1+LA, operands of items 0..LA, MMA of item 0
    {
        Meta m0, m1, m2;
        meta_load(0, m0);
        meta_load(1, m1);
        if (LA) meta_load(2, m2);
        meta_store(0, m0);
        meta_store(1, m1);
        if (LA) meta_store(2, m2);
    }
    __syncthreads();
    if (idx(0) < nitems) {
        stage(0);
        if (LA && idx(1) < nitems) stage(1);
        tc::cp_async_wait_all();
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        mma(0);
    }
    uint32_t phase[2] = {0u, 0u};
    unsigned long long pairs = 0, w_entries = 0, w_rows = 0, w_macs = 0;
    for (int i = 0; idx(i) < nitems; i++) {
        const int s = NSTAGE == 2 ? (i & 1) : 0;
        // MMA i done: its accumulator is ready and its operand stage is free
        tc::mbar_wait(&mbar[s], phase[s]);
        phase[s] ^= 1u;
        tc::fence_after_sync();
        if (LA && idx(i + 1) < nitems) mma(i + 1);
        if (idx(i + 1 + LA) < nitems) stage(i + 1 + LA);
        Meta mnext;
        meta_load(i + 2 + LA, mnext);
        // descriptor of item i+3+LA: a 32-byte async copy straight into smem
        const int nd = i + 3 + LA;
        if (tid == 0 && idx(nd) < nitems) {
            const Item *src = items + idx(nd);
            tc::cp_async16(tc::smem_u32(&s_itemraw[nd & 7][0]), src, 16u);
            tc::cp_async16(tc::smem_u32(&s_itemraw[nd & 7][1]), reinterpret_cast<const int4 *>(src) + 1, 16u);
            tc::cp_async_commit();
        }
        // ---- epilogue of item i (accumulator s, metadata slot i % 4) ----
        // thread = one query row (TMEM lane) x every 4th 16-column chunk;
        // per column: lemma 1, approximate d^2, error band, ~12 instructions
        {
            const int sl = i & 3;
            const int4 d = s_item[i & 7];
            const int size = d.w;
            const int pos = s_pos[i & 7];
            const int N = max(16, (size + 15) & ~15);
            const int qrow = 32 * (warp & 3) + lane;
            const int part = warp >> 2;   // NT / 128 parts of the columns
            const int q = s_rq[sl][qrow];
            const bool valid = q >= 0;
            const float4 rf = s_rf[sl][qrow];
            const float dqp = rf.x, qnorm = rf.z;
            float r = rf.y;
            // folded thresholds: with y - z, y + z per column,
            //   screen    (y - z) - 2 acc - cA dis <= R2 + kq - dq2 + margin  (T1)
            //   ub inside (y + z) - 2 acc + cA dis <= R2 - kq - dq2 - margin  (T2)
            // margin 2^-18 (dq2 + qn^2 + R2) covers the fp32 rounding of the
            // rearranged sums; the band itself has a 2x margin.
            const float dq2 = dqp * dqp;
            const float cA = ((dqp + qnorm) * 0x1p-7f) + ((qnorm) * 0x1p-18f) + 4.f * ix.abs_eps;
            const float kq = 8.f * ix.rel * dq2 + 4.f * ix.abs_eps * (dqp + ix.abs_eps);
            float T1, T2;
            auto set_r = [&](float rr) {
                const float R2 = rr * rr * (1.f + 1e-6f);
                const float mg = ((dq2 + qnorm * qnorm + R2) * 0x1p-18f);
                T1 = R2 + kq - dq2 + mg;
                T2 = R2 - kq - dq2 - mg;
            };
            set_r(r);   // loaded two items ago: stale radii are larger, i.e. conservative
            // lemma-1 window for the item (a kNN shrink inside it narrows only
            // the screen; the wider window counts a few more entries as
            // verified, which float-metric stats allow)
            const float2 rg = lemma1_range(ix, dqp, r);
            float hinv = 0.f;   // kNN histogram: bins per unit distance
            if (fhist && valid) {
                const float R0 = rf.w;
                hinv = (R0 > 0.f && !isinf(R0)) ? (float)kFHist / R0 : 0.f;
            }
            unsigned ver = 0;
            const uint32_t lane_base = tmem + s * acc_cols + ((uint32_t)((warp & 3) * 32) << 16);
            const float4 *cols = s_col[sl];
            for (int c0 = 16 * part; c0 < N; c0 += 16 * (NT / 128)) {
                float acc[16];
                tc::tmem_ld16(lane_base + (uint32_t)c0, acc);   // warp-collective
                uint32_t win = 0, cm = 0;
#pragma unroll
                for (int jj = 0; jj < 16; jj++) {
                    const float4 col = cols[c0 + jj];   // broadcast LDS.128
                    const float m2a = fmaf(-2.f, acc[jj], col.y);
                    win |= (uint32_t)lemma1_in(col.x, rg) << jj;
                    cm |= (uint32_t)(fmaf(-cA, col.w, m2a) <= T1) << jj;
                }
                ver += __popc(win);
                uint32_t fm = 0;
                if (hinv > 0.f && (cm & win)) {
                    // kNN: candidates whose d^2 upper bound is inside the radius
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        const float4 col = cols[c0 + jj];
                        fm |= (uint32_t)(fmaf(cA, col.w, fmaf(-2.f, acc[jj], col.z)) <= T2) << jj;
                    }
                }
                cm &= win;
                fm &= cm;
                if (!valid) cm = fm = 0, ver = 0;
                // warp-aggregated append of the chunk's candidates (most
                // chunks have none: one vote skips the scan)
                if (__any_sync(kFull, cm)) {
                    const unsigned nc = __popc(cm);
                    unsigned incl = nc;
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned v = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const unsigned wtot = __shfl_sync(kFull, incl, 31);
                    unsigned long long base = 0;
                    if (lane == 31) base = atomicAdd(cb.counter, (unsigned long long)wtot);
                    base = __shfl_sync(kFull, base, 31) + (incl - nc);
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        if (!((cm >> jj) & 1u)) continue;
                        if (base < cb.cap) {
                            const float4 col = s_col[sl][c0 + jj];
                            cb.q[base] = q;
                            cb.e[base] = pos + c0 + jj;
                            // d^2 lower bound, rounded down a little
                            cb.lb[base] = (fmaf(-cA, col.w, fmaf(-2.f, acc[jj], col.y)) + dq2 - kq) * (1.f - 1e-5f) -
                                          ((dq2 + qnorm * qnorm) * 0x1p-18f);
                        }
                        base++;
                    }
                }
                if (fm && hinv > 0.f) {
                    // candidates whose d^2 upper bound is inside the radius: their
                    // true distance is <= that bound, so they may shrink it
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        if (!((fm >> jj) & 1u)) continue;
                        const float4 col = s_col[sl][c0 + jj];
                        const float d2u = fmaf(cA, col.w, fmaf(-2.f, acc[jj], col.z)) + dq2 + kq +
                                          ((dq2 + qnorm * qnorm) * 0x1p-18f);
                        const float dub = sqrtf(fmaxf(d2u, 0.f)) * (1.f + 1e-6f) + 1e-30f;
                        const int b = min((int)(dub * hinv * (1.f + 1e-6f)), kFHist - 1);
                        atomicAdd(fhist + (size_t)q * kFHist + b, 1u);
                    }
                    __threadfence();
                    fhist_shrink(fhist, r0, ks, r32, r64, q);
                    r = __ldcg(r32 + q);
                    set_r(r);
                }
            }
            if (valid && stats_on && ver) atomicAdd(verified_stat + q, (unsigned long long)ver);
            pairs += ver;
            if (tid == 0) {
                w_entries += (unsigned long long)size * d.z;
                w_rows += (unsigned long long)d.z;
                w_macs += (unsigned long long)128 * N * ix.Dk;   // MMA MACs issued
            }
        }
        // metadata of item i+2+LA and the descriptor of item i+3+LA (loads done by now)
        meta_store(i + 2 + LA, mnext);
        tc::cp_async_wait_all();
        if (tid == 0) {
            const int4 r0_ = s_itemraw[nd & 7][0], r1_ = s_itemraw[nd & 7][1];
            s_item[nd & 7] = idx(nd) < nitems ? r0_ : make_int4(0, 0, 0, 0);   // {leaf, start, count, size}
            s_pos[nd & 7] = r1_.x;
        }
        // operands of the next staged item visible to the tensor core; TMEM
        // reads of accumulator s ordered before the MMA that overwrites it
        tc::fence_async_smem();
        tc::fence_before_sync();
        __syncthreads();
        if (!LA && idx(i + 1) < nitems) mma(i + 1);
    }
    if (work) {
        for (int o = 16; o > 0; o >>= 1) pairs += __shfl_down_sync(kFull, pairs, o);
        if (lane == 0) atomicAdd(work + kWorkPairs, pairs);
        if (tid == 0) {
            atomicAdd(work + kWorkEntries, w_entries);
            atomicAdd(work + kWorkRows, w_rows);
            atomicAdd(work + kWorkSteps, w_macs);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tmem, NSTAGE * acc_cols);
}

// ---------------------------------------------------------------------------
// k_leafgroup_mma3: the tensor-core L2 screen as a barrier-free pipeline
// (the default; k_leafgroup_mma2 with GTS_MMA_V2=1).  Same algorithm and
// error band as k_leafgroup_mma2; what changes is the synchronisation:
//  * no block barrier per item.  Stage s (A/B operands, two stages) is
//    filled by cp.async from every thread and completes an mbarrier
//    (full[s], 512 noinc arrivals); the MMA's commit completes mma_done[s];
//    each warp waits mma_done[s] before reading accumulator s (two TMEM
//    accumulators) and after its last TMEM read arrives on acc_free[s] (16
//    arrivals); one thread waits full and acc_free and issues the next MMA.
//    Warps drift up to one item apart instead of meeting at a barrier.
//  * no shared-memory metadata rings for rows: a thread owns one
//    accumulator row (TMEM lane) and one quarter of the columns, loads its
//    row's {q, dqp, r, |q|, r0} into registers in three pipelined steps
//    (descriptor four items ahead, row three, radii two) and copies its
//    quarter of the row's bf16 query vector.  The per-entry column terms
//    {dis | NaN, y - z | NaN, y + z, dis} are precomputed per call
//    (k_colrec) and copied with the operands into a four-slot smem ring.
// ---------------------------------------------------------------------------
constexpr int kM3Threads = 512;   // 16 warps: 4 per TMEM lane quadrant

// vcent per leaf in the MMA's shared-memory image: leaf l owns R = rows[l]
// (its slot capacity rounded up to 16) rows; K-block kb of row r, 16-byte
// chunk c sits at off[l] * 128 + kb * R * 128 + sw128_offset(r, c), so one
// bulk copy of N * 128 bytes per K-block lands a leaf's first N rows in
// exactly the SW128 K-major layout the MMA descriptor reads (rows past the
// capacity are zero).  Rebuilt after in-place inserts.
__global__ void k_vtile(const uint4 *__restrict__ vcent, int c16, const int64_t *__restrict__ dpos,
                        const int64_t *__restrict__ cap, const int32_t *__restrict__ off,
                        const int32_t *__restrict__ rows, int nleaf, uint4 *vtile)
{
    for (int l = blockIdx.x; l < nleaf; l += gridDim.x) {
        const int R = rows[l];
        const int64_t p = dpos[l], cp = cap[l];
        uint4 *dst = vtile + (size_t)off[l] * 8;
        for (int t = threadIdx.x; t < R * c16; t += blockDim.x) {
            const int r = t / c16, c = t - r * c16;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (r < cp) v = vcent[(size_t)(p + r) * c16 + c];
            dst[((size_t)(c >> 3) * R * 128 + tc::sw128_offset(r, c & 7)) >> 4] = v;
        }
    }
}

// per-entry column terms of the screen (see k_leafgroup_mma2's meta_store)
__global__ void k_colrec(IndexView ix, int64_t n, float4 *colrec)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n + 16) return;
    const float nan = __int_as_float(0x7fc00000);
    float4 col = make_float4(nan, nan, 0.f, INFINITY);
    if (e < n) {
        const float dis = ix.dis[e], se = ix.vse[e];
        const float y = fmaf(dis, dis, 2.f * se), z = 8.f * ix.rel * dis * dis;
        if (is_alive(ix.alive, (int)e)) {
            col.x = dis;
            col.y = y - z;
        }
        col.z = y + z;
        col.w = dis;
    }
    colrec[e] = col;
}

__global__ void __launch_bounds__(kM3Threads, 1)
k_leafgroup_mma3(IndexView ix, QueryView qv, const Row *__restrict__ srows, const Item *__restrict__ items, int nitems,
                 const float4 *__restrict__ colrec, float *r32, double *r64, CandBuf cb,
                 unsigned long long *verified_stat, int stats_on, unsigned long long *work, uint32_t acc_cols,
                 int nmax, unsigned *fhist, const float *r0, const int32_t *ks)
{
    extern __shared__ __align__(1024) uint8_t smraw[];
    __shared__ uint64_t full[2], mma_done[2], acc_free[2];
    __shared__ float4 s_col[4][256];   // column terms, ring by item % 4 (see below)
    __shared__ uint32_t tmem_slot;
    const uint32_t pad = (1024u - (tc::smem_u32(smraw) & 1023u)) & 1023u;
    uint8_t *sm = smraw + pad;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int qd = warp & 3, part = warp >> 2;
    const int row = 32 * qd + lane;                  // this thread's accumulator row (TMEM lane)
    const int nkb = ix.Dk >> 6;
    const int c16 = ix.Dk >> 3;                      // 16-byte chunks per bf16 row
    const int lc = c16 == 16 ? 4 : 3;
    const size_t a_bytes = (size_t)nkb * 16384;
    const size_t stage_bytes = a_bytes + (size_t)nkb * nmax * 128;
    const int G = gridDim.x;
    auto idx = [&](int i) { return (int)blockIdx.x + i * G; };
    if (warp == 0) tc::tmem_alloc(&tmem_slot, 2 * acc_cols);
    if (tid == 0) {
        for (int k = 0; k < 2; k++) {
            // + 1: the bulk-copy thread's expect_tx arrival
            tc::mbar_init(&full[k], kM3Threads + (ix.vtile ? 1 : 0));
            tc::mbar_init(&mma_done[k], 1);
            tc::mbar_init(&acc_free[k], kM3Threads / 32);
        }
        tc::fence_mbar_init();
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_slot;

    struct It {   // item descriptor; count (<= 128) and size packed in one word
        int start, cs, pos;
        __device__ int count() const { return cs & 0xff; }
        __device__ int size() const { return cs >> 8; }
    };
    auto item_of = [&](int i) {
        It t{0, 0, 0};
        if (idx(i) < nitems) {
            const Item x = items[idx(i)];
            t = It{x.start, x.count | (x.size << 8), x.pos};
        }
        return t;
    };
    // Row metadata in three pipelined steps, one per iteration, so no load
    // of an iteration waits on another load of the same iteration:
    //   descriptor of item i+4 -> this row's (q, dqp) of item i+3 ->
    //   r, |q|, r0 of item i+2 (queries the row holds)
    struct RowMeta {
        int q;
        float dqp, r, qn, r0;
    };
    auto row_of = [&](const It &t) {
        RowMeta m{-1, 0.f, -1.f, 0.f, 0.f};
        if (row < t.count()) {
            const Row lr = srows[t.start + row];
            m.q = lr.q;
            m.dqp = lr.dqp;
        }
        return m;
    };
    auto finish_meta = [&](RowMeta &m) {
        if (m.q >= 0) {
            m.r = __ldcg(r32 + m.q);
            m.qn = qv.qn[m.q];
            m.r0 = r0 ? r0[m.q] : 0.f;
        }
    };
    // operands of item i into stage i & 1, then this thread's noinc arrival
    // on full[i & 1] (fires when its copies have landed)
    auto stage = [&](int i, const It &t, int q) {
        const int st = i & 1;
        const int N = max(16, (t.size() + 15) & ~15);
        const uint32_t A = tc::smem_u32(sm + st * stage_bytes);
        const uint32_t B = A + (uint32_t)a_bytes;
        // A: this row's query vector, quarter `part` of its chunks
        const int per = c16 >> 2;
        const uint4 *qsrc = qv.qbf + (size_t)max(q, 0) * c16;
#pragma unroll 4
        for (int k = 0; k < per; k++) {
            const int c = part * per + k;
            tc::cp_async16(A + (uint32_t)(c >> 3) * 16384u + tc::sw128_offset(row, c & 7), qsrc + c,
                           q >= 0 ? 16u : 0u);
        }
        // column terms of the item into ring slot i % 4: a warp issuing the
        // copies of item i+2 has passed mma_done(i), and MMA i was issued after
        // acc_free(i-2), so no warp still reads slot (i-2) % 4 = (i+2) % 4;
        // slots i-1 .. i+1 may be in use
        if (tid < N) tc::cp_async16(tc::smem_u32(&s_col[i & 3][tid]), colrec + t.pos + tid, 16u);
        // B: the leaf's centred entries, N rows.  With the leaf images
        // (vtile): one thread posts the byte count and issues one bulk copy
        // per K-block (the TMA engine moves the tile; no per-thread copies).
        // Otherwise per-thread cp.async with rows >= size zero-filled (their
        // source stays inside vcent's 16-row zero tail).
        if (ix.vtile) {
            if (tid == 0) {
                const uint32_t bytes = (uint32_t)N * 128u;
                tc::mbar_arrive_expect_tx(&full[st], bytes * (uint32_t)nkb);
                // the item's image word (its descriptor was read four items
                // ago, so this is an L1 hit; kept out of It for registers)
                const uint32_t tr = (uint32_t)items[idx(i)].pad0;
                const uint4 *src = ix.vtile + (size_t)(tr >> 8) * 128;   // 2 KB = 128 uint4
                const size_t kstride = (size_t)(tr & 0xffu) * 128;       // 16 rows x 128 B
                for (int kb = 0; kb < nkb; kb++)
                    tc::bulk_g2s(B + (uint32_t)kb * bytes, src + kb * kstride, bytes, &full[st]);
            }
        } else {
            const int total = N * c16;
            for (int f = tid; f < total; f += kM3Threads) {
                const int r = f >> lc, c = f & (c16 - 1);
                tc::cp_async16(B + (uint32_t)(c >> 3) * (uint32_t)N * 128u + tc::sw128_offset(r, c & 7),
                               ix.vcent + (size_t)(t.pos + r) * c16 + c, r < t.size() ? 16u : 0u);
            }
        }
        tc::cp_async_mbar_arrive(&full[st]);
    };
    auto mma = [&](int i, const It &t) {
        const int st = i & 1;
        const int N = max(16, (t.size() + 15) & ~15);
        const uint32_t idesc = tc::idesc_bf16(128, N);
        const uint32_t a0 = tc::smem_u32(sm + st * stage_bytes), b0 = a0 + (uint32_t)a_bytes;
        for (int kb = 0; kb < nkb; kb++) {
#pragma unroll
            for (int k4 = 0; k4 < 4; k4++) {
                const uint64_t ad = tc::desc_k_sw128(a0 + kb * 16384 + k4 * 32);
                const uint64_t bd = tc::desc_k_sw128(b0 + kb * N * 128 + k4 * 32);
                tc::mma_bf16(tmem + st * acc_cols, ad, bd, idesc, (kb | k4) ? 1u : 0u);
            }
        }
        tc::mma_commit(&mma_done[st]);
    };

    unsigned long long pairs = 0, w_entries = 0, w_rows = 0, w_macs = 0;
    // row metadata runs two items ahead, so the query id a copy needs is in
    // a register when the copy is issued
    It cur = item_of(0), nxt = item_of(1), nx2 = item_of(2), nx3 = item_of(3);
    RowMeta mc = row_of(cur), mn = row_of(nxt), m2 = row_of(nx2);
    finish_meta(mc);
    finish_meta(mn);
    if (idx(0) < nitems) {
        stage(0, cur, mc.q);
        if (tid == 0) {
            tc::mbar_wait(&full[0], 0u);
            tc::fence_async_smem();
            tc::fence_after_sync();
            mma(0, cur);
        }
    }
    for (int i = 0; idx(i) < nitems; i++) {
        const int s = i & 1;
        const uint32_t ph = (uint32_t)(i >> 1) & 1u;
        const It nx4 = item_of(i + 4);     // step 1
        const RowMeta m3 = row_of(nx3);    // step 2 (descriptor loaded last iteration)
        finish_meta(m2);                   // step 3 (row loaded last iteration)
        // operands of item i+1 into the other stage (MMA i-1, its last reader,
        // completed before this thread's epilogue of item i-1)
        if (idx(i + 1) < nitems) stage(i + 1, nxt, mn.q);
        tc::mbar_wait(&mma_done[s], ph);
        tc::mbar_wait(&full[s], ph);   // (complete already) acquire: the column terms landed
        tc::fence_after_sync();
        // ---- epilogue of item i: row `row`, columns 16 * part + 64 k ----
        {
            const int size = cur.size();
            const int N = max(16, (size + 15) & ~15);
            const int q = mc.q;
            const bool valid = q >= 0;
            const float dqp = mc.dqp, qnorm = mc.qn;
            float r = mc.r;
            const float dq2 = dqp * dqp;
            const float cA = ((dqp + qnorm) * 0x1p-7f) + ((qnorm) * 0x1p-18f) + 4.f * ix.abs_eps;
            const float kq = 8.f * ix.rel * dq2 + 4.f * ix.abs_eps * (dqp + ix.abs_eps);
            float T1, T2;
            auto set_r = [&](float rr) {
                const float R2 = rr * rr * (1.f + 1e-6f);
                const float mg = ((dq2 + qnorm * qnorm + R2) * 0x1p-18f);
                T1 = R2 + kq - dq2 + mg;
                T2 = R2 - kq - dq2 - mg;
            };
            set_r(r);
            const float2 rg = lemma1_range(ix, dqp, r);
            float hinv = 0.f;
            if (fhist && valid) {
                const float R0 = mc.r0;
                hinv = (R0 > 0.f && !isinf(R0)) ? (float)kFHist / R0 : 0.f;
            }
            unsigned ver = 0;
            const uint32_t lane_base = tmem + s * acc_cols + ((uint32_t)(qd * 32) << 16);
            const float4 *cols = s_col[i & 3];
            for (int c0 = 16 * part; c0 < N; c0 += 64) {
                uint32_t ar[16];
                tc::tmem_ld16_issue(lane_base + (uint32_t)c0, ar);
                const int nv = size - c0;   // valid columns of this chunk
                const uint32_t vm = nv >= 16 ? 0xffffu : (nv > 0 ? (1u << nv) - 1u : 0u);
                float4 col[16];
#pragma unroll
                for (int jj = 0; jj < 16; jj++) col[jj] = cols[c0 + jj];   // broadcast LDS.128
                tc::tmem_wait_ld();
                tc::tmem_tie(ar);
                uint32_t win = 0, cm = 0;
#pragma unroll
                for (int jj = 0; jj < 16; jj++) {
                    const float m2a = fmaf(-2.f, __uint_as_float(ar[jj]), col[jj].y);
                    win |= (uint32_t)lemma1_in(col[jj].x, rg) << jj;
                    cm |= (uint32_t)(fmaf(-cA, col[jj].w, m2a) <= T1) << jj;
                }
                win &= vm;
                ver += __popc(win);
                uint32_t fm = 0;
                if (hinv > 0.f && (cm & win)) {
#pragma unroll
                    for (int jj = 0; jj < 16; jj++)
                        fm |= (uint32_t)(fmaf(cA, col[jj].w, fmaf(-2.f, __uint_as_float(ar[jj]), col[jj].z)) <= T2)
                              << jj;
                }
                cm &= win;
                fm &= cm;
                if (!valid) cm = fm = 0, ver = 0;
                if (__any_sync(kFull, cm)) {
                    const unsigned nc = __popc(cm);
                    unsigned incl = nc;
                    for (int o = 1; o < 32; o <<= 1) {
                        const unsigned v = __shfl_up_sync(kFull, incl, o);
                        if (lane >= o) incl += v;
                    }
                    const unsigned wtot = __shfl_sync(kFull, incl, 31);
                    unsigned long long base = 0;
                    if (lane == 31) base = atomicAdd(cb.counter, (unsigned long long)wtot);
                    base = __shfl_sync(kFull, base, 31) + (incl - nc);
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        if (!((cm >> jj) & 1u)) continue;
                        if (base < cb.cap) {
                            cb.q[base] = q;
                            cb.e[base] = cur.pos + c0 + jj;
                            cb.lb[base] = (fmaf(-cA, col[jj].w, fmaf(-2.f, __uint_as_float(ar[jj]), col[jj].y)) + dq2 -
                                           kq) * (1.f - 1e-5f) -
                                          ((dq2 + qnorm * qnorm) * 0x1p-18f);
                        }
                        base++;
                    }
                }
                if (fm && hinv > 0.f) {
#pragma unroll
                    for (int jj = 0; jj < 16; jj++) {
                        if (!((fm >> jj) & 1u)) continue;
                        const float d2u = fmaf(cA, col[jj].w, fmaf(-2.f, __uint_as_float(ar[jj]), col[jj].z)) + dq2 +
                                          kq + ((dq2 + qnorm * qnorm) * 0x1p-18f);
                        const float dub = sqrtf(fmaxf(d2u, 0.f)) * (1.f + 1e-6f) + 1e-30f;
                        const int b = min((int)(dub * hinv * (1.f + 1e-6f)), kFHist - 1);
                        atomicAdd(fhist + (size_t)q * kFHist + b, 1u);
                    }
                    __threadfence();
                    fhist_shrink(fhist, r0, ks, r32, r64, q);
                    r = __ldcg(r32 + q);
                    set_r(r);
                }
            }
            if (valid && stats_on && ver) atomicAdd(verified_stat + q, (unsigned long long)ver);
            pairs += ver;
            if (tid == 0) {
                w_entries += (unsigned long long)size * cur.count();
                w_rows += (unsigned long long)cur.count();
                w_macs += (unsigned long long)128 * N * ix.Dk;
            }
        }
        // accumulator s read by this warp
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&acc_free[s]);
        // MMA of item i+1 into accumulator s^1: its operands landed (full) and
        // every warp finished item i-1, the accumulator's previous user.
        // (Letting the last warp to finish item i issue it instead of thread 0
        // measured slower: 359 vs 293 ms per vec128 step.)
        if (tid == 0 && idx(i + 1) < nitems) {
            tc::mbar_wait(&full[s ^ 1], (uint32_t)((i + 1) >> 1) & 1u);
            if (i >= 1) tc::mbar_wait(&acc_free[s ^ 1], (uint32_t)((i - 1) >> 1) & 1u);
            tc::fence_async_smem();
            tc::fence_after_sync();
            mma(i + 1, nxt);
        }
        __syncwarp();
        cur = nxt;
        nxt = nx2;
        nx2 = nx3;
        nx3 = nx4;
        mc = mn;
        mn = m2;
        m2 = m3;
    }
    if (work) {
        for (int o = 16; o > 0; o >>= 1) pairs += __shfl_down_sync(kFull, pairs, o);
        if (lane == 0) atomicAdd(work + kWorkPairs, pairs);
        if (tid == 0) {
            atomicAdd(work + kWorkEntries, w_entries);
            atomicAdd(work + kWorkRows, w_rows);
            atomicAdd(work + kWorkSteps, w_macs);
        }
    }
    // every MMA was waited (mma_done) before its epilogue; all TMEM reads done
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0) tc::tmem_dealloc(tmem, 2 * acc_cols);
}

// Exact float64 recheck of screened candidates against the final radius
// (kNN radii only ever shrink, so the candidates are a superset).
// Candidates whose lower bound (d^2 for L2, d for L1) is already outside the
// final radius are dropped first.  8 lanes per candidate: lane j accumulates
// numpy's pairwise partial r[j] = sum over i = j (mod 8) in order, then the
// lanes combine ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and add the D % 8 tail
// sequentially -- the same float64 operations as pw_sum64 for D <= 128
// (metrics.py:127-133); larger D runs pw_sum64 on the group's first lane.
template <int MET>
__global__ void k_recheck(IndexView ix, QueryView qv, CandBuf cb, unsigned long long ncand, const float *r32,
                          const double *r64, HitBuf out, int prescreen)
{
    const int lane = lane_id(), j = lane & 7;
    const unsigned long long i = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 3;
    bool live = false;
    int q = 0, e = 0;
    if (i < ncand) {
        q = cb.q[i];
        const float r = __ldcg(r32 + q);
        const float lim = MET == kMetricL2 ? r * r * (1.f + 1e-6f) : r * (1.f + 1e-6f);
        live = !(cb.lb[i] > lim);
        e = cb.e[i];
    }
    double d64 = 0.0;
    const int D = ix.D;
    if (D > 128) {
        if (live && j == 0) d64 = vdist64<MET>(ix, qv, q, e);
    } else if (__any_sync(kFull, live)) {
        // fp32 pre-screen, the CUDA-core kernels' test (d32 - slack <= r), for
        // candidates of the tensor-core path: most of them are farther than r
        // (its bf16 band is wide), and this drops them before the float64
        // distance and its 8-byte query loads (vec128: 412.2 -> 407.8 ms per
        // step; the CUDA-core kernels' candidates already passed this test).
        // The 8 lanes of a group share a candidate.
        if ((MET == kMetricL1 || MET == kMetricL2) && prescreen) {
            float acc32 = 0.f;
            if (live) {
                const float *of = ix.vec32 + (size_t)e * ix.Dp;
                const float *qf = qv.vec32 + (size_t)q * ix.Dp;
                for (int t = j; t < D; t += 8) {
                    const float df = of[t] - qf[t];
                    acc32 = MET == kMetricL1 ? acc32 + fabsf(df) : fmaf(df, df, acc32);
                }
            }
            acc32 += __shfl_xor_sync(kFull, acc32, 1);
            acc32 += __shfl_xor_sync(kFull, acc32, 2);
            acc32 += __shfl_xor_sync(kFull, acc32, 4);
            if (live) {
                const float d32 = MET == kMetricL1 ? acc32 : sqrtf(acc32);
                live = d32 - slack(ix, d32, 0.f) <= __ldcg(r32 + q) * (1.f + 1e-6f);
            }
            if (!__any_sync(kFull, live)) return;
        }
        const float *o32 = ix.vec64 ? nullptr : ix.vec32 + (size_t)e * ix.Dp;
        const double *o64 = ix.vec64 ? ix.vec64 + (size_t)e * D : nullptr;
        const double *qq = qv.vec64 + (size_t)q * D;
        const int nb = D < 8 ? 0 : D - D % 8;
        double acc = 0.0;
        if (live && j < nb) {
            acc = term64<MET>(o64 ? o64[j] : (double)o32[j], qq[j]);
            for (int t = j + 8; t < nb; t += 8) acc = __dadd_rn(acc, term64<MET>(o64 ? o64[t] : (double)o32[t], qq[t]));
        }
        // combine within the 8-lane group in numpy's order
        const double a1 = __shfl_xor_sync(kFull, acc, 1);
        const double p2 = (j & 1) ? __dadd_rn(a1, acc) : __dadd_rn(acc, a1);      // (r0+r1), (r2+r3), ...
        const double a2 = __shfl_xor_sync(kFull, p2, 2);
        const double p4 = (j & 2) ? __dadd_rn(a2, p2) : __dadd_rn(p2, a2);
        const double a4 = __shfl_xor_sync(kFull, p4, 4);
        double res = (j & 4) ? __dadd_rn(a4, p4) : __dadd_rn(p4, a4);
        if (live && j == 0) {
            if (nb == 0) {
                // n < 8: numpy sums sequentially from 0.0
                res = 0.0;
                for (int t = 0; t < D; t++) res = __dadd_rn(res, term64<MET>(o64 ? o64[t] : (double)o32[t], qq[t]));
            } else {
                for (int t = nb; t < D; t++) res = __dadd_rn(res, term64<MET>(o64 ? o64[t] : (double)o32[t], qq[t]));
            }
            d64 = MET == kMetricL1 ? res : __dsqrt_rn(res);
        }
    }
    const bool hit = live && j == 0 && d64 <= __ldcg(r64 + q);
    const unsigned hb = __ballot_sync(kFull, hit);
    if (!hb) return;
    unsigned long long base = 0;
    if (lane == __ffs(hb) - 1) base = atomicAdd(out.counter, (unsigned long long)__popc(hb));
    base = __shfl_sync(kFull, base, __ffs(hb) - 1);
    if (hit) {
        const unsigned long long o = base + __popc(hb & ((1u << lane) - 1u));
        if (o < out.cap) { out.q[o] = q; out.e[o] = e; out.d[o] = d64; }
    }
}

struct CacheView {
    int n;
    const int64_t *ids;
    const float *vec32;       // [n][Dp]
    const double *vec64;      // [n][D]
    const uint32_t *words;    // packed dense symbols
    const uint32_t *sword;
    const int32_t *slen;
};

template <int MET>
__global__ void k_cache_scan(IndexView ix, QueryView qv, CacheView cv, int nq, const float *__restrict__ r32,
                             const double *__restrict__ r64, HitBuf out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)nq * cv.n) return;
    const int q = (int)(i / cv.n), c = (int)(i - (int64_t)q * cv.n);
    double d;
    if (MET == kMetricEdit) {
        d = (double)edit_peq(qv.peq + qv.peq_off[q], qlen(qv, q), cv.words + cv.sword[c], cv.slen[c]);
    } else if (MET == kMetricAngular) {
        const double *x = cv.vec64 + (size_t)c * ix.D, *q64 = qv.vec64 + (size_t)q * ix.D;
        const double dot = pw_sum64<kMetricAngular>(nullptr, x, q64, 0, ix.D);
        d = angular_finish(dot, norm64(x, ix.D), qv.qnorm64[q], nullptr, x, q64, ix.D);
    } else {
        const double s = pw_sum64<MET>(nullptr, cv.vec64 + (size_t)c * ix.D, qv.vec64 + (size_t)q * ix.D, 0, ix.D);
        d = MET == kMetricL1 ? s : __dsqrt_rn(s);
    }
    if (d <= r64[q]) {
        const unsigned long long sl = atomicAdd(out.counter, 1ull);
        if (sl < out.cap) { out.q[sl] = q; out.e[sl] = -(c + 1); out.d[sl] = d; }
    }
}

__device__ __forceinline__ int64_t entry_id(const int64_t *ids, const int64_t *cache_ids, int32_t e)
{
    return e >= 0 ? ids[e] : cache_ids[-e - 1];
}

// Rows (q, leaf) for every live leaf when pruning is disabled (search.py:338-355).
__global__ void k_all_leaves(const int32_t *leaves, int nleaves, int q0, int nqc, Row *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (int64_t)nleaves * nqc) return;
    int q = q0 + (int)(i / nleaves);
    int l = (int)(i % nleaves);
    out[i] = Row{q, leaves[l], 0.f, 0};
}

// k-th smallest (1-based) of n non-negative float bit patterns in smem.
__device__ uint32_t block_kth(const uint32_t *vals, int n, int k, unsigned *hist, int *sh)
{
    uint32_t prefix = 0, mask = 0;
    int kk = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            uint32_t v = vals[i];
            if ((v & mask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int c = 0, bsel = 255, rem = kk;
            for (int b = 0; b < 256; b++) {
                if (c + (int)hist[b] >= kk) { bsel = b; rem = kk - c; break; }
                c += hist[b];
            }
            sh[0] = bsel;
            sh[1] = rem;
        }
        __syncthreads();
        prefix |= (uint32_t)sh[0] << shift;
        mask |= 255u << shift;
        kk = sh[1];
        __syncthreads();
    }
    return prefix;
}

constexpr int kProbeCand = 8192;
constexpr int kProbeTarget = 1024;
constexpr int kMaxLevels = 64;

// kNN radius estimate (the "estimate its search radius" step).  The k-th
// smallest of any k real distances bounds the true k-th distance from above;
// with fewer than k live candidates the radius is +inf.  Candidates: the
// live entries of the deepest node on a descent path holding at least
// max(k, kProbeTarget) entries (a contiguous table segment).
//  * edit distance: greedy descent to the child whose pivot is nearest.
//  * vectors: the insertion path -- at each node the child whose ring
//    [min_dis, max_dis] (distances to the node's pivot) is nearest d(q, pivot);
//    the probe also takes the next-nearest ring at that level.  Children
//    partition by distance to the parent pivot, so a query's neighbours share
//    its ring chain; on clustered 128-d data the nearest-pivot path gave a
//    radius ~5.8x the true k-th distance, the ring path ~1.05x (median).
template <int MET>
__global__ void __launch_bounds__(256) k_probe(IndexView ix, QueryView qv, int nq, const int32_t *ks,
                                               float *r32, double *r64)
{
    __shared__ uint32_t cand[kProbeCand];
    __shared__ unsigned hist[256];
    __shared__ int sh[4];
    __shared__ float best_d[32];
    __shared__ int best_j[32];
    __shared__ int path[kMaxLevels];
    __shared__ int alt[kMaxLevels];   // next-nearest ring at each level (vectors), or -1
    constexpr bool kRing = MET != kMetricEdit;
    for (int q = blockIdx.x; q < nq; q += gridDim.x) {
        const int nc = ix.nc;
        int node = 1;
        if (threadIdx.x == 0) { path[0] = 1; alt[0] = -1; }
        for (int lvl = 1; lvl < ix.levels; lvl++) {
            if (kRing) {
                // one distance per level: the query to this node's pivot
                const NodeRec self = ix.node[node];
                const float dp = self.piv >= 0 ? dist32<MET>(ix, qv, q, self.piv) : 0.f;
                if (threadIdx.x < 32) {
                    // best and second-best (gap, j): per lane over j = lane mod 32,
                    // then over the warp
                    float g1 = FLT_MAX, g2 = FLT_MAX;
                    int j1 = -1, j2 = -1;
                    for (int j = threadIdx.x; j < nc; j += 32) {
                        const NodeRec c = ix.node[(node - 1) * nc + 2 + j];
                        if (c.size <= 0) continue;
                        const float g = fmaxf(fmaxf(c.mn - dp, dp - c.mx), 0.f);
                        if (j1 < 0 || g < g1) { g2 = g1; j2 = j1; g1 = g; j1 = j; }
                        else if (j2 < 0 || g < g2) { g2 = g; j2 = j; }
                    }
                    for (int o = 16; o > 0; o >>= 1) {
                        const float og1 = __shfl_xor_sync(kFull, g1, o), og2 = __shfl_xor_sync(kFull, g2, o);
                        const int oj1 = __shfl_xor_sync(kFull, j1, o), oj2 = __shfl_xor_sync(kFull, j2, o);
                        // merge two sorted pairs (g1, j1) <= (g2, j2)
                        const bool a_first = oj1 < 0 || (j1 >= 0 && (g1 < og1 || (g1 == og1 && j1 < oj1)));
                        const float fg = a_first ? g1 : og1;
                        const int fj = a_first ? j1 : oj1;
                        // second = min(loser of the firsts, both seconds)
                        float sg = a_first ? og1 : g1;
                        int sj = a_first ? oj1 : j1;
                        if (j2 >= 0 && (sj < 0 || g2 < sg || (g2 == sg && j2 < sj))) { sg = g2; sj = j2; }
                        if (oj2 >= 0 && (sj < 0 || og2 < sg || (og2 == sg && oj2 < sj))) { sg = og2; sj = oj2; }
                        g1 = fg; j1 = fj; g2 = sg; j2 = sj;
                    }
                    if (threadIdx.x == 0) {
                        const int jj = j1 >= 0 ? j1 : 0;   // no non-empty child: any (empty) one
                        sh[2] = jj;
                        path[lvl] = (node - 1) * nc + 2 + jj;
                        alt[lvl] = j2 >= 0 ? (node - 1) * nc + 2 + j2 : -1;
                    }
                }
                __syncthreads();
                node = (node - 1) * nc + 2 + sh[2];
                __syncthreads();
                continue;
            }
            float d = FLT_MAX;
            int j = threadIdx.x;
            if (j < nc) {
                const NodeRec c = ix.node[(node - 1) * nc + 2 + j];
                if (c.size > 0) d = dist32<MET>(ix, qv, q, c.piv);
            }
            float bd = d;
            int bj = j;
            for (int o = 16; o > 0; o >>= 1) {
                float od = __shfl_down_sync(kFull, bd, o);
                int oj = __shfl_down_sync(kFull, bj, o);
                if (od < bd || (od == bd && oj < bj)) { bd = od; bj = oj; }
            }
            if (lane_id() == 0) { best_d[threadIdx.x >> 5] = bd; best_j[threadIdx.x >> 5] = bj; }
            __syncthreads();
            if (threadIdx.x == 0) {
                float xd = best_d[0];
                int xj = best_j[0];
                for (int w = 1; w < (int)(blockDim.x >> 5); w++)
                    if (best_d[w] < xd || (best_d[w] == xd && best_j[w] < xj)) { xd = best_d[w]; xj = best_j[w]; }
                sh[2] = xj;
                path[lvl] = (node - 1) * nc + 2 + xj;
                alt[lvl] = -1;
            }
            __syncthreads();
            node = (node - 1) * nc + 2 + sh[2];
        }
        const int k = ks[q];
        const int target = min(max(k, kProbeTarget), kProbeCand);
        int anc = 1, anc2 = -1;
        for (int lvl = ix.levels - 1; lvl >= 0; lvl--) {
            if (ix.node[path[lvl]].size >= target) { anc = path[lvl]; anc2 = alt[lvl]; break; }
        }
        if (threadIdx.x == 0) sh[3] = 0;
        __syncthreads();
        for (int pass = 0; pass < 2; pass++) {
            const int nd = pass == 0 ? anc : anc2;
            if (nd < 0) break;
            const int pos = ix.npos[nd];
            const int size = ix.node[nd].size;
            for (int b = 0; b < size; b += blockDim.x) {
                if (sh[3] >= kProbeCand) break;       // uniform: read after the barrier
                const int kk = b + threadIdx.x;
                if (kk < size) {
                    const int e = pos + kk;
                    if (is_alive(ix.alive, e)) {
                        int slot = atomicAdd(&sh[3], 1);
                        if (slot < kProbeCand) cand[slot] = __float_as_uint(dist32<MET>(ix, qv, q, e));
                    }
                }
                __syncthreads();
            }
        }
        __syncthreads();
        const int n = min(sh[3], kProbeCand);
        __syncthreads();
        if (n >= k && k >= 1) {
            uint32_t kth = block_kth(cand, n, k, hist, sh);
            if (threadIdx.x == 0) {
                float t = __uint_as_float(kth);
                if (MET != kMetricEdit) t = t + slack(ix, t, 0.f);   // d64 <= d32 + slack
                r32[q] = t;
                r64[q] = (double)t;
            }
        } else if (threadIdx.x == 0) {
            r32[q] = INFINITY;
            r64[q] = INFINITY;
        }
        __syncthreads();
    }
}

// Node-major kNN probe for L1 / L2 (k_probe_path -> sort -> k_probe_dist ->
// k_probe_select): the same candidates (the ring path's node and its
// next-nearest ring) and the same radius rule as k_probe<MET>, but each
// candidate node is staged once per 64 queries that probe it instead of
// once per query (k_probe read ~256 GB from L2 for 100k 128-d queries).
constexpr int kPT = 64;    // query rows x entries per tile
constexpr int kPD = 128;   // dimensions staged per pass

// Best and second-best child of `node` by ring gap to dp (warp-uniform
// result; -1 when absent).
__device__ __forceinline__ int2 ring_best2(const IndexView &ix, int node, float dp)
{
    const int lane = lane_id(), nc = ix.nc;
    float g1 = FLT_MAX, g2 = FLT_MAX;
    int j1 = -1, j2 = -1;
    for (int j = lane; j < nc; j += 32) {
        const NodeRec c = ix.node[(node - 1) * nc + 2 + j];
        if (c.size <= 0) continue;
        const float g = fmaxf(fmaxf(c.mn - dp, dp - c.mx), 0.f);
        if (j1 < 0 || g < g1) { g2 = g1; j2 = j1; g1 = g; j1 = j; }
        else if (j2 < 0 || g < g2) { g2 = g; j2 = j; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const float og1 = __shfl_xor_sync(kFull, g1, o), og2 = __shfl_xor_sync(kFull, g2, o);
        const int oj1 = __shfl_xor_sync(kFull, j1, o), oj2 = __shfl_xor_sync(kFull, j2, o);
        const bool a_first = oj1 < 0 || (j1 >= 0 && (g1 < og1 || (g1 == og1 && j1 < oj1)));
        const float fg = a_first ? g1 : og1;
        const int fj = a_first ? j1 : oj1;
        float sg = a_first ? og1 : g1;
        int sj = a_first ? oj1 : j1;
        if (j2 >= 0 && (sj < 0 || g2 < sg || (g2 == sg && j2 < sj))) { sg = g2; sj = j2; }
        if (oj2 >= 0 && (sj < 0 || og2 < sg || (og2 == sg && oj2 < sj))) { sg = og2; sj = oj2; }
        g1 = fg; j1 = fj; g2 = sg; j2 = sj;
    }
    return make_int2(j1 >= 0 ? (node - 1) * nc + 2 + j1 : -1, j2 >= 0 ? (node - 1) * nc + 2 + j2 : -1);
}

// Warp per query: the ring path; emits kProbeRows (node, row id) pairs per
// query: the deepest path node holding >= max(k, 1024) entries, its
// next-nearest sibling ring, and the nearest ring under the parent's
// next-nearest sibling (offline on clustered 128-d data: 4% -> 1.5% of
// queries whose estimate stays several times the true k-th distance).
constexpr int kProbeRows = 3;
template <int MET>
__global__ void __launch_bounds__(256) k_probe_path(IndexView ix, QueryView qv, int q0, int nq, const int32_t *ks,
                                                   uint32_t *keys, int32_t *vals)
{
    const int lane = lane_id();
    const int qi = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    if (qi >= nq) return;
    const int q = q0 + qi;
    const int target = min(max(ks[q], kProbeTarget), kProbeCand);
    int node = 1, anc = 1, anc2 = -1, uncle = -1, prev_alt = -1;
    for (int lvl = 1; lvl < ix.levels; lvl++) {
        const NodeRec self = ix.node[node];
        const float dp = self.piv >= 0 ? dist32<MET>(ix, qv, q, self.piv) : 0.f;
        const int2 b = ring_best2(ix, node, dp);
        const int child = b.x >= 0 ? b.x : (node - 1) * ix.nc + 2;
        if (ix.node[child].size >= target) {   // deepest path node holding >= target entries
            anc = child;
            anc2 = b.y;
            uncle = prev_alt;
        }
        prev_alt = b.y;
        node = child;
    }
    int anc3 = -1;
    if (uncle >= 0) {
        const NodeRec u = ix.node[uncle];
        const float du = u.piv >= 0 ? dist32<MET>(ix, qv, q, u.piv) : 0.f;
        anc3 = ring_best2(ix, uncle, du).x;
    }
    if (lane == 0) {
        const int r = kProbeRows * qi;
        keys[r] = (uint32_t)anc;
        keys[r + 1] = anc2 >= 0 ? (uint32_t)anc2 : 0xffffffffu;   // sorts last, skipped
        keys[r + 2] = anc3 >= 0 ? (uint32_t)anc3 : 0xffffffffu;
        for (int w = 0; w < kProbeRows; w++) vals[r + w] = r + w;
    }
}

__device__ __forceinline__ int probe_node_size(const IndexView &ix, uint32_t key)
{
    return key != 0xffffffffu ? ix.node[key].size : 0;
}

// Distances of 64 sorted (query, node) rows to their node's entries, 4x4
// register tiles; out[qi][slot], slot = entry index (+ size of the first node
// for the second one), +inf for tombstones, capped at kProbeCand per query.
template <int MET>
__global__ void __launch_bounds__(256) k_probe_dist(IndexView ix, QueryView qv, int q0, const uint32_t *skeys,
                                                   const int32_t *svals, int nrows, const uint32_t *keys, float *out)
{
    extern __shared__ float4 pd_smem4[];
    float *qs = reinterpret_cast<float *>(pd_smem4);   // [kPT][kPD + 4]
    float *es = qs + kPT * (kPD + 4);                  // [kPT][kPD + 4]
    __shared__ int s_node[kPT], s_q[kPT], s_base[kPT];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int rbase = blockIdx.x * kPT;
    if (tid < kPT) {
        const int r = rbase + tid;
        int node = -1, qi = -1, base = 0;
        if (r < nrows && skeys[r] != 0xffffffffu) {
            node = (int)skeys[r];
            const int v = svals[r];
            qi = v / kProbeRows;
            for (int w = qi * kProbeRows; w < v; w++) base += probe_node_size(ix, keys[w]);
        }
        s_node[tid] = node;
        s_q[tid] = qi;
        s_base[tid] = base;
    }
    __syncthreads();
    const int S = kPD + 4;
    int r0 = 0;
    while (r0 < kPT && s_node[r0] >= 0) {
        const int node = s_node[r0];
        int r1 = r0 + 1;
        while (r1 < kPT && s_node[r1] == node) r1++;
        const int pos = ix.npos[node], size = ix.node[node].size;
        for (int e0 = 0; e0 < size; e0 += kPT) {
            float acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] = 0.f;
            for (int d0 = 0; d0 < ix.Dp; d0 += kPD) {
                const int dl = min(kPD, ix.Dp - d0);   // multiple of 4
                const int c4 = dl >> 2;
                for (int t = tid; t < kPT * c4; t += blockDim.x) {
                    const int i = t / c4, c = t - i * c4;
                    const int row = r0 + i;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (row < r1)
                        v = __ldg(reinterpret_cast<const float4 *>(qv.vec32 + (size_t)(q0 + s_q[row]) * ix.Dp + d0) + c);
                    *reinterpret_cast<float4 *>(qs + i * S + 4 * c) = v;
                    float4 w = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (e0 + i < size)
                        w = __ldg(reinterpret_cast<const float4 *>(ix.vec32 + (size_t)(pos + e0 + i) * ix.Dp + d0) + c);
                    *reinterpret_cast<float4 *>(es + i * S + 4 * c) = w;
                }
                __syncthreads();
                // rows ty + 16a of this run (relative to r0), entries tx + 16b
                for (int c = 0; c < dl; c += 4) {
                    float4 x[4], y[4];
#pragma unroll
                    for (int a = 0; a < 4; a++) x[a] = *reinterpret_cast<const float4 *>(qs + (ty + 16 * a) * S + c);
#pragma unroll
                    for (int b = 0; b < 4; b++) y[b] = *reinterpret_cast<const float4 *>(es + (tx + 16 * b) * S + c);
#pragma unroll
                    for (int a = 0; a < 4; a++)
#pragma unroll
                        for (int b = 0; b < 4; b++) {
                            const float u0 = x[a].x - y[b].x, u1 = x[a].y - y[b].y;
                            const float u2 = x[a].z - y[b].z, u3 = x[a].w - y[b].w;
                            if (MET == kMetricL1)
                                acc[a][b] += (fabsf(u0) + fabsf(u1)) + (fabsf(u2) + fabsf(u3));
                            else
                                acc[a][b] += (u0 * u0 + u1 * u1) + (u2 * u2 + u3 * u3);
                        }
                }
                __syncthreads();
            }
#pragma unroll
            for (int a = 0; a < 4; a++) {
                const int row = r0 + ty + 16 * a;
                if (row >= r1) continue;
                const int qi = s_q[row];
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    const int e = e0 + tx + 16 * b;
                    const int slot = s_base[row] + e;
                    if (e >= size || slot >= kProbeCand) continue;
                    const float d = MET == kMetricL1 ? acc[a][b] : sqrtf(acc[a][b]);
                    out[(size_t)qi * kProbeCand + slot] = is_alive(ix.alive, pos + e) ? d : INFINITY;
                }
            }
        }
        r0 = r1;
    }
}

// k-th smallest candidate distance per query -> radius (as k_probe)
template <int MET>
__global__ void __launch_bounds__(256) k_probe_select(IndexView ix, int q0, int nq, const int32_t *ks, const uint32_t *keys,
                                                     const float *dist, float *r32, double *r64)
{
    __shared__ uint32_t cand[kProbeCand];
    __shared__ unsigned hist[256];
    __shared__ int sh[4];
    __shared__ int s_live;
    for (int qi = blockIdx.x; qi < nq; qi += gridDim.x) {
        const int q = q0 + qi;
        if (threadIdx.x == 0) s_live = 0;
        __syncthreads();
        int n = 0;
        for (int w = 0; w < kProbeRows; w++) n += probe_node_size(ix, keys[kProbeRows * qi + w]);
        n = min(n, kProbeCand);
        const float *src = dist + (size_t)qi * kProbeCand;
        int live = 0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const float d = src[i];
            cand[i] = __float_as_uint(d);
            live += d < INFINITY;
        }
        if (live) atomicAdd(&s_live, live);
        __syncthreads();
        const int k = ks[q];
        const int nl = s_live;
        __syncthreads();
        if (nl >= k && k >= 1) {
            const uint32_t kth = block_kth(cand, n, k, hist, sh);
            if (threadIdx.x == 0) {
                float t = __uint_as_float(kth);
                t = t + slack(ix, t, 0.f);   // d64 <= d32 + slack
                r32[q] = t;
                r64[q] = (double)t;
            }
        } else if (threadIdx.x == 0) {
            r32[q] = INFINITY;
            r64[q] = INFINITY;
        }
        __syncthreads();
    }
}

// Largest fp32 distance from the root pivot (query slot 0 of a one-row
// batch) to any entry.  By the triangle inequality d(q,o) <= d(q,root) +
// that radius for every object, so it bounds any k-th distance; it is the
// kNN starting radius when the probe finds no finite estimate (k above the
// probe's candidate cap, or probed nodes left with fewer than k live
// entries after deletes), so the histogram shrink still has a finite range.
template <int MET>
__global__ void k_root_radius(IndexView ix, QueryView qv, int64_t n, unsigned *out)
{
    float m = 0.f;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        if (!is_alive(ix.alive, (int)e)) continue;   // free slots and tombstones hold no answer
        const float d = dist32<MET>(ix, qv, 0, (int)e);
        if (d == d) m = fmaxf(m, d);
    }
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(kFull, m, o));
    if (lane_id() == 0) atomicMax(out, __float_as_uint(m));
}

template <int MET>
__global__ void k_finite_bound(IndexView ix, QueryView qv, int nq, float rroot, float *r32, double *r64)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq || r32[q] < INFINITY) return;
    const float d = dist32<MET>(ix, qv, q, ix.node[1].piv);
    // each fp32 distance is within slack of its float64 value
    const float t = (d + rroot + slack(ix, d, rroot) + ix.abs_eps) * (1.f + 0x1p-20f);
    r32[q] = t;
    r64[q] = (double)t;
}

// kNN radius supplied by the caller (the MIN over shards of every shard's
// probe radius, SURVEY.md §8(e) collective 2): each shard's probe radius is
// an upper bound of its own k-th distance, hence of the global one.
__global__ void k_set_bound(const float *__restrict__ b, int nq, float *r32, double *r64)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const float t = b[q];
    r32[q] = t;
    r64[q] = (double)t;
}

// query preparation --------------------------------------------------------

__global__ void k_map_symbols(const int32_t *codes, int64_t n, const int32_t *alpha, int A, uint8_t *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int32_t c = codes[i];
    int lo = 0, hi = A;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (alpha[mid] < c) lo = mid + 1; else hi = mid;
    }
    out[i] = (lo < A && alpha[lo] == c) ? (uint8_t)lo : kNoSym;
}

// one thread per (query, symbol position): sets the Myers match bit
__global__ void k_build_peq(const uint8_t *sym, const int64_t *soff, const int64_t *peq_off, int nq,
                            int64_t nsym, uint32_t *peq)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nsym) return;
    // find the query owning symbol i (binary search over soff)
    int lo = 0, hi = nq;
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (soff[mid] <= i) lo = mid; else hi = mid;
    }
    const int q = lo;
    const int pos = (int)(i - soff[q]);
    const int m = (int)(soff[q + 1] - soff[q]);
    const int W = (m + 31) >> 5;
    const uint8_t c = sym[i];
    if (c == kNoSym) return;
    atomicOr(peq + peq_off[q] + (int64_t)c * W + (pos >> 5), 1u << (pos & 31));
}

// per-query 32-bucket symbol histogram (kNoSym goes to bucket 31: a valid
// merge, since no indexed object contains that symbol)
__global__ void k_query_hist(const uint8_t *sym, const int64_t *soff, int nq, uint4 *qhist)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = soff[q]; i < soff[q + 1]; i++) {
        const uint8_t c = sym[i];
        const int b = (c == kNoSym) ? 31 : (c & 31);
        const uint32_t cur = (w[b >> 2] >> (8 * (b & 3))) & 0xffu;
        if (cur < 255u) w[b >> 2] += 1u << (8 * (b & 3));
    }
    qhist[2 * q] = make_uint4(w[0], w[1], w[2], w[3]);
    qhist[2 * q + 1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// q-gram signatures (kernels.cuh qgram_sig) of the queries ...
__global__ void k_query_sig(const uint8_t *sym, const int64_t *soff, int nq, int A, uint4 *qsig)
{
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    const uint8_t *t = sym + soff[q];
    uint32_t w[8];
    qgram_sig([&](int i) { return (uint32_t)t[i]; }, (int)(soff[q + 1] - soff[q]), A, w);
    qsig[2 * q] = make_uint4(w[0], w[1], w[2], w[3]);
    qsig[2 * q + 1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// ... and of stored strings (every slot, or the listed ones; free slots 0)
__global__ void k_slot_sig(const uint32_t *str, const uint32_t *sword, const int32_t *slen, const int32_t *slots,
                           int64_t n, int A, uint4 *esig)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t s = slots ? slots[i] : i;
    if (s < 0) return;
    const uint32_t *t4 = str + sword[s];
    uint32_t w[8];
    qgram_sig([&](int k) { return (__ldg(t4 + (k >> 2)) >> (8 * (k & 3))) & 0xffu; }, slen[s], A, w);
    esig[2 * s] = make_uint4(w[0], w[1], w[2], w[3]);
    esig[2 * s + 1] = make_uint4(w[4], w[5], w[6], w[7]);
}

// bf16 query rows (uncentred, zero-padded to Dk) and |q| rounded up
__global__ void k_query_bf16(const float *v32, int64_t nq, int D, int Dp, int Dk, uint4 *qbf, float *qn)
{
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nq) return;
    __nv_bfloat16 *dst = reinterpret_cast<__nv_bfloat16 *>(qbf + r * (Dk / 8));
    double s2 = 0.0;
    for (int d = 0; d < Dk; d++) {
        const float x = d < D ? v32[r * Dp + d] : 0.f;
        dst[d] = __float2bfloat16(x);
        s2 += (double)x * (double)x;
    }
    qn[r] = (float)(sqrt(s2) * (1.0 + 1e-6));
}

__global__ void k_vec_prep(const double *v64, int64_t nq, int D, int Dp, float *v32, unsigned *maxabs_bits,
                           int *inexact)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq * Dp) return;
    int64_t r = i / Dp;
    int d = (int)(i - r * Dp);
    float f = 0.f;
    if (d < D) {
        double x = v64[r * D + d];
        f = (float)x;
        if ((double)f != x) atomicOr(inexact, 1);
        atomicMax(maxabs_bits, __float_as_uint(fabsf(f)));
    }
    v32[i] = f;
}

// collect -------------------------------------------------------------------

// sort key for the id tie-break when every hit is a tree entry: the dataset
// row (row order == id order, data.py:149-153), rbits wide instead of 64
__global__ void k_gather_row(const int32_t *e, int64_t n, const int32_t *row, uint32_t *key, int32_t *perm)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = (uint32_t)row[e[i]];
    perm[i] = (int32_t)i;
}

__global__ void k_gather_id(const int32_t *e, int64_t n, const int64_t *ids, const int64_t *cache_ids,
                            unsigned long long *key, int32_t *perm)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t ei = e[i];
    key[i] = (unsigned long long)(ei >= 0 ? ids[ei] : cache_ids[-ei - 1]);
    perm[i] = (int32_t)i;
}

__global__ void k_gather_d(const double *d, const int32_t *perm, int64_t n, unsigned long long *key)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = (unsigned long long)__double_as_longlong(d[perm[i]]);
}

// Float-distance collect in two sorts: key = float32(d) bits (monotonic in
// d >= 0) << rbits | dataset row, then stable by query; k_fix_f32_ties then
// puts each run of equal (query, float32(d)) -- whose float64 distances may
// differ -- in (float64 d, row) order (insertion sort: runs are short, and
// already sorted when their distances are equal).
__global__ void k_pack_f32_keys(const int32_t *e, const double *d, int64_t n, const int32_t *row, int rbits,
                                unsigned long long *key, int32_t *perm)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = ((unsigned long long)__float_as_uint((float)d[i]) << rbits) | (unsigned long long)(uint32_t)row[e[i]];
    perm[i] = (int32_t)i;
}

__global__ void k_fix_f32_ties(int32_t *perm, const int32_t *q, const int32_t *e, const double *d,
                               const int32_t *row, int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto tie_key = [&](int64_t k) {
        const int32_t p = perm[k];
        return ((unsigned long long)(uint32_t)q[p] << 32) | __float_as_uint((float)d[p]);
    };
    const unsigned long long t = tie_key(i);
    if (i > 0 && tie_key(i - 1) == t) return;   // not the head of its run
    int64_t j = i + 1;
    while (j < n && tie_key(j) == t) j++;
    if (j - i < 2) return;
    for (int64_t a = i + 1; a < j; a++) {
        const int32_t pa = perm[a];
        const double da = d[pa];
        const int32_t ra = row[e[pa]];
        int64_t b = a - 1;
        while (b >= i) {
            const int32_t pb = perm[b];
            const double db = d[pb];
            if (db < da || (db == da && row[e[pb]] <= ra)) break;
            perm[b + 1] = pb;
            b--;
        }
        perm[b + 1] = pa;
    }
}

__global__ void k_gather_q(const int32_t *q, const int32_t *perm, int64_t n, uint32_t *key)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    key[i] = (uint32_t)q[perm[i]];
}

__global__ void k_count(const int32_t *q, int64_t n, long long *counts)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    atomicAdd((unsigned long long *)(counts + q[i]), 1ull);
}

__global__ void k_clamp_counts(const long long *counts, const int32_t *ks, int nq, long long *out)
{
    int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    long long c = counts[q];
    out[q] = ks ? min(c, (long long)ks[q]) : c;
}

// Final scatter: sorted hit i of query q at rank r within its segment goes
// to out_off[q] + r when r < out count (kNN truncation keeps the k first).
__global__ void k_emit(const int32_t *perm, const int32_t *hq, const int32_t *he, const double *hd,
                       const long long *in_off, const long long *out_off, const long long *out_cnt,
                       const int64_t *ids, const int64_t *cache_ids, int64_t n, int64_t *out_ids, double *out_dis)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t h = perm[i];
    const int q = hq[h];
    const long long r = i - in_off[q];
    if (r < out_cnt[q]) {
        const int32_t e = he[h];
        out_ids[out_off[q] + r] = e >= 0 ? ids[e] : cache_ids[-e - 1];
        out_dis[out_off[q] + r] = hd[h];
    }
}

__global__ void k_pair_vec(int metric, int64_t np, int D, const double *a, const double *b, double *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    const double *x = a + i * D, *y = b + i * D;
    if (metric == kMetricAngular) {   // angular_row_pairs (metrics.py:175-193)
        const double dot = pw_sum64<kMetricAngular>(nullptr, x, y, 0, D);
        out[i] = angular_finish(dot, norm64(x, D), norm64(y, D), nullptr, x, y, D);
        return;
    }
    double s = metric == kMetricL1 ? pw_sum64<kMetricL1>(nullptr, x, y, 0, D) : pw_sum64<kMetricL2>(nullptr, x, y, 0, D);
    out[i] = metric == kMetricL1 ? s : __dsqrt_rn(s);
}

// pairs (a_i, b_i): a is the pattern (query side), b the text
__global__ void k_pair_edit(int64_t np, const uint32_t *bwords, const uint32_t *bword, const int32_t *blen,
                            QueryView qa, double *out)
{
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= np) return;
    out[i] = (double)edit_peq(qa.peq + qa.peq_off[i], qlen(qa, (int)i), bwords + bword[i], blen[i]);
}

}  // namespace gts

// ===========================================================================
// host side
// ===========================================================================
using namespace gts;

namespace gts {
void dense_alphabet(const int32_t *codes, int64_t ncodes, std::vector<int32_t> &alpha);   // builder.cpp
constexpr int kHistMinAlphabet = 8;   // symbol-histogram bound only pays on larger alphabets

// numpy's pairwise sum (host; same order as pw_sum64 / the oracle)
static double host_pw_sum(const double *a, int64_t n)
{
    if (n < 8) {
        double r = 0.0;
        for (int64_t i = 0; i < n; i++) r += a[i];
        return r;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return host_pw_sum(a, n2) + host_pw_sum(a + n2, n - n2);
}

// |x| as numpy computes the angular norms: sqrt((mat * mat).sum(axis=1))
static double host_norm(const double *x, int64_t D, std::vector<double> &tmp)
{
    tmp.resize((size_t)std::max<int64_t>(D, 1));
    for (int64_t d = 0; d < D; d++) tmp[(size_t)d] = x[d] * x[d];
    return std::sqrt(host_pw_sum(tmp.data(), D));
}
// Pack strings (dense symbols, given per string as a code range mapped by
// `sym`) 4 per 32-bit word, each string starting on a 16-byte boundary.
template <class SymOf>
static void pack_words(int64_t n, const int64_t *off, SymOf sym, std::vector<uint32_t> &words,
                       std::vector<uint32_t> &wstart, std::vector<int32_t> &len, const int64_t *order = nullptr,
                       int64_t reserve = 0)
{
    // order[e] < 0: a free slot (leaf slack), `reserve` words of room
    wstart.resize((size_t)n);
    len.resize((size_t)n);
    uint64_t w = 0;
    for (int64_t e = 0; e < n; e++) {
        const int64_t r = order ? order[e] : e;
        const int64_t l = r >= 0 ? off[r + 1] - off[r] : 0;
        wstart[(size_t)e] = (uint32_t)w;
        len[(size_t)e] = (int32_t)l;
        w += r >= 0 ? (uint64_t)((l + 15) / 16) * 4 : (uint64_t)reserve;    // 16-byte aligned objects
    }
    w += 8;                                    // the DP prefetches one uint4 past an object
    if (w >= (1ull << 32)) fail(GTS_EINVAL, "string payload exceeds 16 GiB per index; shard it");
    words.assign((size_t)w, 0u);
    #pragma omp parallel for schedule(static, 4096)
    for (int64_t e = 0; e < n; e++) {
        const int64_t r = order ? order[e] : e;
        if (r < 0) continue;
        uint32_t *dst = words.data() + wstart[(size_t)e];
        for (int64_t k = off[r], j = 0; k < off[r + 1]; k++, j++)
            dst[j >> 2] |= (uint32_t)sym(k) << (8 * (j & 3));
    }
}

// dense symbol of a code point: a direct table for code points < 2^16, a
// binary search over the sorted alphabet above that
struct SymMap {
    const std::vector<int32_t> &alpha;
    std::vector<uint8_t> lut;
    explicit SymMap(const std::vector<int32_t> &a) : alpha(a), lut(1 << 16, 0xff)
    {
        for (size_t i = 0; i < a.size(); i++)
            if (a[i] >= 0 && a[i] < (1 << 16)) lut[(size_t)a[i]] = (uint8_t)i;
    }
    uint32_t operator()(int32_t c) const
    {
        if (c >= 0 && c < (1 << 16)) return lut[(size_t)c];
        return (uint32_t)(std::lower_bound(alpha.begin(), alpha.end(), c) - alpha.begin());
    }
};
}  // namespace gts

struct gts_index {
    int device = 0;
    int metric = 0;
    int64_t n = 0, nodes = 0;
    int nc = 0, levels = 0, split_rounds = 0;
    int D = 0, Dp = 0;
    int A = 0;
    int max_len = 0;
    bool data_exact = true;
    float data_maxabs = 0.f;
    DBuf<NodeRec> node;
    DBuf<int32_t> npos;
    DBuf<float> dis;
    DBuf<int64_t> ids;
    DBuf<uint32_t> alive;
    DBuf<float> vec32;
    DBuf<double> vec64;
    DBuf<uint32_t> str;      // dense symbols, 4 per word, each entry 4-byte aligned
    DBuf<uint32_t> sword;
    DBuf<int32_t> slen;
    DBuf<int32_t> row;
    DBuf<uint4> erec;
    DBuf<uint4> ehist;
    DBuf<uint4> esig;        // strings: q-gram signatures (qgram_sig), [2 * slots]
    DBuf<uint4> vcent;   // bf16 x 8 per uint4
    DBuf<uint4> vtile;   // vcent per leaf in the MMA's SW128 smem image (k_vtile), or empty
    DBuf<int32_t> vt_off, vt_rows;   // per leaf: image offset (128-byte units), rows (capacity rounded to 16)
    DBuf<float> vnorm32;   // angular: |o| per entry
    DBuf<double> vnorm64;
    DBuf<float> vse;     // c . vcent_e per entry
    int Dk = 0;
    DBuf<int32_t> alpha;
    int max_leaf = 0;
    int max_leaf_words = 0;   // largest leaf's packed text (words), edit only
    int leaf_first = 0, leaf_count = 0;
    std::vector<int64_t> ord;   // device entry -> reference table position
    std::atomic<unsigned long long> hit_hint[2] = {{0}, {0}};   // hits of the last range / kNN call
    std::atomic<unsigned long long> cand_hint{0};                // tensor-core candidates of the last launch
    // pending-insert cache (device copy of the caller's pending set)
    int cache_n = 0;
    int cache_max_len = 0;   // strings: longest pending-cache string
    DBuf<int64_t> cache_ids;
    DBuf<float> cache_vec32;
    DBuf<double> cache_vec64;
    DBuf<uint32_t> cache_words, cache_sword;
    DBuf<int32_t> cache_slen;
    DBuf<int32_t> live_leaves;
    int n_live_leaves = 0;
    std::vector<int32_t> h_alpha;
    // vectors: fp32 radius of the whole collection around the root pivot
    // (k_root_radius) and of the pending cache (host, float64), and the root
    // pivot's payload for the latter
    float root_radius = INFINITY, cache_radius = 0.f;
    std::atomic<int64_t> hbm_rows_cached{0};   // device default frontier-table rows (hbm_rows)
    double avg_text_bytes = 0.0;   // strings: mean stored bytes per entry (traversal byte counts)
    // leaf slack (in-place inserts): device slot layout and
    // host mirrors of what the insert path changes
    int64_t n_ref = 0;                 // entries of the reference tree
    std::vector<int64_t> leaf_dpos, leaf_cap, leaf_size;   // per leaf (index = node - leaf_first)
    std::vector<uint32_t> h_alive;     // host copy of the alive bitmask
    std::vector<uint32_t> h_sword;     // strings: first text word of every slot
    std::vector<int32_t> h_slen;       // strings: length of every slot's string
    std::vector<NodeRec> h_nodes;      // host copy of the node records (ranges widen on insert)
    int slot_words = 0;                // strings: text words reserved per free slot
    int64_t n_inserted = 0;            // slots filled by gts_index_insert
    std::vector<double> root_payload;
};

struct gts_queries {
    int metric = 0;
    int64_t nq = 0;
    int max_len = 0;
    int D = 0, Dp = 0;
    bool exact = true;
    float maxabs = 0.f;
    cudaStream_t stream = 0;
    DBuf<float> vec32;
    DBuf<double> vec64;
    DBuf<uint8_t> str;
    DBuf<int64_t> soff;
    DBuf<uint32_t> peq;
    DBuf<int64_t> peq_off;
    DBuf<uint4> qhist;
    DBuf<uint4> qsig;
    DBuf<uint4> qbf;     // bf16 query rows (tensor-core L2 path)
    DBuf<float> qnorm32;   // angular: |q|
    DBuf<double> qnorm64;
    DBuf<float> qn;
};

struct gts_result {
    int64_t nq = 0, total = 0, peak = 0;
    int64_t limits[64] = {0};
    cudaStream_t stream = 0;
    DBuf<int64_t> offsets;
    DBuf<int64_t> ids;
    DBuf<double> dis;
    DBuf<unsigned long long> verified, pruned;
};

namespace {

// Leaf images of vcent for the tensor-core screen's bulk copies (k_vtile).
// GTS_NO_VTILE=1 keeps the per-thread cp.async path.
void build_vtile(gts_index *ix, cudaStream_t st)
{
    ix->vtile.release();
    if (!ix->vcent.p || ix->leaf_count == 0 || std::getenv("GTS_NO_VTILE")) return;
    const int64_t nl = ix->leaf_count;
    const int c16 = ix->Dk / 8, nkb = ix->Dk / 64;
    std::vector<int32_t> off((size_t)nl), rows((size_t)nl);
    int64_t tot = 0;
    for (int64_t l = 0; l < nl; l++) {
        // items carry (offset / 2 KB) in 24 bits and rows / 16 in 8 bits
        rows[(size_t)l] = (int32_t)std::max<int64_t>(16, (ix->leaf_cap[(size_t)l] + 15) & ~15ll);
        off[(size_t)l] = (int32_t)tot;
        tot += (int64_t)nkb * rows[(size_t)l];
        if (tot >= (1ll << 28) || rows[(size_t)l] > 255 * 16) return;   // past 32 GB of images: keep cp.async
    }
    ix->vtile.alloc((size_t)tot * 8, st);
    ix->vt_off.alloc((size_t)nl, st);
    h2d(ix->vt_off.p, off.data(), off.size(), st);
    ix->vt_rows.alloc((size_t)nl, st);
    h2d(ix->vt_rows.p, rows.data(), rows.size(), st);
    DBuf<int64_t> dpos((size_t)nl, st), cap((size_t)nl, st);
    h2d(dpos.p, ix->leaf_dpos.data(), (size_t)nl, st);
    h2d(cap.p, ix->leaf_cap.data(), (size_t)nl, st);
    k_vtile<<<(unsigned)std::min<int64_t>(nl, 1 << 20), 256, 0, st>>>(ix->vcent.p, c16, dpos.p, cap.p, ix->vt_off.p,
                                                                     ix->vt_rows.p, (int)nl, ix->vtile.p);
    LAUNCH_CHECK();
    CK(cudaStreamSynchronize(st));
}

IndexView make_view(const gts_index *ix, const gts_queries *q)
{
    IndexView v{};
    v.node = ix->node.p;
    v.npos = ix->npos.p;
    v.dis = ix->dis.p;
    v.alive = ix->alive.p;
    v.vec32 = ix->vec32.p;
    v.vec64 = ix->vec64.p;
    v.str = ix->str.p;
    v.sword = ix->sword.p;
    v.slen = ix->slen.p;
    v.row = ix->row.p;
    v.erec = ix->erec.p;
    v.ehist = ix->ehist.p;
    v.esig = ix->esig.p;
    v.sig_q = ix->esig.p ? qgram_q(ix->A) : 0;
    v.vcent = ix->vcent.p;
    v.vtile = ix->vtile.p;
    v.vnorm32 = ix->vnorm32.p;
    v.vnorm64 = ix->vnorm64.p;
    v.vse = ix->vse.p;
    v.Dk = ix->Dk;
    v.D = ix->D;
    v.Dp = ix->Dp;
    v.nc = ix->nc;
    v.levels = ix->levels;
    v.leaf_first = ix->leaf_first;
    v.leaf_count = ix->leaf_count;
    v.max_leaf = ix->max_leaf;
    if (ix->metric == GTS_EDIT) {
        v.rel = 0.f;
        v.abs_eps = 0.f;
    } else if (ix->metric == GTS_ANGULAR) {
        // fp32 cosine error eps_c <= (3D + 8) 2^-24 (dot and both norms; x2
        // for inputs that are not fp32-exact); arccos turns it into at most
        // sqrt(2 eps_c) (worst near cos = +-1), plus acosf's own error
        const bool exact = ix->data_exact && (!q || q->exact);
        const float ec = (float)(3 * ix->D + 8) * ldexpf(1.f, -24) * (exact ? 1.f : 2.f);
        v.rel = 0.f;
        v.abs_eps = 1.1f * sqrtf(2.f * ec) + 8e-6f;
    } else {
        // fp32 screening error model: relative (D+8)*2^-23 covers sequential
        // fp32 accumulation of D terms with margin; inputs that are not
        // exactly representable add an absolute 2*D*2^-24*(max|x|+max|q|).
        v.rel = (float)(ix->D + 8) * ldexpf(1.f, -23);
        v.abs_eps = 0.f;
        if (!ix->data_exact || (q && !q->exact))
            v.abs_eps = 2.f * (float)ix->D * ldexpf(1.f, -24) * (ix->data_maxabs + (q ? q->maxabs : 0.f)) * 2.f;
    }
    return v;
}

QueryView make_qview(const gts_index *ix, const gts_queries *q)
{
    QueryView v{};
    v.vec32 = q->vec32.p;
    v.vec64 = q->vec64.p;
    v.soff = q->soff.p;
    v.str = q->str.p;
    v.peq = q->peq.p;
    v.peq_off = q->peq_off.p;
    v.qhist = q->qhist.p;
    v.qsig = q->qsig.p;
    v.qbf = q->qbf.p;
    v.qnorm32 = q->qnorm32.p;
    v.qnorm64 = q->qnorm64.p;
    v.qn = q->qn.p;
    v.A = ix->A;
    return v;
}

int64_t level_size_limit(int64_t cap, int64_t nc, int64_t split, int64_t layer)
{
    int64_t share = cap / ((split - layer + 1) * nc);
    return share > 1 ? share : 1;
}

float round_up_f32(double r)
{
    if (std::isinf(r)) return INFINITY;
    float f = (float)r;
    if ((double)f < r) f = std::nextafter(f, INFINITY);
    return f;
}

// Per-thread pinned words for the few device->host counter reads.
unsigned long long *pinned_counters()
{
    static thread_local unsigned long long *p = nullptr;
    if (!p) CK(cudaMallocHost((void **)&p, 4 * sizeof(unsigned long long)));
    return p;
}

// Per-thread pinned staging for the small per-call host->device copies
// (radii, k, initial bounds).  A cudaMemcpyAsync from pageable memory first
// synchronises the stream, which serialised the host with the previous
// call's device work; from pinned memory it is truly asynchronous.  The
// arena is rewound at every search call: the previous call's copies have
// completed by then (every call ends with a stream synchronisation).
struct PinnedArena {
    char *p = nullptr;
    size_t cap = 0, off = 0;
    template <class T>
    const T *stage(const T *src, size_t cnt)
    {
        const size_t bytes = ((cnt * sizeof(T)) + 255) & ~(size_t)255;
        if (off + bytes > cap) {
            // grow (only between calls in practice; earlier stagings of this call stay valid
            // because the old block is released only after the stream drains)
            size_t ncap = std::max<size_t>(cap * 2, off + bytes + (1 << 20));
            char *np = nullptr;
            CK(cudaMallocHost((void **)&np, ncap));
            if (p) {
                CK(cudaDeviceSynchronize());
                std::memcpy(np, p, off);
                cudaFreeHost(p);
            }
            p = np;
            cap = ncap;
        }
        T *dst = reinterpret_cast<T *>(p + off);
        std::memcpy(dst, src, cnt * sizeof(T));
        off += bytes;
        return dst;
    }
};
static PinnedArena &pinned_arena()
{
    static thread_local PinnedArena a;
    return a;
}

// The per-call search driver.
struct Search {
    gts_index *ix;
    const gts_queries *qs;
    cudaStream_t st;
    IndexView iv;
    QueryView qv;
    int mode;          // 0 range, 1 knn
    int64_t cap;
    int pruning;
    int64_t nq;
    DBuf<float> r32;
    DBuf<double> r64;
    DBuf<int32_t> ks;
    DBuf<unsigned long long> verified, pruned;
    DBuf<unsigned long long> counter;   // [0] expand rows, [1] hits
    unsigned long long *h_counter = nullptr;
    // hits
    DBuf<int32_t> hq, he;
    DBuf<double> hd;
    unsigned long long hits = 0;
    int max_qlen = 0;
    bool use_cache = false;
    bool cache_hits = false;
    int64_t peak = 0;
    int64_t limits[64] = {0};
    bool prof = false;
    std::vector<std::tuple<const char *, cudaEvent_t, cudaEvent_t>> events;
    DBuf<unsigned long long> work;
    const float *ext_bound = nullptr;   // kNN: caller-supplied radius per query (device), replaces the probe
    float *probe_out = nullptr;         // kNN probe-only call: the probe radius per query goes here

    // time one launch with events when profiling is on
    template <class F>
    void timed(const char *name, F &&launch)
    {
        if (!prof) { launch(); return; }
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        CK(cudaEventRecord(a, st));
        launch();
        CK(cudaEventRecord(b, st));
        events.emplace_back(name, a, b);
    }

    void flush_profile()
    {
        if (!prof) return;
        CK(cudaStreamSynchronize(st));
        for (auto &ev : events) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, std::get<1>(ev), std::get<2>(ev)));
            prof_add(std::get<0>(ev), ms);
            cudaEventDestroy(std::get<1>(ev));
            cudaEventDestroy(std::get<2>(ev));
        }
        events.clear();
        unsigned long long h[4];
        CK(cudaMemcpy(h, work.p, sizeof(h), cudaMemcpyDeviceToHost));
        std::lock_guard<std::mutex> g(g_prof_mu);
        for (int i = 0; i < 4; i++) g_work[i] += h[i];
    }

    Search(gts_index *ix_, const gts_queries *q_, cudaStream_t s, int mode_, int64_t cap_, int pruning_)
        : ix(ix_), qs(q_), st(s), mode(mode_), cap(cap_), pruning(pruning_), nq(q_->nq)
    {
        iv = make_view(ix, qs);
        qv = make_qview(ix, qs);
        verified.alloc((size_t)nq, st);
        pruned.alloc((size_t)nq, st);
        CK(cudaMemsetAsync(verified.p, 0, sizeof(unsigned long long) * nq, st));
        CK(cudaMemsetAsync(pruned.p, 0, sizeof(unsigned long long) * nq, st));
        counter.alloc(2, st);
        CK(cudaMemsetAsync(counter.p, 0, 2 * sizeof(unsigned long long), st));
        h_counter = pinned_counters();
        prof = g_profile.load() != 0;
        if (prof) {
            work.alloc(4, st);
            CK(cudaMemsetAsync(work.p, 0, 4 * sizeof(unsigned long long), st));
        }
        size_t hcap = (size_t)std::max<int64_t>(1 << 16, nq * 16);
        hcap = std::max<size_t>(hcap, (size_t)ix->hit_hint[mode].load());
        // a fresh index (e.g. after a StreamingIndex rebuild) has no hint yet:
        // use the largest hits-per-query ratio this process has seen, +25%
        hcap = std::max<size_t>(hcap, (size_t)std::min(g_hits_per_query[mode].load() * (double)nq * 1.25,
                                                       (double)(1ll << 27)));
        // test hooks: GTS_HIT_CAP0 = initial hit-buffer rows (no hints), so the
        // grow-and-re-run path runs; GTS_COMPACT_AT = kNN hit compaction threshold
        if (const char *e = std::getenv("GTS_HIT_CAP0")) hcap = (size_t)std::max(1ll, std::atoll(e));
        if (const char *e = std::getenv("GTS_COMPACT_AT")) compact_at = (unsigned long long)std::max(1ll, std::atoll(e));
        hq.alloc(hcap, st);
        he.alloc(hcap, st);
        hd.alloc(hcap, st);
    }

    unsigned long long read_counter(int i)
    {
        CK(cudaMemcpyAsync(h_counter + i, counter.p + i, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return h_counter[i];
    }

    // smem bytes of k_leafgroup_vec for this index (0 = does not fit)
    size_t grouped_smem() const
    {
        const size_t b = ((size_t)ix->max_leaf * (ix->Dp + 4) + 8 * (size_t)ix->Dp) * sizeof(float);
        return b <= 200 * 1024 ? b : 0;
    }

    // rows grouped by leaf into items of <= kItemQueries rows (counting sort)
    struct Grouped {
        DBuf<Row> srows;
        DBuf<Item> items;
        int nitems = 0;
    };

    void group_rows(const Row *rows, int64_t m, Grouped &G, int per = kItemQueries, int first = -1, int count = -1)
    {
        if (first < 0) { first = ix->leaf_first; count = ix->leaf_count; }
        const int nleaf = count;
        DBuf<int> cnt((size_t)nleaf + 1, st), off((size_t)nleaf + 1, st), cur((size_t)nleaf + 1, st);
        DBuf<int> nit((size_t)nleaf + 1, st), ioff((size_t)nleaf + 1, st);
        G.srows.alloc((size_t)m, st);
        CK(cudaMemsetAsync(cnt.p, 0, sizeof(int) * (nleaf + 1), st));
        // block-private counters when the leaves fit in shared memory
        // (GTS_GROUP_ATOMIC=1: the per-row global-atomic kernels)
        static const bool atomic_only = std::getenv("GTS_GROUP_ATOMIC") != nullptr;
        const bool priv = !atomic_only && nleaf <= kPrivLeaves && m >= (int64_t)kPrivThreads * 64;
        static const bool trace = std::getenv("GTS_TRACE") != nullptr;
        if (trace) fprintf(stderr, "[gts] group_rows m=%lld nodes=%d private=%d\n", (long long)m, nleaf, (int)priv);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
        const unsigned pgrid = 2u * (unsigned)sms;
        DBuf<int> bbase;
        if (priv) {
            const size_t sb = (size_t)nleaf * sizeof(int);
            smem_optin((const void *)k_leaf_hist_priv, sb);
            smem_optin((const void *)k_leaf_scatter_priv, sb);
            bbase.alloc((size_t)pgrid * nleaf, st);
            k_leaf_hist_priv<<<pgrid, kPrivThreads, sb, st>>>(rows, m, first, nleaf, cnt.p, bbase.p);
        } else {
            k_leaf_hist<<<grid_for(m, 256), 256, 0, st>>>(rows, m, first, cnt.p);
        }
        LAUNCH_CHECK();
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, nleaf + 1, st);
        DBuf<uint8_t> tmp(tb, st);
        CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, nleaf + 1, st));
        if (priv) {
            k_leaf_scatter_priv<<<pgrid, kPrivThreads, (size_t)nleaf * sizeof(int), st>>>(rows, m, first, nleaf, off.p,
                                                                                         bbase.p, G.srows.p);
        } else {
            CK(cudaMemcpyAsync(cur.p, off.p, sizeof(int) * (nleaf + 1), cudaMemcpyDeviceToDevice, st));
            k_leaf_scatter<<<grid_for(m, 256), 256, 0, st>>>(rows, m, first, cur.p, G.srows.p);
        }
        LAUNCH_CHECK();
        k_item_counts<<<grid_for(nleaf, 256), 256, 0, st>>>(cnt.p, nleaf, per, nit.p);
        LAUNCH_CHECK();
        CK(cudaMemsetAsync(nit.p + nleaf, 0, sizeof(int), st));
        CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, nit.p, ioff.p, nleaf + 1, st));
        g_launches += 4;
        int *h_nitems = reinterpret_cast<int *>(h_counter + 2);
        CK(cudaMemcpyAsync(h_nitems, ioff.p + nleaf, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        G.nitems = *h_nitems;
        if (G.nitems == 0) return;
        G.items.alloc((size_t)G.nitems, st);
        k_make_items<<<grid_for(G.nitems, 256), 256, 0, st>>>(cnt.p, off.p, ioff.p, nleaf, G.nitems, first, per,
                                                              ix->node.p, ix->npos.p, G.items.p, ix->vt_off.p,
                                                              ix->vt_rows.p);
        LAUNCH_CHECK();
    }

    // shared-memory layout of k_leafgroup_edit for this index and batch
    // (total == 0: does not fit, use k_leaf_edit)
    LgEditLayout edit_layout() const
    {
        LgEditLayout L{};
        const int wmax = std::max(1, (qs->max_len + 31) >> 5);
        if (wmax > 4 || ix->max_len > 65535) return L;
        L.cap_e = std::max(ix->max_leaf, 1);
        L.tstride = (((ix->max_len + 3) >> 2)) | 1;
        L.cap_w = L.cap_e * L.tstride;
        L.wmax = wmax;
        L.slot_words = ((wmax * ix->A + 7) & ~7) | 8;   // odd multiple of 8: slots land on different banks
        L.use_hist = ix->ehist.p != nullptr;
        L.two = 2u;
        auto al = [](size_t x) { return (int)((x + 15) & ~(size_t)15); };
        size_t o = al((size_t)L.cap_e * 4);
        L.off_meta = (int)o;
        o += al((size_t)L.cap_e * 4);
        L.off_h0 = (int)o;
        if (L.use_hist) o += (size_t)L.cap_e * 16;
        L.off_h1 = (int)o;
        if (L.use_hist) o += (size_t)L.cap_e * 16;
        L.off_text = (int)o;
        o += al((size_t)L.cap_w * 4);
        L.off_peq = (int)o;
        o += al((size_t)kLgWarps * kLgSlots * L.slot_words * 4);
        L.off_queue = (int)o;
        o += (size_t)kLgWarps * 64 * 4;
        L.off_slot = (int)o;
        o += (size_t)kLgWarps * 4 * kLgSlots * 4;
        if (o > 100 * 1024) return LgEditLayout{};
        L.total = (int)o;
        return L;
    }

    void launch_grouped_edit(const Row *rows, int64_t m, int stats_on, const LgEditLayout &L)
    {
        Grouped G;
        group_rows(rows, m, G, kLgItemRows);
        if (G.nitems == 0) return;
        HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
        smem_optin((const void *)k_leafgroup_edit, 100 * 1024);
        int sms = 148, per = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_leafgroup_edit, 32 * kLgWarps, L.total));
        const unsigned grid = (unsigned)std::min<int64_t>(G.nitems, (int64_t)sms * std::max(per, 1));
        CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), st));
        timed("k_leafgroup_edit", [&] {
            k_leafgroup_edit<<<grid, 32 * kLgWarps, L.total, st>>>(iv, qv, G.srows.p, G.items.p, G.nitems, counter.p, L,
                                                                  pruning, r32.p, hb, verified.p, stats_on,
                                                                  stats_on ? work.p : nullptr,
                                                                  stats_on ? hist.p : nullptr, ks.p);
        });
        LAUNCH_CHECK();
    }

    // tensor-core screen (k_leafgroup_mma2) + exact float64 recheck of the
    // candidate pairs (k_recheck)
    void launch_mma2(const Row *srows, const Item *items, int nitems, int stats_on)
    {
        if (std::getenv("GTS_MMA_V2") == nullptr) {
            launch_mma3(srows, items, nitems, stats_on);
            return;
        }
        // default: one 512-thread CTA per SM, two stages (343 ms per vec128
        // step); GTS_MMA_SHAPE=256 runs two 256-thread one-stage CTAs per SM
        // (measured 443 ms: the shorter epilogues do not cover the exposed
        // MMA and copy latency)
        static const bool two_cta = std::getenv("GTS_MMA_SHAPE") && std::atoi(std::getenv("GTS_MMA_SHAPE")) == 256;
        if (two_cta) launch_mma2_shape<256, 1>(srows, items, nitems, stats_on, 2);
        else launch_mma2_shape<512, 2>(srows, items, nitems, stats_on, 1);
    }

    // barrier-free pipelined tensor-core screen (k_leafgroup_mma3)
    void launch_mma3(const Row *srows, const Item *items, int nitems, int stats_on)
    {
        const int nmax = std::max(16, (ix->max_leaf + 15) & ~15);
        uint32_t cols = 32;
        while ((int)cols < nmax) cols <<= 1;
        const size_t nkb = (size_t)ix->Dk / 64;
        const size_t smb = 2 * (nkb * 16384 + nkb * (size_t)nmax * 128) + 1024;
        smem_optin((const void *)k_leafgroup_mma3, smb);
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
        const unsigned grid = (unsigned)std::min<int>(nitems, sms);
        // column terms of every slot (+16 padding records past the end)
        DBuf<float4> colrec((size_t)ix->n + 16, st);
        k_colrec<<<grid_for(ix->n + 16, 256), 256, 0, st>>>(iv, ix->n, colrec.p);
        LAUNCH_CHECK();
        with_candidates<kMetricL2>([&](const CandBuf &cb, int first) {
            timed("k_leafgroup_mma3", [&] {
                const int on = first && stats_on;
                k_leafgroup_mma3<<<grid, kM3Threads, smb, st>>>(iv, qv, srows, items, nitems, colrec.p, r32.p, r64.p,
                                                               cb, verified.p, on, on ? work.p : nullptr, cols, nmax,
                                                               on ? fhist.p : nullptr, r0.p, ks.p);
            });
            LAUNCH_CHECK();
        }, true);
    }

    template <int NT, int NSTAGE>
    void launch_mma2_shape(const Row *srows, const Item *items, int nitems, int stats_on, int per_sm)
    {
        const int nmax = std::max(16, (ix->max_leaf + 15) & ~15);
        uint32_t cols = 32;
        while ((int)cols < nmax) cols <<= 1;
        const size_t nkb = (size_t)ix->Dk / 64;
        const size_t smb = NSTAGE * (nkb * 16384 + nkb * (size_t)nmax * 128) + 1024;
        smem_optin((const void *)k_leafgroup_mma2<NT, NSTAGE>, smb);
        int sms = 148, fit = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, k_leafgroup_mma2<NT, NSTAGE>, NT, smb));
        per_sm = std::max(1, std::min(per_sm, fit));
        const unsigned grid = (unsigned)std::min<int>(nitems, sms * per_sm);   // items i, i + grid, ... per CTA
        DBuf<unsigned long long> cur(1, st);
        with_candidates<kMetricL2>([&](const CandBuf &cb, int first) {
            CK(cudaMemsetAsync(cur.p, 0, sizeof(unsigned long long), st));
            timed("k_leafgroup_mma2", [&] {
                const int on = first && stats_on;
                k_leafgroup_mma2<NT, NSTAGE><<<grid, NT, smb, st>>>(iv, qv, srows, items, nitems, cur.p, r32.p, r64.p,
                                                                  cb, verified.p, on, on ? work.p : nullptr, cols,
                                                                  nmax, on ? fhist.p : nullptr, r0.p, ks.p);
            });
            LAUNCH_CHECK();
        }, true);
    }

    // Run a screening kernel that appends (query, entry, lower bound) candidates,
    // growing the buffer and re-running (stats off: counts and histograms must
    // not double) on overflow, then recheck them exactly (k_recheck<MET>).
    template <int MET, class Launch>
    // prescreen: the candidates come from the tensor-core screen (wide bf16
    // band), so k_recheck tests them in fp32 before the float64 distance
    void with_candidates(Launch &&launch, bool prescreen = false)
    {
        // the hint is the largest count seen; 50% headroom, since kNN counts vary
        // from call to call (the shrinking radius is order-dependent) and an
        // overflow costs a full re-run of the screening kernel
        const size_t hint = (size_t)ix->cand_hint.load();
        size_t cap = std::max<size_t>((size_t)1 << 22, hint + hint / 2);
        // test hook: GTS_CAND_CAP0 = initial candidate-buffer rows (no hint)
        if (const char *e = std::getenv("GTS_CAND_CAP0")) cap = (size_t)std::max(1ll, std::atoll(e));
        DBuf<unsigned long long> cnt(1, st);
        for (int attempt = 0;; attempt++) {
            if (cq.n < cap) {
                cq.alloc(cap, st);
                ce.alloc(cap, st);
                clb.alloc(cap, st);
            }
            CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
            CandBuf cb{cq.p, ce.p, clb.p, (unsigned long long)cq.n, cnt.p};
            launch(cb, attempt == 0 ? 1 : 0);
            CK(cudaMemcpyAsync(h_counter + 2, cnt.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const unsigned long long nc = h_counter[2];
            {
                unsigned long long c0 = ix->cand_hint.load();
                while (nc > c0 && !ix->cand_hint.compare_exchange_weak(c0, nc)) {}
            }
            static const bool trace = std::getenv("GTS_TRACE") != nullptr;
            if (trace) fprintf(stderr, "[gts] screen candidates=%llu cap=%zu\n", nc, (size_t)cq.n);
            if (nc > cq.n) { cap = (size_t)nc + nc / 2; reruns++; continue; }
            if (nc) {
                HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
                timed("k_recheck", [&] {
                    k_recheck<MET><<<grid_for((int64_t)nc * 8, 256), 256, 0, st>>>(iv, qv, cb, nc, r32.p, r64.p, hb,
                                                                                   prescreen ? 1 : 0);
                });
                LAUNCH_CHECK();
            }
            return;
        }
    }
    int reruns = 0;         // screening launches re-run after a buffer overflow (trace)
    DBuf<int32_t> cq, ce;   // tensor-core candidate pairs
    DBuf<float> clb;        // their d^2 lower bounds

    template <int MET>
    void launch_grouped(const Row *rows, int64_t m, int stats_on)
    {
        Grouped G;
        group_rows(rows, m, G);
        const int nitems = G.nitems;
        if (nitems == 0) return;
        DBuf<Row> &srows = G.srows;
        DBuf<Item> &items = G.items;
        HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
        const size_t sm = grouped_smem();
        if (MET == kMetricL2 && ix->vcent.p && pruning && qs->qbf.p && std::getenv("GTS_MMA_V1") == nullptr) {
            launch_mma2(srows.p, items.p, nitems, stats_on);
            return;
        }
        if (MET == kMetricL2 && ix->vcent.p && pruning) {
            const int nmax = std::max(16, (ix->max_leaf + 15) & ~15);
            const size_t smb = (size_t)(ix->Dk / 64) * (128 * 128 + (size_t)nmax * 128) + 1024;
            smem_optin((const void *)k_leafgroup_mma, 220 * 1024);
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ix->device);
            uint32_t cols = 32;
            while ((int)cols < nmax) cols <<= 1;
            const int per_sm = std::max(1, std::min(3, (int)(512 / cols)));
            unsigned gridm = (unsigned)std::min<int>(nitems, sms * per_sm);
            timed("k_leafgroup_mma", [&] {
                k_leafgroup_mma<<<gridm, kMmaThreads, smb, st>>>(iv, qv, srows.p, items.p, nitems, r32.p, r64.p, hb,
                                                         verified.p, stats_on, stats_on ? work.p : nullptr, cols,
                                                         g_phase_dev, stats_on ? fhist.p : nullptr, r0.p, ks.p);
            });
            LAUNCH_CHECK();
            return;
        }
        {
            // register-tiled kernel when the leaf + 128 query rows fit
            const size_t tsm = ((size_t)ix->max_leaf * (ix->Dp + 4) + (size_t)128 * (ix->Dp + 4) + ix->max_leaf +
                                6 * 128) * sizeof(float);
            if (tsm <= 200 * 1024 && std::getenv("GTS_VEC_ROWWARP") == nullptr) {
                smem_optin((const void *)k_leafgroup_tile<MET>, 200 * 1024);
                int per = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_leafgroup_tile<MET>, 256, tsm));
                const unsigned tgrid = (unsigned)std::min<int64_t>(nitems, (int64_t)148 * std::max(per, 1));
                with_candidates<MET>([&](const CandBuf &cb, int first) {
                    const int on = first && stats_on;
                    timed("k_leafgroup_tile", [&] {
                        k_leafgroup_tile<MET><<<tgrid, 256, tsm, st>>>(iv, qv, srows.p, items.p, nitems, pruning,
                                                                      r32.p, r64.p, cb, verified.p, on,
                                                                      on ? work.p : nullptr, on ? fhist.p : nullptr,
                                                                      r0.p, ks.p);
                    });
                    LAUNCH_CHECK();
                });
                return;
            }
        }
        smem_optin((const void *)k_leafgroup_vec<MET>, 200 * 1024);
        unsigned grid = (unsigned)std::min<int>(nitems, 148 * 8);
        timed("k_leafgroup_vec", [&] {
            k_leafgroup_vec<MET><<<grid, 256, sm, st>>>(iv, qv, srows.p, items.p, nitems, pruning, r32.p, r64.p, hb,
                                                       verified.p, stats_on, stats_on ? work.p : nullptr,
                                                       stats_on ? fhist.p : nullptr, r0.p, ks.p);
        });
        LAUNCH_CHECK();
    }

    template <int MET>
    void launch_verify(const Row *rows, int64_t m, int stats_on)
    {
        // angular: the row-wise kernel (fp32 cosine screen + float64 recheck)
        if constexpr (MET != kMetricAngular) {
            if (grouped_smem() && ix->Dp >= 8 && std::getenv("GTS_NO_GROUPED") == nullptr) {
                launch_grouped<MET>(rows, m, stats_on);
                return;
            }
        }
        HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
        unsigned grid = grid_for(m * 32, 256, 148u * 64u);
        timed("k_verify", [&] {
            k_verify<MET><<<grid, 256, 0, st>>>(iv, qv, rows, m, pruning, r32.p, r64.p, hb, verified.p, stats_on,
                                                stats_on ? work.p : nullptr);
        });
        LAUNCH_CHECK();
    }

    void verify(const Row *rows, int64_t m)
    {
        const unsigned long long before = hits;
        dispatch_verify(rows, m, 1);
        unsigned long long after = read_counter(1);
        if (after > hq.n) {
            reruns++;
            // grow the hit buffer and redo this launch (stats already counted)
            size_t ncap = (size_t)std::max<unsigned long long>(after * 2, hq.n * 2);
            DBuf<int32_t> nq_(ncap, st), ne_(ncap, st);
            DBuf<double> nd_(ncap, st);
            if (before) {
                CK(cudaMemcpyAsync(nq_.p, hq.p, before * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(ne_.p, he.p, before * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(nd_.p, hd.p, before * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
            hq = std::move(nq_);
            he = std::move(ne_);
            hd = std::move(nd_);
            h_counter[1] = before;
            CK(cudaMemcpyAsync(counter.p + 1, h_counter + 1, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
            dispatch_verify(rows, m, 0);
            after = read_counter(1);
        }
        hits = after;
        if (mode == 1 && hits > compact_at) compact_hits();
    }

    // kNN hit buffers: keep only the hits inside the current radii (bounds
    // the buffers and the final sort; a 1M-query k = 100 batch over 100M
    // objects otherwise collects > 2^31 tie-inclusive hits)
    unsigned long long compact_at = 1ull << 26;
    void compact_hits()
    {
        const int64_t n = (int64_t)hits;
        DBuf<int32_t> nq_((size_t)n, st), ne_((size_t)n, st);
        DBuf<double> nd_((size_t)n, st);
        CK(cudaMemsetAsync(counter.p + 1, 0, sizeof(unsigned long long), st));
        k_compact_hits<<<grid_for(n, 256), 256, 0, st>>>(hq.p, he.p, hd.p, n, r32.p,
                                                         ix->metric == GTS_EDIT ? nullptr : r64.p, nq_.p, ne_.p,
                                                         nd_.p, counter.p + 1);
        LAUNCH_CHECK();
        const unsigned long long kept = read_counter(1);
        CK(cudaMemcpyAsync(hq.p, nq_.p, kept * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(he.p, ne_.p, kept * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(hd.p, nd_.p, kept * sizeof(double), cudaMemcpyDeviceToDevice, st));
        hits = kept;
        compact_at = std::max<unsigned long long>(compact_at, 2 * kept);
    }

    DBuf<unsigned> hist;   // kNN edit: per-query distance histogram (shrinking bound)
    DBuf<unsigned> fhist;  // kNN vectors: per-query 64-bin histogram over [0, r0]
    DBuf<float> r0;        // kNN vectors: the probe radius (histogram scale)

    void dispatch_verify(const Row *rows, int64_t m, int stats_on)
    {
        switch (ix->metric) {
        case GTS_EDIT: {
            // k_leafgroup_edit is opt-in: the DP and the per-entry filters are
            // ALU-pipe bound, not L2 bound, and the row-wise kernel measured
            // faster on words (87.6 vs 129.6 ms/step) and DNA (4.93 vs 5.05 s)
            const LgEditLayout L = edit_layout();
            if (L.total && std::getenv("GTS_EDIT_GROUPED") != nullptr && std::getenv("GTS_NO_GROUPED") == nullptr) {
                launch_grouped_edit(rows, m, stats_on, L);
                break;
            }
            HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
            // at most 2^24 rows per launch (GTS_EDIT_LAUNCH_ROWS overrides):
            // larger launches measured superlinearly slower for the same work
            static const int64_t env_lr = std::getenv("GTS_EDIT_LAUNCH_ROWS") ? std::atoll(std::getenv("GTS_EDIT_LAUNCH_ROWS")) : 0;
            const int64_t launch_rows = env_lr > 0 ? env_lr : (1ll << 24);
            if (m > launch_rows) {
                for (int64_t o = 0; o < m; o += launch_rows)
                    dispatch_verify(rows + o, std::min<int64_t>(launch_rows, m - o), stats_on);
                break;
            }
            // one warp per ~contiguous run of rows; enough warps to fill the GPU
            // rows per cursor claim: 16 (GTS_EDIT_CLAIM overrides).  Larger kNN
            // claims (one warp walking a query's leaves in order) did not cut
            // the DP work -- the probe radius is already near the final one --
            // and cost balance (words: 88.7 vs 83.6 ms)
            static const int env_claim = std::getenv("GTS_EDIT_CLAIM") ? std::atoi(std::getenv("GTS_EDIT_CLAIM")) : 0;
            const int claim = env_claim > 0 ? std::max(kRowChunk, env_claim) : kRowChunk;
            unsigned grid = grid_for((m + kRowChunk - 1) / kRowChunk, kLeafWarps, 148u * 4u);   // 4 resident per SM
            // opt-in (GTS_EDIT_SMEM_TEXT=1): texts staged in smem for the DP
            // (byte loads, no symbol extraction).  Measured slower on words
            // (92.2 vs 83.9 ms): the staging copies cost more than the one ALU
            // op per symbol they save
            const char *env_tx = std::getenv("GTS_EDIT_SMEM_TEXT");
            int tstride = 0;
            if (ix->max_len <= 64 && env_tx && env_tx[0] == '1') tstride = (((ix->max_len + 3) >> 2) | 1);
            const size_t dyn = (size_t)tstride * kWarp * kLeafWarps * sizeof(uint32_t);
            // static 38.9 KB + up to 17 KB of staged texts
            // the q-gram signature test is compiled in only where the index has
            // signatures (small alphabets), so the words kernel stays as it was
            using KernT = decltype(&k_leaf_edit<false, true, true>);
            static const KernT kerns[2][2][2] = {
                {{k_leaf_edit<false, false, false>, k_leaf_edit<false, false, true>},
                 {k_leaf_edit<false, true, false>, k_leaf_edit<false, true, true>}},
                {{k_leaf_edit<true, false, false>, k_leaf_edit<true, false, true>},
                 {k_leaf_edit<true, true, false>, k_leaf_edit<true, true, true>}}};
            auto *kern = kerns[ix->esig.p ? 1 : 0][pruning ? 1 : 0][ix->ehist.p ? 1 : 0];
            smem_optin((const void *)kern, 64 * 1024);
            CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), st));
            timed("k_leaf_edit", [&] {
                kern<<<grid, 32 * kLeafWarps, dyn, st>>>(iv, qv, rows, m, pruning, r32.p, hb, verified.p,
                                                               stats_on, stats_on ? work.p : nullptr, counter.p,
                                                               // a re-run (stats_on == 0) must not count twice
                                                               stats_on ? hist.p : nullptr, ks.p, claim, tstride);
            });
            LAUNCH_CHECK();
            break;
        }
        case GTS_L1: launch_verify<kMetricL1>(rows, m, stats_on); break;
        case GTS_ANGULAR: launch_verify<kMetricAngular>(rows, m, stats_on); break;
        default: launch_verify<kMetricL2>(rows, m, stats_on); break;
        }
    }

    template <int MET>
    int64_t launch_expand(const Row *in, int64_t m, int own, Row *out, int layer)
    {
        if ((MET == kMetricL1 || MET == kMetricL2) && ix->D >= 16 && std::getenv("GTS_NO_GROUPED") == nullptr) {
            // parent rows of this layer are nodes [first, first + count)
            int64_t c = 1;
            for (int l = 1; l < layer; l++) c *= ix->nc;
            const int first = (int)((c - 1) / (ix->nc - 1) + 1);
            Grouped G;
            group_rows(in, m, G, kItemQueries, first, (int)c);
            CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), st));
            if (G.nitems == 0) return 0;
            if (ix->nc <= 32 && ix->Dp <= 128 && std::getenv("GTS_EXPAND_NOTILE") == nullptr) {
                const int need = (ix->nc + 3) / 4;
                const int cpg = need <= 2 ? 2 : (need <= 5 ? 5 : 8);   // the kernel's CPG (smem sized for it)
                const size_t smt = ((size_t)4 * cpg * (ix->Dp + 4) + (size_t)kXtRows * (ix->Dp + 4)) * sizeof(float) +
                                   (size_t)4 * cpg * sizeof(NodeRec);
                const unsigned gt = (unsigned)std::min<int>(G.nitems, 148 * 2);
                auto go = [&](auto kern) {
                    smem_optin((const void *)kern, smt);
                    timed("k_expand", [&] {
                        kern<<<gt, 256, smt, st>>>(iv, qv, G.srows.p, G.items.p, G.nitems, own, pruning, r32.p, out,
                                                   counter.p, pruned.p);
                    });
                };
                if (cpg == 2) go(k_expand_tile<MET, 2>);
                else if (cpg == 5) go(k_expand_tile<MET, 5>);
                else go(k_expand_tile<MET, 8>);
                LAUNCH_CHECK();
                return (int64_t)read_counter(0);
            }
            const size_t smb = (size_t)ix->nc * (ix->Dp + 4) * sizeof(float) + (size_t)ix->nc * sizeof(NodeRec);
            smem_optin((const void *)k_expand_grouped<MET>, smb);
            const unsigned grid = (unsigned)std::min<int>(G.nitems, 148 * 8);
            timed("k_expand", [&] {
                k_expand_grouped<MET><<<grid, 256, smb, st>>>(iv, qv, G.srows.p, G.items.p, G.nitems, own, pruning,
                                                            r32.p, out, counter.p, pruned.p);
            });
            LAUNCH_CHECK();
            return (int64_t)read_counter(0);
        }
        CK(cudaMemsetAsync(counter.p, 0, sizeof(unsigned long long), st));
        unsigned grid = grid_for(m * ix->nc, 256, 148u * 32u);
        timed("k_expand", [&] {
            k_expand<MET><<<grid, 256, 0, st>>>(iv, qv, in, m, own, pruning, r32.p, out, counter.p, pruned.p);
        });
        LAUNCH_CHECK();
        return (int64_t)read_counter(0);
    }

    int64_t expand(const Row *in, int64_t m, int layer, Row *out)
    {
        const int own = (layer + 1) == ix->levels;
        int64_t cnt;
        switch (ix->metric) {
        case GTS_EDIT: cnt = launch_expand<kMetricEdit>(in, m, own, out, layer); break;
        case GTS_L1: cnt = launch_expand<kMetricL1>(in, m, own, out, layer); break;
        case GTS_ANGULAR: cnt = launch_expand<kMetricAngular>(in, m, own, out, layer); break;
        default: cnt = launch_expand<kMetricL2>(in, m, own, out, layer); break;
        }
        if (prof) {
            // algorithmic traversal bytes: the parent row,
            // N_c 16-byte child records, the pivot payload of every child
            // whose distance is evaluated (internal levels: the survivors of
            // the parent-range pre-screen = the emitted rows; the leaf level:
            // every child) and the emitted 16-byte rows
            const int64_t evaluated = own ? m * ix->nc : cnt;
            const double pay = ix->metric == GTS_EDIT ? ix->avg_text_bytes : 4.0 * ix->Dp;
            std::lock_guard<std::mutex> g(g_prof_mu);
            g_expand[0] += (double)m * 16.0 * (1 + ix->nc) + (double)evaluated * pay + (double)cnt * 16.0;
            g_expand[1] += (double)m;
            g_expand[2] += (double)cnt;
            g_expand[3] += (double)evaluated;
        }
        return cnt;
    }

    // depth-first over layers in chunks of level_size_limit parent rows
    void process(int layer, const Row *rows, int64_t m)
    {
        if (m == 0) return;
        if (layer == ix->levels) { verify(rows, m); return; }
        const int64_t s = level_size_limit(cap, ix->nc, ix->split_rounds, layer);
        if (layer < 64 && limits[layer] == 0) limits[layer] = s;
        for (int64_t off = 0; off < m; off += s) {
            const int64_t mm = std::min<int64_t>(s, m - off);
            DBuf<Row> child((size_t)(mm * ix->nc), st);
            int64_t cnt = expand(rows + off, mm, layer, child.p);
            peak = std::max(peak, cnt);
            if (cnt > cap) fail(GTS_EBUDGET, "table of %lld rows overflows budget %lld", (long long)cnt, (long long)cap);
            process(layer + 1, child.p, cnt);
        }
    }

    template <int MET>
    void launch_root(Row *out)
    {
        timed("k_root", [&] { k_root<MET><<<grid_for(nq, 256), 256, 0, st>>>(iv, qv, (int)nq, out); });
        LAUNCH_CHECK();
    }

    template <int MET>
    void launch_probe()
    {
        // node-major for wide vectors; low-dimensional probes are cheap per query
        if ((MET == kMetricL1 || MET == kMetricL2) && ix->D >= 16 && std::getenv("GTS_PROBE_PERQUERY") == nullptr) {
            launch_probe_grouped<MET>();
            return;
        }
        timed("k_probe", [&] {
            k_probe<MET><<<grid_for(nq, 1, 148u * 16u), 256, 0, st>>>(iv, qv, (int)nq, ks.p, r32.p, r64.p);
        });
        LAUNCH_CHECK();
    }

    template <int MET>
    void launch_finite_bound()
    {
        const float rr = std::max(ix->root_radius, ix->cache_radius);
        if (!(rr < INFINITY)) return;
        k_finite_bound<MET><<<grid_for(nq, 256), 256, 0, st>>>(iv, qv, (int)nq, rr, r32.p, r64.p);
        LAUNCH_CHECK();
    }

    template <int MET>
    void launch_probe_grouped()
    {
        // 2^17 queries per pass: <= 4 GiB of candidate distances (kProbeCand
        // floats per query, 2% of HBM).  Smaller passes measured slower:
        // 2^15 took the vec128 probe from 17.5 to 26.8 ms (fewer queries per
        // probed node, so k_probe_dist's node-major tiles are emptier)
        const int64_t qchunk = std::min<int64_t>(nq, 1 << 17);
        const size_t pd_smem = (size_t)2 * kPT * (kPD + 4) * sizeof(float);
        smem_optin((const void *)k_probe_dist<kMetricL1>, pd_smem);
        smem_optin((const void *)k_probe_dist<kMetricL2>, pd_smem);
        DBuf<uint32_t> keys((size_t)kProbeRows * qchunk, st), skeys((size_t)kProbeRows * qchunk, st);
        DBuf<int32_t> vals((size_t)kProbeRows * qchunk, st), svals((size_t)kProbeRows * qchunk, st);
        DBuf<float> dist((size_t)qchunk * kProbeCand, st);
        size_t tmp_bytes = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys.p, skeys.p, vals.p, svals.p, (int)(kProbeRows * qchunk), 0, 32, st);
        DBuf<uint8_t> tmp(tmp_bytes, st);
        for (int64_t q0 = 0; q0 < nq; q0 += qchunk) {
            const int nqc = (int)std::min<int64_t>(qchunk, nq - q0);
            const int nrows = kProbeRows * nqc;
            timed("k_probe", [&] {
                k_probe_path<MET><<<grid_for((int64_t)nqc * 32, 256), 256, 0, st>>>(iv, qv, (int)q0, nqc, ks.p, keys.p,
                                                                                  vals.p);
                CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, keys.p, skeys.p, vals.p, svals.p, nrows, 0, 32, st));
                k_probe_dist<MET><<<(unsigned)((nrows + kPT - 1) / kPT), 256, pd_smem, st>>>(
                    iv, qv, (int)q0, skeys.p, svals.p, nrows, keys.p, dist.p);
                k_probe_select<MET><<<grid_for(nqc, 1, 148u * 16u), 256, 0, st>>>(iv, (int)q0, nqc, ks.p, keys.p, dist.p,
                                                                                  r32.p, r64.p);
            });
            LAUNCH_CHECK();
            g_launches += 2;   // path, dist, select (+ the CUB sort)
        }
    }

    void run()
    {
        if (ix->levels == 0 || ix->n == 0 || nq == 0) return;
        if (mode == 1 && ix->metric == GTS_EDIT) {
            hist.alloc((size_t)nq * kHistBins, st);
            CK(cudaMemsetAsync(hist.p, 0, sizeof(unsigned) * (size_t)nq * kHistBins, st));
        }
        if (mode == 1 && pruning) {
            if (ext_bound) {
                k_set_bound<<<grid_for(nq, 256), 256, 0, st>>>(ext_bound, (int)nq, r32.p, r64.p);
                LAUNCH_CHECK();
            } else {
                switch (ix->metric) {
                case GTS_EDIT: launch_probe<kMetricEdit>(); break;
                case GTS_L1: launch_probe<kMetricL1>(); launch_finite_bound<kMetricL1>(); break;
                case GTS_ANGULAR: launch_probe<kMetricAngular>(); launch_finite_bound<kMetricAngular>(); break;
                default: launch_probe<kMetricL2>(); launch_finite_bound<kMetricL2>(); break;
                }
            }
            if (probe_out) {
                CK(cudaMemcpyAsync(probe_out, r32.p, sizeof(float) * nq, cudaMemcpyDeviceToDevice, st));
                return;
            }
            if (ix->metric != GTS_EDIT) {
                fhist.alloc((size_t)nq * kFHist, st);
                CK(cudaMemsetAsync(fhist.p, 0, sizeof(unsigned) * (size_t)nq * kFHist, st));
                r0.alloc((size_t)nq, st);
                CK(cudaMemcpyAsync(r0.p, r32.p, sizeof(float) * nq, cudaMemcpyDeviceToDevice, st));
            }
        }
        if (!pruning) {
            // every live entry of every leaf is verified (search.py:338-355)
            const int64_t nl = std::max(ix->n_live_leaves, 1);
            const int64_t qchunk = std::max<int64_t>(1, cap / nl);
            for (int64_t q0 = 0; q0 < nq; q0 += qchunk) {
                const int64_t nqc = std::min<int64_t>(qchunk, nq - q0);
                const int64_t m = nqc * ix->n_live_leaves;
                if (m == 0) continue;
                DBuf<Row> rows((size_t)m, st);
                k_all_leaves<<<grid_for(m, 256), 256, 0, st>>>(ix->live_leaves.p, ix->n_live_leaves, (int)q0,
                                                               (int)nqc, rows.p);
                LAUNCH_CHECK();
                verify(rows.p, m);
            }
            return;
        }
        DBuf<Row> root((size_t)nq, st);
        switch (ix->metric) {
        case GTS_EDIT: launch_root<kMetricEdit>(root.p); break;
        case GTS_L1: launch_root<kMetricL1>(root.p); break;
        case GTS_ANGULAR: launch_root<kMetricAngular>(root.p); break;
        default: launch_root<kMetricL2>(root.p); break;
        }
        process(1, root.p, nq);
    }

    template <int MET>
    void launch_cache_scan()
    {
        CacheView cv{ix->cache_n, ix->cache_ids.p, ix->cache_vec32.p, ix->cache_vec64.p, ix->cache_words.p,
                     ix->cache_sword.p, ix->cache_slen.p};
        HitBuf hb{hq.p, he.p, hd.p, (unsigned long long)hq.n, counter.p + 1};
        k_cache_scan<MET><<<grid_for((int64_t)nq * cv.n, 256), 256, 0, st>>>(iv, qv, cv, (int)nq, r32.p, r64.p, hb);
        LAUNCH_CHECK();
    }

    // the pending-insert cache after the tree (the radius is final for kNN)
    void scan_cache()
    {
        if (!use_cache || ix->cache_n == 0 || nq == 0) return;
        const unsigned long long before = hits;
        for (int attempt = 0; attempt < 2; attempt++) {
            h_counter[1] = before;
            CK(cudaMemcpyAsync(counter.p + 1, h_counter + 1, sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
            switch (ix->metric) {
            case GTS_EDIT: launch_cache_scan<kMetricEdit>(); break;
            case GTS_L1: launch_cache_scan<kMetricL1>(); break;
            case GTS_ANGULAR: launch_cache_scan<kMetricAngular>(); break;
            default: launch_cache_scan<kMetricL2>(); break;
            }
            const unsigned long long after = read_counter(1);
            if (after <= hq.n) { cache_hits = after > before; hits = after; return; }
            const size_t ncap = (size_t)after * 2;
            DBuf<int32_t> nq_(ncap, st), ne_(ncap, st);
            DBuf<double> nd_(ncap, st);
            if (before) {
                CK(cudaMemcpyAsync(nq_.p, hq.p, before * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(ne_.p, he.p, before * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
                CK(cudaMemcpyAsync(nd_.p, hd.p, before * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
            hq = std::move(nq_);
            he = std::move(ne_);
            hd = std::move(nd_);
        }
        fail(GTS_ECUDA, "cache scan: hit buffer growth failed");
    }

    // sort hits by (q, d, id) and build the CSR result (search.py:298-314)
    void collect(gts_result *res)
    {
        cudaEvent_t ca = nullptr, cb = nullptr;
        if (prof) {
            CK(cudaEventCreate(&ca));
            CK(cudaEventCreate(&cb));
            CK(cudaEventRecord(ca, st));
        }
        collect_impl(res);
        if (prof) {
            CK(cudaEventRecord(cb, st));
            events.emplace_back("collect", ca, cb);
        }
        flush_profile();
    }

    void collect_impl(gts_result *res)
    {
        const int64_t n = (int64_t)hits;
        // the CUB sorts index with int: fail loudly instead of truncating
        if (n > (int64_t)INT32_MAX)
            fail(GTS_EBUDGET, "%lld answers in one batch exceed 2^31-1; split the query batch", (long long)n);
        res->nq = nq;
        res->peak = peak;
        std::memcpy(res->limits, limits, sizeof(limits));
        res->stream = st;
        res->offsets.alloc((size_t)nq + 1, st);
        res->verified = std::move(verified);
        res->pruned = std::move(pruned);
        DBuf<long long> counts((size_t)nq + 1, st), outcnt((size_t)nq + 1, st);
        DBuf<long long> in_off((size_t)nq + 1, st), out_off((size_t)nq + 1, st);
        CK(cudaMemsetAsync(counts.p, 0, sizeof(long long) * (nq + 1), st));
        DBuf<int32_t> perm_a, perm_b;
        // packed-key fast path for exact integer distances (edit)
        int qbits = 1;
        while ((1ll << qbits) < nq) qbits++;
        int dbits = 1;
        while ((1ll << dbits) <= (long long)std::max(ix->max_len, max_qlen)) dbits++;
        int rbits = 1;
        while ((1ll << rbits) < ix->n) rbits++;
        // ids in slot order no longer follow row order once a slot was filled
        // by an insert: sort by the 64-bit id then
        const bool by_id = cache_hits || ix->n_inserted > 0;
        const bool packed = ix->metric == GTS_EDIT && qbits + dbits + rbits <= 64 && !by_id;
        if (n > 0 && packed) {
            DBuf<unsigned long long> ka((size_t)n, st), kb((size_t)n, st);
            perm_a.alloc((size_t)n, st);
            perm_b.alloc((size_t)n, st);
            const unsigned g = grid_for(n, 256);
            k_pack_keys<<<g, 256, 0, st>>>(hq.p, he.p, hd.p, ix->row.p, n, rbits, rbits + dbits, ka.p, perm_a.p);
            LAUNCH_CHECK();
            size_t tmp_bytes = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0,
                                            qbits + dbits + rbits, st);
            DBuf<uint8_t> tmp(tmp_bytes, st);
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0,
                                               qbits + dbits + rbits, st));
            g_launches += 4;
            k_seg_counts<<<grid_for(nq, 256), 256, 0, st>>>(kb.p, n, rbits + dbits, (int)nq, counts.p);
            LAUNCH_CHECK();
        } else if (n > 0 && !by_id && 32 + rbits <= 64 && std::getenv("GTS_COLLECT_3SORT") == nullptr) {
            // float distances: (float32(d), row) sort, stable query sort, tie fix-up
            DBuf<unsigned long long> ka((size_t)n, st), kb((size_t)n, st);
            perm_a.alloc((size_t)n, st);
            perm_b.alloc((size_t)n, st);
            const unsigned g = grid_for(n, 256);
            k_pack_f32_keys<<<g, 256, 0, st>>>(he.p, hd.p, n, ix->row.p, rbits, ka.p, perm_a.p);
            LAUNCH_CHECK();
            size_t tmp_bytes = 0, t2 = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0, 32 + rbits, st);
            cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr, perm_a.p,
                                            perm_b.p, (int)n, 0, 32, st);
            tmp_bytes = std::max(tmp_bytes, t2);
            DBuf<uint8_t> tmp(tmp_bytes, st);
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0, 32 + rbits,
                                               st));
            DBuf<uint32_t> qa((size_t)n, st), qb((size_t)n, st);
            k_gather_q<<<g, 256, 0, st>>>(hq.p, perm_b.p, n, qa.p);
            LAUNCH_CHECK();
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, qa.p, qb.p, perm_b.p, perm_a.p, (int)n, 0, qbits, st));
            k_fix_f32_ties<<<g, 256, 0, st>>>(perm_a.p, hq.p, he.p, hd.p, ix->row.p, n);
            LAUNCH_CHECK();
            std::swap(perm_a, perm_b);   // k_emit reads perm_b
            g_launches += 8;
            k_count<<<g, 256, 0, st>>>(hq.p, n, counts.p);
            LAUNCH_CHECK();
        } else if (n > 0) {
            DBuf<unsigned long long> ka((size_t)n, st), kb((size_t)n, st);
            perm_a.alloc((size_t)n, st);
            perm_b.alloc((size_t)n, st);
            const unsigned g = grid_for(n, 256);
            if (by_id) {
                k_gather_id<<<g, 256, 0, st>>>(he.p, n, ix->ids.p, ix->cache_ids.p, ka.p, perm_a.p);
                LAUNCH_CHECK();
            }
            size_t tmp_bytes = 0, t2 = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0, 64, st);
            cub::DeviceRadixSort::SortPairs(nullptr, t2, (uint32_t *)nullptr, (uint32_t *)nullptr, perm_a.p,
                                            perm_b.p, (int)n, 0, 32, st);
            tmp_bytes = std::max(tmp_bytes, t2);
            DBuf<uint8_t> tmp(tmp_bytes, st);
            // 1) by id (by dataset row, rbits wide, when no cache or inserted entry is among the hits)
            if (!by_id) {
                DBuf<uint32_t> ra((size_t)n, st), rb((size_t)n, st);
                k_gather_row<<<g, 256, 0, st>>>(he.p, n, ix->row.p, ra.p, perm_a.p);
                LAUNCH_CHECK();
                CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ra.p, rb.p, perm_a.p, perm_b.p, (int)n, 0, rbits,
                                                   st));
            } else {
                CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, perm_a.p, perm_b.p, (int)n, 0, 64, st));
            }
            g_launches += 4;
            // 2) stable by distance bits (non-negative doubles order as integers)
            k_gather_d<<<g, 256, 0, st>>>(hd.p, perm_b.p, n, ka.p);
            LAUNCH_CHECK();
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, ka.p, kb.p, perm_b.p, perm_a.p, (int)n, 0, 64, st));
            g_launches += 4;
            // 3) stable by query
            DBuf<uint32_t> qa((size_t)n, st), qb((size_t)n, st);
            k_gather_q<<<g, 256, 0, st>>>(hq.p, perm_a.p, n, qa.p);
            LAUNCH_CHECK();
            CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, qa.p, qb.p, perm_a.p, perm_b.p, (int)n, 0, qbits, st));
            g_launches += 2;
            k_count<<<g, 256, 0, st>>>(hq.p, n, counts.p);
            LAUNCH_CHECK();
        }
        k_clamp_counts<<<grid_for(nq, 256), 256, 0, st>>>(counts.p, mode == 1 ? ks.p : nullptr, (int)nq, outcnt.p);
        LAUNCH_CHECK();
        size_t sb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, sb, counts.p, in_off.p, (int)nq + 1, st);
        DBuf<uint8_t> stmp(sb, st);
        CK(cub::DeviceScan::ExclusiveSum(stmp.p, sb, counts.p, in_off.p, (int)nq + 1, st));
        CK(cub::DeviceScan::ExclusiveSum(stmp.p, sb, outcnt.p, out_off.p, (int)nq + 1, st));
        g_launches += 2;
        long long total = 0;
        CK(cudaMemcpyAsync(&total, out_off.p + nq, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        res->total = total;
        res->ids.alloc((size_t)std::max<long long>(total, 1), st);
        res->dis.alloc((size_t)std::max<long long>(total, 1), st);
        CK(cudaMemcpyAsync(res->offsets.p, out_off.p, sizeof(long long) * (nq + 1), cudaMemcpyDeviceToDevice, st));
        if (n > 0) {
            k_emit<<<grid_for(n, 256), 256, 0, st>>>(perm_b.p, hq.p, he.p, hd.p, in_off.p, out_off.p, outcnt.p,
                                                     ix->ids.p, ix->cache_ids.p, n, res->ids.p, res->dis.p);
            LAUNCH_CHECK();
        }
    }
};

void check_queries(const gts_index *ix, const gts_queries *q)
{
    if (!ix || !q) fail(GTS_EINVAL, "null index or queries");
    if (q->metric != ix->metric) fail(GTS_EMETRIC, "query metric %d != index metric %d", q->metric, ix->metric);
    if (ix->metric != GTS_EDIT && ix->n > 0 && q->D != ix->D)
        fail(GTS_EMETRIC, "query dimensionality %d != dataset dimensionality %d", q->D, ix->D);
}

gts_queries *upload_queries(gts_index *ix, const gts_query_batch *qb, cudaStream_t st)
{
    if (!qb) fail(GTS_EINVAL, "null query batch");
    if (qb->nq < 0 || qb->nq > (1ll << 31) - 2) fail(GTS_EINVAL, "bad query count");
    if (qb->metric != ix->metric) fail(GTS_EMETRIC, "query metric %d != index metric %d", qb->metric, ix->metric);
    CK(cudaSetDevice(ix->device));
    auto *q = new gts_queries();
    try {
        q->metric = qb->metric;
        q->nq = qb->nq;
        q->stream = st;
        const int64_t nq = qb->nq;
        if (ix->metric == GTS_EDIT) {
            const int64_t nsym = nq ? qb->offsets[nq] : 0;
            std::vector<int64_t> peq_off((size_t)nq + 1, 0);
            for (int64_t i = 0; i < nq; i++) {
                int64_t m = qb->offsets[i + 1] - qb->offsets[i];
                if (m < 0) fail(GTS_EINVAL, "query offsets not monotone");
                // patterns beyond 32 * kMaxWords symbols run the row-band DP
                // (myers_banded), which holds per-text-column carries: one
                // side of every pair must fit 32 * kMaxWords symbols
                if (m > 32 * kMaxWords && std::max(ix->max_len, ix->cache_max_len) > 32 * kMaxWords)
                    fail(GTS_EINVAL, "query of %lld symbols against stored strings of more than %d symbols",
                         (long long)m, 32 * kMaxWords);
                q->max_len = std::max<int>(q->max_len, (int)m);
                peq_off[(size_t)i + 1] = peq_off[(size_t)i] + (int64_t)ix->A * ((m + 31) / 32);
            }
            q->soff.alloc((size_t)nq + 1, st);
            h2d(q->soff.p, qb->offsets, (size_t)nq + 1, st);
            q->peq_off.alloc((size_t)nq + 1, st);
            h2d(q->peq_off.p, peq_off.data(), (size_t)nq + 1, st);
            q->str.alloc((size_t)std::max<int64_t>(nsym, 1), st);   // u8 symbols (Peq build only)
            q->peq.alloc((size_t)std::max<int64_t>(peq_off[(size_t)nq], 1), st);
            CK(cudaMemsetAsync(q->peq.p, 0, sizeof(uint32_t) * q->peq.n, st));
            if (nsym) {
                DBuf<int32_t> codes((size_t)nsym, st);
                h2d(codes.p, qb->codes, (size_t)nsym, st);
                k_map_symbols<<<grid_for(nsym, 256), 256, 0, st>>>(codes.p, nsym, ix->alpha.p, ix->A, q->str.p);
                LAUNCH_CHECK();
                k_build_peq<<<grid_for(nsym, 256), 256, 0, st>>>(q->str.p, q->soff.p, q->peq_off.p, (int)nq, nsym,
                                                                 q->peq.p);
                LAUNCH_CHECK();
            }
            if (ix->esig.p && nq) {
                q->qsig.alloc((size_t)nq * 2, st);
                k_query_sig<<<grid_for(nq, 128), 128, 0, st>>>(q->str.p, q->soff.p, (int)nq, ix->A, q->qsig.p);
                LAUNCH_CHECK();
            }
            if (ix->ehist.p && nq) {
                q->qhist.alloc((size_t)nq * 2, st);
                k_query_hist<<<grid_for(nq, 128), 128, 0, st>>>(q->str.p, q->soff.p, (int)nq, q->qhist.p);
                LAUNCH_CHECK();
            }
        } else {
            q->D = (int)qb->dim;
            q->Dp = (q->D + 3) & ~3;
            if (ix->n > 0 && q->D != ix->D)
                fail(GTS_EMETRIC, "query dimensionality %d != dataset dimensionality %d", q->D, ix->D);
            q->vec64.alloc((size_t)std::max<int64_t>(nq * q->D, 1), st);
            h2d(q->vec64.p, qb->vectors, (size_t)(nq * q->D), st);
            q->vec32.alloc((size_t)std::max<int64_t>(nq * q->Dp, 1), st);
            DBuf<unsigned> flags(2, st);
            CK(cudaMemsetAsync(flags.p, 0, 2 * sizeof(unsigned), st));
            if (nq * q->Dp) {
                k_vec_prep<<<grid_for(nq * q->Dp, 256), 256, 0, st>>>(q->vec64.p, nq, q->D, q->Dp, q->vec32.p,
                                                                      flags.p, (int *)(flags.p + 1));
                LAUNCH_CHECK();
            }
            if (ix->metric == GTS_ANGULAR && nq) {
                std::vector<double> nrm((size_t)nq), tmp;
                std::vector<float> nrm32((size_t)nq);
                for (int64_t i = 0; i < nq; i++) {
                    nrm[(size_t)i] = host_norm(qb->vectors + i * q->D, q->D, tmp);
                    nrm32[(size_t)i] = (float)nrm[(size_t)i];
                }
                q->qnorm64.alloc((size_t)nq, st);
                h2d(q->qnorm64.p, nrm.data(), (size_t)nq, st);
                q->qnorm32.alloc((size_t)nq, st);
                h2d(q->qnorm32.p, nrm32.data(), (size_t)nq, st);
                CK(cudaStreamSynchronize(st));
            }
            if (ix->vcent.p && nq) {
                q->qbf.alloc((size_t)nq * (ix->Dk / 8), st);
                q->qn.alloc((size_t)nq, st);
                k_query_bf16<<<grid_for(nq, 128), 128, 0, st>>>(q->vec32.p, nq, q->D, q->Dp, ix->Dk, q->qbf.p, q->qn.p);
                LAUNCH_CHECK();
            }
            unsigned hf[2];
            CK(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            float mx;
            std::memcpy(&mx, &hf[0], 4);
            q->maxabs = mx;
            q->exact = hf[1] == 0;
        }
        return q;
    } catch (...) {
        delete q;
        throw;
    }
}

static double now_ms()
{
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int64_t hbm_rows_query(const gts_index *ix)
{
    static const char *env = std::getenv("GTS_DEFAULT_ROWS");
    if (env) return std::max<int64_t>(std::atoll(env), ix->nc);
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
        cudaGetLastError();
        return 1ll << 24;
    }
    const int64_t rows = (int64_t)(free_b / 4 / (16 * (size_t)std::max(ix->levels, 1)));
    // Cap per table, measured on B200: strings 2^24 rows (words: 84 ms of
    // k_leaf_edit per step at 2^24-row tables vs 119 ms at 2^25 and 153 ms at
    // 2^26 for the same DP work); vectors 2^26 rows (fewer, larger launches:
    // 128-d L2 497 vs 508 ms per step, 32-d L1 shard 517 vs 578 ms)
    const int64_t cap = ix->metric == GTS_EDIT ? (1ll << 24) : (1ll << 26);
    return std::max<int64_t>(std::min<int64_t>(rows, cap), std::max<int64_t>(ix->nc, 1ll << 16));
}

// cudaMemGetInfo asks the resource manager and measured 50-80 ms when it
// coincided with other driver activity (words bench, B200): query free HBM
// once per index and reuse it
int64_t hbm_rows(gts_index *ix)
{
    int64_t v = ix->hbm_rows_cached.load();
    if (v <= 0) {
        v = hbm_rows_query(ix);
        ix->hbm_rows_cached.store(v);
    }
    return v;
}

gts_result *run_search(gts_index *ix, const gts_queries *q, int mode, const double *radii, const int64_t *ks,
                       int64_t memory_units, int pruning, cudaStream_t st, bool use_cache = false,
                       const float *ext_bound = nullptr, float *probe_out = nullptr)
{
    static const bool trace = std::getenv("GTS_TRACE") != nullptr;
    const double t0 = trace ? now_ms() : 0.0;
    check_queries(ix, q);
    CK(cudaSetDevice(ix->device));
    // 0 = device default, sized to HBM: the depth-first driver keeps at most
    // one child table per layer alive (16-byte rows), and those tables may
    // take a quarter of the free device memory, capped at 2^26 rows per
    // table (1 GiB) -- the reference's 1<<20 (runtime.py:18) was sized for a
    // CPU; the chunking formula (level_size_limit) is the same
    const int64_t cap = memory_units > 0 ? memory_units : hbm_rows(ix);
    if (ix->n > 0 && cap < ix->nc) fail(GTS_EBUDGET, "memory_units %lld below fan-out %d", (long long)cap, ix->nc);
    const int64_t nq = q->nq;
    PinnedArena &pa = pinned_arena();
    pa.off = 0;
    Search s(ix, q, st, mode, cap, pruning);
    s.max_qlen = q->max_len;
    s.r32.alloc((size_t)std::max<int64_t>(nq, 1), st);
    s.r64.alloc((size_t)std::max<int64_t>(nq, 1), st);
    if (mode == 0) {
        std::vector<float> h32((size_t)nq);
        for (int64_t i = 0; i < nq; i++) {
            if (!(radii[i] >= 0)) fail(GTS_EINVAL, "radius must be >= 0");
            if (ix->metric == GTS_EDIT) {
                double f = std::floor(radii[i]);
                h32[(size_t)i] = (float)std::min(f, 16777216.0);
            } else {
                h32[(size_t)i] = round_up_f32(radii[i]);
            }
        }
        h2d(s.r32.p, pa.stage(h32.data(), (size_t)nq), (size_t)nq, st);
        h2d(s.r64.p, pa.stage(radii, (size_t)nq), (size_t)nq, st);
    } else {
        std::vector<int32_t> hk((size_t)nq);
        for (int64_t i = 0; i < nq; i++) {
            if (ks[i] < 1) fail(GTS_EINVAL, "k must be >= 1");
            hk[(size_t)i] = (int32_t)std::min<int64_t>(ks[i], (1ll << 31) - 1);
        }
        s.ks.alloc((size_t)std::max<int64_t>(nq, 1), st);
        h2d(s.ks.p, pa.stage(hk.data(), (size_t)nq), (size_t)nq, st);
        // +inf until the probe (if any) estimates a radius
        std::vector<float> inf32((size_t)nq, INFINITY);
        std::vector<double> inf64((size_t)nq, INFINITY);
        h2d(s.r32.p, pa.stage(inf32.data(), (size_t)nq), (size_t)nq, st);
        h2d(s.r64.p, pa.stage(inf64.data(), (size_t)nq), (size_t)nq, st);
    }
    const double t1 = trace ? now_ms() : 0.0;
    s.use_cache = use_cache;
    s.ext_bound = mode == 1 ? ext_bound : nullptr;
    s.probe_out = mode == 1 ? probe_out : nullptr;
    s.run();
    if (s.probe_out) {
        if (!pruning || ix->levels == 0 || ix->n == 0) {
            std::vector<float> inf32((size_t)nq, INFINITY);
            h2d(probe_out, inf32.data(), (size_t)nq, st);
        }
        CK(cudaStreamSynchronize(st));
        return nullptr;
    }
    s.scan_cache();
    const double t2 = trace ? now_ms() : 0.0;
    {
        const unsigned long long want = s.hits + s.hits / 4;
        unsigned long long cur = ix->hit_hint[mode].load();
        while (want > cur && !ix->hit_hint[mode].compare_exchange_weak(cur, want)) {}
        if (nq > 0) {
            const double hpq = (double)s.hits / (double)nq;
            double c0 = g_hits_per_query[mode].load();
            while (hpq > c0 && !g_hits_per_query[mode].compare_exchange_weak(c0, hpq)) {}
        }
    }
    auto *res = new gts_result();
    try {
        s.collect(res);
    } catch (...) {
        delete res;
        throw;
    }
    if (trace) {
        const double t3 = now_ms();
        fprintf(stderr, "[gts] %s nq=%lld setup=%.2fms run=%.2fms collect=%.2fms hits=%llu reruns=%d\n",
                mode ? "knn" : "range", (long long)nq, t1 - t0, t2 - t1, t3 - t2, (unsigned long long)s.hits,
                s.reruns);
        if (g_phase_dev) {
            unsigned long long ph[3];
            cudaMemcpy(ph, g_phase_dev, sizeof(ph), cudaMemcpyDeviceToHost);
            cudaMemset(g_phase_dev, 0, 3 * sizeof(unsigned long long));
            const double tot = (double)(ph[0] + ph[1] + ph[2]) + 1e-9;
            fprintf(stderr, "[gts]   mma phases (CTA clocks): stage %.3f  mma-wait %.3f  epilogue %.3f\n",
                    ph[0] / tot, ph[1] / tot, ph[2] / tot);
        }
    }
    return res;
}

}  // namespace

// Device slot layout: every leaf keeps its reference entries in order,
// followed by free slots for in-place inserts (leaf slack: size/8, at least
// 4, none for empty leaves; GTS_LEAF_SLACK=<d> sets size/d, 0 = none).
// Internal nodes span their leaves' slots.
struct SlotLayout {
    std::vector<int64_t> dpos, span;   // per node: first slot, slot count (leaves: capacity)
    int64_t n_slots = 0;
};

SlotLayout slot_layout(const gts_tree *t)
{
    SlotLayout L;
    L.dpos.assign((size_t)t->nodes + 1, 0);
    L.span.assign((size_t)t->nodes + 1, 0);
    static const int den = std::getenv("GTS_LEAF_SLACK") ? std::atoi(std::getenv("GTS_LEAF_SLACK")) : 8;
    __int128 c = 1;
    for (int64_t l = 1; l < t->levels; l++) c *= t->nc;
    const int64_t lfirst = (int64_t)((c - 1) / (t->nc - 1) + 1), lcount = (int64_t)c;
    int64_t p = 0;
    for (int64_t i = lfirst; i < lfirst + lcount; i++) {
        const int64_t sz = t->size[i];
        const int64_t cap = (sz > 0 && den > 0) ? sz + std::max<int64_t>(4, sz / den) : sz;
        L.dpos[(size_t)i] = p;
        L.span[(size_t)i] = cap;
        p += cap;
    }
    L.n_slots = p;
    for (int64_t level = t->levels - 1; level >= 1; level--) {
        __int128 cc = 1;
        for (int64_t l = 1; l < level; l++) cc *= t->nc;
        const int64_t first = (int64_t)((cc - 1) / (t->nc - 1) + 1), count = (int64_t)cc;
        for (int64_t v = first; v < first + count; v++) {
            const int64_t c0 = (v - 1) * t->nc + 2;
            L.dpos[(size_t)v] = L.dpos[(size_t)c0];
            int64_t sp = 0;
            for (int64_t j = 0; j < t->nc; j++) sp += L.span[(size_t)(c0 + j)];
            L.span[(size_t)v] = sp;
        }
    }
    return L;
}

// reference-position order (ord[k] for reference slot k) -> slot order
// (ord_s[e] = reference position of slot e, -1 for a free slot)
std::vector<int64_t> slot_order(const gts_tree *t, const SlotLayout &L, const std::vector<int64_t> &ord)
{
    std::vector<int64_t> os((size_t)L.n_slots, -1);
    __int128 c = 1;
    for (int64_t l = 1; l < t->levels; l++) c *= t->nc;
    const int64_t lfirst = (int64_t)((c - 1) / (t->nc - 1) + 1), lcount = (int64_t)c;
    #pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = lfirst; i < lfirst + lcount; i++)
        for (int64_t k = 0; k < t->size[i]; k++) os[(size_t)(L.dpos[(size_t)i] + k)] = ord[(size_t)(t->pos[i] + k)];
    return os;
}

// The tables every index has, from the host tree arrays (reference
// tree.py:155-175): node records with fp32 ranges rounded outward, node
// positions, live leaves, entry rows / pivot distances / ids / alive bits
// in device slot order (ord[e] = reference table position of slot e, -1 =
// free slot).  Leaf records carry their entry count, internal ones their
// slot span (> 0 iff the node holds entries).
void upload_tables(gts_index *ix, const gts_tree *t, const std::vector<int64_t> &ord, const int64_t *row_ids,
                   cudaStream_t st, std::vector<int64_t> &drow, std::vector<NodeRec> &nodes, const SlotLayout &lay)
{
    const int64_t n = (int64_t)ord.size();
    ix->n = n;
    ix->n_ref = t->n;
    drow.assign((size_t)n, -1);
    std::vector<int32_t> tpos((size_t)t->n, -1);
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; e++) drow[(size_t)e] = ord[(size_t)e] >= 0 ? t->rows[ord[(size_t)e]] : -1;
    ix->ord = ord;
    #pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < n; e++)
        if (drow[(size_t)e] >= 0) tpos[(size_t)drow[(size_t)e]] = (int32_t)e;
    __int128 c = 1;
    for (int l = 1; l < ix->levels; l++) c *= ix->nc;
    const int64_t lfirst = (int64_t)((c - 1) / (ix->nc - 1) + 1), lcount = (int64_t)c;
    nodes.assign((size_t)t->nodes + 1, NodeRec{});
    std::vector<int32_t> npos((size_t)t->nodes + 1);
    for (int64_t i = 0; i <= t->nodes; i++) {
        NodeRec r;
        float mn = (float)t->min_dis[i], mx = (float)t->max_dis[i];
        if ((double)mn > t->min_dis[i]) mn = std::nextafter(mn, -INFINITY);
        if ((double)mx < t->max_dis[i]) mx = std::nextafter(mx, INFINITY);
        r.mn = mn;
        r.mx = mx;
        const bool leaf = i >= lfirst && i < lfirst + lcount;
        r.size = (int32_t)(leaf ? t->size[i] : lay.span[(size_t)i]);
        r.piv = t->pivot_row[i] >= 0 ? tpos[(size_t)t->pivot_row[i]] : -1;
        nodes[(size_t)i] = r;
        npos[(size_t)i] = (int32_t)lay.dpos[(size_t)i];
    }
    ix->h_nodes = nodes;
    ix->node.alloc(nodes.size(), st);
    h2d(ix->node.p, nodes.data(), nodes.size(), st);
    ix->npos.alloc(npos.size(), st);
    h2d(ix->npos.p, npos.data(), npos.size(), st);
    // live leaves (for pruning-disabled scans); the largest leaf capacity
    {
        std::vector<int32_t> lv;
        ix->leaf_dpos.assign((size_t)lcount, 0);
        ix->leaf_cap.assign((size_t)lcount, 0);
        ix->leaf_size.assign((size_t)lcount, 0);
        for (int64_t i = lfirst; i < lfirst + lcount; i++) {
            if (t->size[i] > 0) lv.push_back((int32_t)i);
            ix->max_leaf = std::max<int>(ix->max_leaf, (int)lay.span[(size_t)i]);
            ix->leaf_dpos[(size_t)(i - lfirst)] = lay.dpos[(size_t)i];
            ix->leaf_cap[(size_t)(i - lfirst)] = lay.span[(size_t)i];
            ix->leaf_size[(size_t)(i - lfirst)] = t->size[i];
        }
        ix->n_live_leaves = (int)lv.size();
        ix->live_leaves.alloc(std::max<size_t>(lv.size(), 1), st);
        h2d(ix->live_leaves.p, lv.data(), lv.size(), st);
        ix->leaf_first = (int)lfirst;
        ix->leaf_count = (int)lcount;
    }
    {
        std::vector<int32_t> row((size_t)n);
        #pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < n; e++) row[(size_t)e] = (int32_t)drow[(size_t)e];
        ix->row.alloc((size_t)n, st);
        h2d(ix->row.p, row.data(), (size_t)n, st);
    }
    std::vector<float> dis((size_t)n);
    std::vector<int64_t> ids((size_t)n);
    std::vector<uint32_t> alive((size_t)((n + 31) / 32), 0u);
    #pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < (n + 31) / 32; w++) {
        uint32_t bits = 0;
        for (int64_t e = w * 32; e < std::min<int64_t>(n, w * 32 + 32); e++) {
            const int64_t o = ord[(size_t)e];
            if (o < 0) {
                dis[(size_t)e] = NAN;
                ids[(size_t)e] = -1;
                continue;
            }
            dis[(size_t)e] = (float)t->dis[o];
            ids[(size_t)e] = row_ids[drow[(size_t)e]];
            if (!t->tombstone || t->tombstone[o] == 0) bits |= 1u << (e & 31);
        }
        alive[(size_t)w] = bits;
    }
    ix->h_alive = alive;
    ix->dis.alloc((size_t)n, st);
    h2d(ix->dis.p, dis.data(), (size_t)n, st);
    ix->ids.alloc((size_t)n, st);
    h2d(ix->ids.p, ids.data(), (size_t)n, st);
    ix->alive.alloc(alive.size(), st);
    h2d(ix->alive.p, alive.data(), alive.size(), st);
}

// Device memory pool of an index's device: keep freed blocks mapped and
// map a large block once (see below).
void prime_pool(int device)
{
    // search scratch comes from the device's default stream-ordered pool;
    // keep freed blocks mapped between calls instead of unmapping them at
    // every synchronisation (release threshold 0 is the CUDA default)
    CK(cudaSetDevice(device));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        // Prime the pool once: map a large block up front so batch-sized
        // scratch (frontier tables, hit / candidate buffers, sort space:
        // GBs for 100k-query kNN) is carved from mapped memory instead of
        // growing the pool -- mapping new physical memory mid-call costs
        // 100s of ms.  GTS_POOL_PRIME_GB overrides (0 = off).
        const char *env = std::getenv("GTS_POOL_PRIME_GB");
        size_t free_b = 0, total_b = 0;
        cudaMemGetInfo(&free_b, &total_b);
        size_t want = env ? (size_t)std::atoll(env) << 30 : std::min<size_t>((size_t)24 << 30, total_b / 6);
        uint64_t reserved = 0;
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved);
        if (want > reserved && want < free_b / 2) {
            void *p = nullptr;
            if (cudaMallocAsync(&p, want, 0) == cudaSuccess) {
                cudaFreeAsync(p, 0);
                cudaStreamSynchronize(0);
            }
            cudaGetLastError();
        }
    }
}

// fp32 radius of the collection around the root pivot (k_root_radius):
// the root pivot's payload is uploaded as a one-row query batch.
void compute_root_radius(gts_index *ix, const gts_dataset *ds, const gts_tree *t, cudaStream_t st);

void root_radius_of(gts_index *ix, std::vector<double> payload, cudaStream_t st)
{
    ix->root_payload = std::move(payload);
    gts_query_batch qb{ix->metric, 1, ix->D, ix->root_payload.data(), nullptr, nullptr};
    gts_queries *q = upload_queries(ix, &qb, st);
    DBuf<unsigned> m(1, st);
    CK(cudaMemsetAsync(m.p, 0, sizeof(unsigned), st));
    const IndexView iv = make_view(ix, q);
    const QueryView qv = make_qview(ix, q);
    const unsigned grid = grid_for(ix->n, 256, 148u * 8u);
    switch (ix->metric) {
    case GTS_L1: k_root_radius<kMetricL1><<<grid, 256, 0, st>>>(iv, qv, ix->n, m.p); break;
    case GTS_ANGULAR: k_root_radius<kMetricAngular><<<grid, 256, 0, st>>>(iv, qv, ix->n, m.p); break;
    default: k_root_radius<kMetricL2><<<grid, 256, 0, st>>>(iv, qv, ix->n, m.p); break;
    }
    LAUNCH_CHECK();
    unsigned h = 0;
    CK(cudaMemcpyAsync(&h, m.p, sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    delete q;
    float r;
    std::memcpy(&r, &h, sizeof(r));
    ix->root_radius = r;
}

void compute_root_radius(gts_index *ix, const gts_dataset *ds, const gts_tree *t, cudaStream_t st)
{
    const int64_t prow = t->pivot_row[1];
    if (prow < 0 || prow >= ds->n) return;
    root_radius_of(ix, std::vector<double>(ds->vectors + prow * ix->D, ds->vectors + (prow + 1) * ix->D), st);
}

// float64 radius of the pending cache around the root pivot, rounded up
double host_metric(int metric, const double *a, const double *b, int64_t D)
{
    double acc = 0.0;
    if (metric == GTS_L1) {
        for (int64_t i = 0; i < D; i++) acc += std::fabs(a[i] - b[i]);
        return acc;
    }
    if (metric == GTS_L2) {
        for (int64_t i = 0; i < D; i++) acc += (a[i] - b[i]) * (a[i] - b[i]);
        return std::sqrt(acc);
    }
    double na = 0.0, nb = 0.0;
    for (int64_t i = 0; i < D; i++) { acc += a[i] * b[i]; na += a[i] * a[i]; nb += b[i] * b[i]; }
    if (na == 0.0 || nb == 0.0) return M_PI;
    return std::acos(std::max(-1.0, std::min(1.0, acc / std::sqrt(na * nb))));
}

// ===========================================================================
// C ABI
// ===========================================================================
#define ABI_BEGIN try {
#define ABI_END                                                                          \
    }                                                                                    \
    catch (const Error &e) { return e.code; }                                            \
    catch (const std::bad_alloc &) { return set_error(GTS_EOOM, "host allocation failed"); } \
    catch (...) { return set_error(GTS_EINVAL, "unexpected C++ exception"); }

extern "C" const char *gts_last_error(void) { return g_err; }
extern "C" const char *gts_version(void) { return "gts-b200 0.1 sm_100a"; }
extern "C" int64_t gts_launch_count(void) { return g_launches.load(); }
extern "C" int gts_device_count(void)
{
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

extern "C" int gts_profile_enable(int on)
{
    g_profile.store(on ? 1 : 0);
    return GTS_OK;
}

extern "C" int gts_profile_read(char *buf, int64_t cap, int reset)
{
    std::lock_guard<std::mutex> g(g_prof_mu);
    std::string js = "{\"kernels\": {";
    bool first = true;
    for (auto &kv : g_prof) {
        char tmp[256];
        snprintf(tmp, sizeof(tmp), "%s\"%s\": {\"count\": %lld, \"ms\": %.6f}", first ? "" : ", ", kv.first.c_str(),
                 (long long)kv.second.count, kv.second.ms);
        js += tmp;
        first = false;
    }
    char tmp[256];
    snprintf(tmp, sizeof(tmp), "}, \"work\": {\"pairs\": %llu, \"word_steps\": %llu, \"entries\": %llu, \"rows\": %llu}",
             g_work[0], g_work[1], g_work[2], g_work[3]);
    js += tmp;
    snprintf(tmp, sizeof(tmp),
             ", \"expand\": {\"bytes\": %.0f, \"rows_in\": %.0f, \"rows_out\": %.0f, \"evaluated\": %.0f}}",
             g_expand[0], g_expand[1], g_expand[2], g_expand[3]);
    js += tmp;
    if (reset) {
        g_prof.clear();
        for (auto &w : g_work) w = 0;
        for (auto &w : g_expand) w = 0;
    }
    if (!buf || cap <= (int64_t)js.size()) return set_error(GTS_EINVAL, "profile buffer too small (%zu)", js.size());
    std::memcpy(buf, js.c_str(), js.size() + 1);
    return GTS_OK;
}

// Integer peak microbenchmarks: 16 chains per thread (enough ILP that issue,
// not latency, bounds them).  Variant 0: LOP3 only (alu pipe); 1: IMAD only
// (fma pipe); 2: alternating LOP3 / IMAD (both pipes).  Each op reads a
// neighbouring chain through inline PTX, so neither NVVM nor ptxas can fold
// iterations together (a self-contained (a^b)|c or a*m+b chain has a closed
// form and was collapsed).  The reported peak is the best variant, in
// executed integer instructions (thread-ops) per second.
__device__ __forceinline__ uint32_t lop3_xor3(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c)
{
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

template <int VAR>
__global__ void k_int_peak(uint32_t seed, uint32_t mul, int iters, uint32_t *sink)
{
    uint32_t a[16];
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = seed ^ (threadIdx.x * 2654435761u + i * 40503u);
    const uint32_t c = seed * 7u + mul;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (VAR == 0 || (VAR == 2 && (i & 1) == 0)) a[i] = lop3_xor3(a[i], a[(i + 1) & 15], c);   // 1 LOP3
            else a[i] = mad_lo(a[i], a[(i + 1) & 15], c);                                                // 1 IMAD
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 16; i++) r ^= a[i];
    if (r == 0x9e3779b9u) sink[0] = r;
}

template <int VAR>
static double int_peak_variant(cudaStream_t st, int blocks, uint32_t *sink)
{
    const int iters = 2048, block = 256;
    k_int_peak<VAR><<<blocks, block, 0, st>>>(1u, 0x9e3779b1u, 32, sink);   // warm-up
    LAUNCH_CHECK();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    k_int_peak<VAR><<<blocks, block, 0, st>>>(1u, 0x9e3779b1u, iters, sink);
    LAUNCH_CHECK();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (double)blocks * block * iters * 16 / (ms * 1e-3);
}

// FP32 pipe: 16 independent FADD (VAR 0) or FFMA (VAR 1) chains per thread
template <int VAR>
__global__ void k_fp32_peak(float seed, int iters, float *sink)
{
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; i++) a[i] = seed + (float)(threadIdx.x * 16 + i) * 1e-7f;
    const float c = seed * 0.5f;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (VAR == 0) a[i] = __fadd_rn(a[i], a[(i + 1) & 15]);
            else a[i] = __fmaf_rn(a[i], c, a[(i + 1) & 15]);
        }
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 16; i++) r += a[i];
    if (r == 1.2345f) sink[0] = r;
}

template <int VAR>
static double fp32_peak_variant(cudaStream_t st, int blocks, float *sink)
{
    const int iters = 2048, block = 256;
    k_fp32_peak<VAR><<<blocks, block, 0, st>>>(1e-9f, 32, sink);   // warm-up
    LAUNCH_CHECK();
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaEventRecord(a, st));
    k_fp32_peak<VAR><<<blocks, block, 0, st>>>(1e-9f, iters, sink);
    LAUNCH_CHECK();
    CK(cudaEventRecord(b, st));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return (double)blocks * block * iters * 16 / (ms * 1e-3);
}

// FP32 lane-operation throughput (FADD / FFMA instructions x 32 lanes per
// second), the denominator of the CUDA-core distance kernels' rooflines
extern "C" int gts_bench_fp32_peak(double *ops_per_s, void *stream)
{
    ABI_BEGIN
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<float> sink(1, st);
    const int blocks = sms * 8;
    ops_per_s[0] = std::max(fp32_peak_variant<0>(st, blocks, sink.p), fp32_peak_variant<1>(st, blocks, sink.p));
    return GTS_OK;
    ABI_END
}

extern "C" int gts_bench_int_peak(double *ops_per_s, void *stream)
{
    ABI_BEGIN
    cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    DBuf<uint32_t> sink(1, st);
    const int blocks = sms * 8;
    const double v0 = int_peak_variant<0>(st, blocks, sink.p);
    const double v1 = int_peak_variant<1>(st, blocks, sink.p);
    const double v2 = int_peak_variant<2>(st, blocks, sink.p);
    ops_per_s[0] = std::max(v0, std::max(v1, v2));
    return GTS_OK;
    ABI_END
}

extern "C" int gts_index_create(const gts_dataset *ds, const gts_tree *t, int device, gts_index **out)
{
    ABI_BEGIN
    static const bool trace = std::getenv("GTS_TRACE") != nullptr;
    const double c0 = trace ? now_ms() : 0.0;
    prime_pool(device);
    const double c1 = trace ? now_ms() : 0.0;
    if (!ds || !t || !out) fail(GTS_EINVAL, "null argument");
    if (ds->metric != GTS_EDIT && ds->metric != GTS_L1 && ds->metric != GTS_L2 && ds->metric != GTS_ANGULAR)
        fail(GTS_EMETRIC, "metric %d not supported on the device path (edit, l1, l2, angular)", ds->metric);
    if (ds->n > (1ll << 31) - 64) fail(GTS_EINVAL, "index larger than 2^31 entries; shard it");
    CK(cudaSetDevice(device));
    if (std::getenv("GTS_PHASES") && !g_phase_dev) {
        CK(cudaMalloc((void **)&g_phase_dev, 4 * sizeof(unsigned long long)));
        CK(cudaMemset(g_phase_dev, 0, 4 * sizeof(unsigned long long)));
    }
    {
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t thr = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    auto *ix = new gts_index();
    try {
        cudaStream_t st = 0;
        ix->device = device;
        ix->metric = ds->metric;
        ix->n = ds->n;
        ix->nc = (int)t->nc;
        ix->levels = (int)t->levels;
        ix->split_rounds = (int)t->split_rounds;
        ix->nodes = t->nodes;
        const int64_t n = ds->n;
        if (n == 0 || t->levels == 0) { *out = ix; return GTS_OK; }
        // Device table order: the reference table order, except that string
        // entries are stably sorted by length inside each leaf (leaves are
        // scanned, never ordered, search.py:518-524), so DP lanes of a warp
        // see similar lengths.  ord[e] = reference position of device entry e.
        std::vector<int64_t> ord((size_t)n);
        for (int64_t e = 0; e < n; e++) ord[(size_t)e] = e;
        {
            // strings: by length (DP lanes see similar lengths).  (Vector leaves
            // sorted by pivot distance, with rows ranked by dqp and warp-uniform
            // skipping of 32-entry blocks outside the rows' lemma-1 windows in
            // k_leafgroup_tile: no change on the L1 shard, 441 vs 430 ms --
            // the windows of 16 rows cover whole leaves.)
            __int128 c = 1;
            for (int l = 1; l < ix->levels; l++) c *= ix->nc;
            const int64_t lfirst = (int64_t)((c - 1) / (ix->nc - 1) + 1), lcount = (int64_t)c;
            for (int64_t i = lfirst; i < lfirst + lcount; i++) {
                const int64_t p0 = t->pos[i], sz = t->size[i];
                if (sz <= 1) continue;
                if (ds->metric == GTS_EDIT)
                    std::stable_sort(ord.begin() + p0, ord.begin() + p0 + sz, [&](int64_t a, int64_t b) {
                        const int64_t ra = t->rows[a], rb = t->rows[b];
                        return ds->offsets[ra + 1] - ds->offsets[ra] < ds->offsets[rb + 1] - ds->offsets[rb];
                    });
            }
        }
        // every leaf is followed by free slots (leaf slack) for in-place inserts
        const SlotLayout lay = slot_layout(t);
        ord = slot_order(t, lay, ord);
        const int64_t ns = lay.n_slots;
        std::vector<int64_t> drow;
        std::vector<NodeRec> nodes;
        upload_tables(ix, t, ord, ds->ids, st, drow, nodes, lay);
        const double c2 = trace ? now_ms() : 0.0;
        if (ds->metric == GTS_EDIT) {
            const int64_t ncodes = ds->offsets[n];
            std::vector<int32_t> alpha;
            dense_alphabet(ds->codes, ncodes, alpha);   // builder.cpp: no sort of every code
            if (alpha.size() > 254)
                fail(GTS_EMETRIC, "string alphabet of %zu symbols exceeds the device's 254", alpha.size());
            ix->A = (int)alpha.size();
            ix->h_alpha = alpha;
            int64_t maxlen = 0;
            for (int64_t r = 0; r < n; r++) maxlen = std::max<int64_t>(maxlen, ds->offsets[r + 1] - ds->offsets[r]);
            // a free slot reserves room for a string as long as the longest stored one
            ix->slot_words = (int)(((maxlen + 15) / 16) * 4);
            std::vector<uint32_t> words, wstart;
            std::vector<int32_t> lens;
            const SymMap smap(alpha);
            auto symof = [&](int64_t k) { return smap(ds->codes[k]); };
            pack_words(ns, ds->offsets, symof, words, wstart, lens, drow.data(), ix->slot_words);
            for (auto l : lens) ix->max_len = std::max<int>(ix->max_len, l);
            ix->alpha.alloc(std::max<size_t>(alpha.size(), 1), st);
            h2d(ix->alpha.p, alpha.data(), alpha.size(), st);
            ix->str.alloc(words.size(), st);
            h2d(ix->str.p, words.data(), words.size(), st);
            ix->avg_text_bytes = 4.0 * (double)words.size() / (double)std::max<int64_t>(n, 1);
            ix->h_sword = wstart;
            ix->sword.alloc(wstart.size(), st);
            h2d(ix->sword.p, wstart.data(), wstart.size(), st);
            ix->slen.alloc(lens.size(), st);
            h2d(ix->slen.p, lens.data(), lens.size(), st);
            ix->h_slen = lens;
            std::vector<uint4> rec((size_t)ns);
            #pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < ns; e++) {
                const float d = ord[(size_t)e] >= 0 ? (float)t->dis[ord[(size_t)e]] : NAN;
                uint32_t db;
                std::memcpy(&db, &d, 4);
                const float lf = (float)lens[(size_t)e];
                uint32_t lb;
                std::memcpy(&lb, &lf, 4);
                rec[(size_t)e] = make_uint4(db, (uint32_t)lens[(size_t)e], wstart[(size_t)e], lb);
            }
            for (int64_t i = ix->leaf_first; i < (int64_t)ix->leaf_first + ix->leaf_count; i++) {
                if (lay.span[(size_t)i] <= 0) continue;
                const int64_t a = lay.dpos[(size_t)i], b = a + lay.span[(size_t)i] - 1;
                const int64_t wend = (int64_t)wstart[(size_t)b] + std::max<int64_t>(((lens[(size_t)b] + 15) / 16) * 4,
                                                                                  ord[(size_t)b] < 0 ? ix->slot_words : 0);
                ix->max_leaf_words = std::max<int>(ix->max_leaf_words, (int)std::min<int64_t>(wend - wstart[(size_t)a], 1 << 30));
            }
            ix->erec.alloc(rec.size(), st);
            h2d(ix->erec.p, rec.data(), rec.size(), st);
            k_erec_alive<<<grid_for(ns, 256), 256, 0, st>>>(ix->erec.p, ix->dis.p, ix->alive.p, ns);
            LAUNCH_CHECK();
            if (ix->A <= 16 && std::getenv("GTS_NO_QSIG") == nullptr) {
                // q-gram signatures of every slot (free slots: the empty set)
                ix->esig.alloc((size_t)ns * 2, st);
                CK(cudaMemsetAsync(ix->esig.p, 0, sizeof(uint4) * 2 * (size_t)ns, st));
                k_slot_sig<<<grid_for(ns, 128), 128, 0, st>>>(ix->str.p, ix->sword.p, ix->slen.p, nullptr, ns, ix->A,
                                                              ix->esig.p);
                LAUNCH_CHECK();
            }
            if (ix->A > kHistMinAlphabet) {
                // 32 byte-buckets of symbol counts per entry (saturating)
                std::vector<uint8_t> hb((size_t)ns * 32, 0);
                #pragma omp parallel for schedule(static, 4096)
                for (int64_t e = 0; e < ns; e++) {
                    const int64_t r = drow[(size_t)e];
                    if (r < 0) continue;
                    uint8_t *h = hb.data() + e * 32;
                    for (int64_t k = ds->offsets[r]; k < ds->offsets[r + 1]; k++) {
                        const int sym = (int)(std::lower_bound(alpha.begin(), alpha.end(), ds->codes[k]) - alpha.begin());
                        uint8_t &c = h[sym & 31];
                        if (c < 255) c++;
                    }
                }
                ix->ehist.alloc((size_t)ns * 2, st);
                CK(cudaMemcpyAsync(ix->ehist.p, hb.data(), hb.size(), cudaMemcpyHostToDevice, st));
                CK(cudaStreamSynchronize(st));
            }
        } else {
            ix->D = (int)ds->dim;
            ix->Dp = (ix->D + 3) & ~3;
            std::vector<float> v32((size_t)(ns * ix->Dp), 0.f);
            bool exact = true;
            float mx = 0.f;
            #pragma omp parallel for schedule(static, 4096) reduction(&& : exact) reduction(max : mx)
            for (int64_t e = 0; e < ns; e++) {
                if (drow[(size_t)e] < 0) continue;
                const double *src = ds->vectors + drow[(size_t)e] * ix->D;
                for (int d = 0; d < ix->D; d++) {
                    float f = (float)src[d];
                    if ((double)f != src[d]) exact = false;
                    mx = std::max(mx, std::fabs(f));
                    v32[(size_t)(e * ix->Dp + d)] = f;
                }
            }
            ix->data_exact = exact;
            ix->data_maxabs = mx;
            // tensor-core L2 path: entries centred on their leaf's pivot, bf16, K padded to 64
            if (ds->metric == GTS_L2 && ix->D >= 32 && ix->D <= 128 && ix->max_leaf <= 256 &&
                std::getenv("GTS_NO_MMA") == nullptr) {
                ix->Dk = (ix->D + 63) & ~63;
                std::vector<__nv_bfloat16> vc((size_t)ns * ix->Dk, __float2bfloat16(0.f));
                const int64_t lfirst = ix->leaf_first, lcount = ix->leaf_count;
                #pragma omp parallel for schedule(dynamic, 64)
                for (int64_t i = lfirst; i < lfirst + lcount; i++) {
                    const int64_t p0 = lay.dpos[(size_t)i], sz = t->size[i];
                    if (sz <= 0) continue;
                    const int pvp = nodes[(size_t)i].piv;
                    for (int64_t e = p0; e < p0 + sz; e++)
                        for (int d = 0; d < ix->D; d++)
                            vc[(size_t)e * ix->Dk + d] = __float2bfloat16(
                                v32[(size_t)(e * ix->Dp + d)] - v32[(size_t)((int64_t)pvp * ix->Dp + d)]);
                }
                // se_e = c . bf16(o_e - c): the pivot term of the uncentred
                // query product (k_leafgroup_mma2), from the same rounded values
                std::vector<float> se((size_t)ns, 0.f);
                #pragma omp parallel for schedule(dynamic, 64)
                for (int64_t i = lfirst; i < lfirst + lcount; i++) {
                    const int64_t p0 = lay.dpos[(size_t)i], sz = t->size[i];
                    if (sz <= 0) continue;
                    const int pvp = nodes[(size_t)i].piv;
                    for (int64_t e = p0; e < p0 + sz; e++) {
                        double acc = 0.0;
                        for (int d = 0; d < ix->D; d++)
                            acc += (double)v32[(size_t)((int64_t)pvp * ix->Dp + d)] *
                                   (double)__bfloat162float(vc[(size_t)e * ix->Dk + d]);
                        se[(size_t)e] = (float)acc;
                    }
                }
                // + 16 zero rows: k_leafgroup_mma2 pads a leaf to a multiple of
                // 16 rows and forms (never dereferences) those rows' addresses
                const size_t tail = (size_t)16 * ix->Dk / 8;
                ix->vcent.alloc(vc.size() / 8 + tail, st);
                CK(cudaMemcpyAsync(ix->vcent.p, vc.data(), vc.size() * sizeof(__nv_bfloat16), cudaMemcpyHostToDevice, st));
                CK(cudaMemsetAsync(ix->vcent.p + vc.size() / 8, 0, tail * sizeof(uint4), st));
                ix->vse.alloc((size_t)ns, st);
                h2d(ix->vse.p, se.data(), (size_t)ns, st);
                CK(cudaStreamSynchronize(st));
                build_vtile(ix, st);
            }
            if (ds->metric == GTS_ANGULAR) {
                std::vector<double> nrm((size_t)ns, 0.0), tmp;
                std::vector<float> nrm32((size_t)ns, 0.f);
                for (int64_t e = 0; e < ns; e++) {
                    if (drow[(size_t)e] < 0) continue;
                    nrm[(size_t)e] = host_norm(ds->vectors + drow[(size_t)e] * ix->D, ix->D, tmp);
                    nrm32[(size_t)e] = (float)nrm[(size_t)e];
                }
                ix->vnorm64.alloc((size_t)ns, st);
                h2d(ix->vnorm64.p, nrm.data(), (size_t)ns, st);
                ix->vnorm32.alloc((size_t)ns, st);
                h2d(ix->vnorm32.p, nrm32.data(), (size_t)ns, st);
                CK(cudaStreamSynchronize(st));
            }
            ix->vec32.alloc(v32.size(), st);
            h2d(ix->vec32.p, v32.data(), v32.size(), st);
            if (!exact) {
                std::vector<double> v64((size_t)(ns * ix->D), 0.0);
                #pragma omp parallel for schedule(static, 4096)
                for (int64_t e = 0; e < ns; e++)
                    if (drow[(size_t)e] >= 0)
                        std::memcpy(v64.data() + e * ix->D, ds->vectors + drow[(size_t)e] * ix->D, sizeof(double) * ix->D);
                ix->vec64.alloc(v64.size(), st);
                h2d(ix->vec64.p, v64.data(), v64.size(), st);
            }
        }
        CK(cudaStreamSynchronize(st));
        const double c3 = trace ? now_ms() : 0.0;
        if (ds->metric != GTS_EDIT && n > 0 && ix->levels > 0) compute_root_radius(ix, ds, t, st);
        if (trace)
            fprintf(stderr, "[gts] index_create n=%lld slots=%lld pool=%.1fms tables=%.1fms payload=%.1fms root=%.1fms\n",
                    (long long)n, (long long)ns, c1 - c0, c2 - c1, c3 - c2, now_ms() - c3);
        *out = ix;
        return GTS_OK;
    } catch (...) {
        delete ix;
        throw;
    }
    ABI_END
}

extern "C" int gts_index_destroy(gts_index *ix)
{
    ABI_BEGIN
    if (ix) {
        cudaSetDevice(ix->device);
        cudaDeviceSynchronize();
        delete ix;
    }
    return GTS_OK;
    ABI_END
}

extern "C" int gts_index_set_tombstones(gts_index *ix, const uint8_t *tomb, void *stream)
{
    ABI_BEGIN
    if (!ix || !tomb) fail(GTS_EINVAL, "null argument");
    if (ix->n == 0) return GTS_OK;
    CK(cudaSetDevice(ix->device));
    // reference entries follow `tomb`; slots filled by gts_index_insert keep
    // their own state (gts_index_erase)
    std::vector<uint32_t> &alive = ix->h_alive;
    #pragma omp parallel for schedule(static)
    for (int64_t w = 0; w < (ix->n + 31) / 32; w++) {
        uint32_t bits = alive[(size_t)w];
        for (int64_t e = w * 32; e < std::min<int64_t>(ix->n, w * 32 + 32); e++) {
            const int64_t o = ix->ord[(size_t)e];
            if (o < 0) continue;
            const uint32_t b = 1u << (e & 31);
            bits = tomb[o] == 0 ? (bits | b) : (bits & ~b);
        }
        alive[(size_t)w] = bits;
    }
    cudaStream_t st = (cudaStream_t)stream;
    h2d(ix->alive.p, alive.data(), alive.size(), st);
    if (ix->erec.p) {
        k_erec_alive<<<grid_for(ix->n, 256), 256, 0, st>>>(ix->erec.p, ix->dis.p, ix->alive.p, ix->n);
        LAUNCH_CHECK();
    }
    CK(cudaStreamSynchronize(st));
    return GTS_OK;
    ABI_END
}

extern "C" int gts_queries_upload(gts_index *ix, const gts_query_batch *qb, void *stream, gts_queries **out)
{
    ABI_BEGIN
    if (!ix || !out) fail(GTS_EINVAL, "null argument");
    *out = upload_queries(ix, qb, (cudaStream_t)stream);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_queries_free(gts_queries *q)
{
    ABI_BEGIN
    delete q;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_range_batch(gts_index *ix, const gts_queries *q, const double *radii, int64_t memory_units,
                               int pruning, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!out || (!radii && q && q->nq)) fail(GTS_EINVAL, "null argument");
    *out = run_search(ix, q, 0, radii, nullptr, memory_units, pruning, (cudaStream_t)stream);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_knn_batch(gts_index *ix, const gts_queries *q, const int64_t *ks, int64_t memory_units,
                             int pruning, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!out || (!ks && q && q->nq)) fail(GTS_EINVAL, "null argument");
    *out = run_search(ix, q, 1, nullptr, ks, memory_units, pruning, (cudaStream_t)stream);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_knn_probe(gts_index *ix, const gts_queries *q, const int64_t *ks, void *stream, float *radius_out)
{
    ABI_BEGIN
    if (!ix || !q || !radius_out || (!ks && q->nq)) fail(GTS_EINVAL, "null argument");
    run_search(ix, q, 1, nullptr, ks, 0, 1, (cudaStream_t)stream, false, nullptr, radius_out);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_knn_batch_bounded(gts_index *ix, const gts_queries *q, const int64_t *ks, const float *radius,
                                     int64_t memory_units, int flags, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!out || (!ks && q && q->nq)) fail(GTS_EINVAL, "null argument");
    *out = run_search(ix, q, 1, nullptr, ks, memory_units, (flags & GTS_FLAG_PRUNING) ? 1 : 0, (cudaStream_t)stream,
                      (flags & GTS_FLAG_CACHE) != 0, radius, nullptr);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_range_batch_host(gts_index *ix, const gts_query_batch *qb, const double *radii,
                                    int64_t memory_units, int pruning, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!ix || !out) fail(GTS_EINVAL, "null argument");
    gts_queries *q = upload_queries(ix, qb, (cudaStream_t)stream);
    try {
        *out = run_search(ix, q, 0, radii, nullptr, memory_units, pruning, (cudaStream_t)stream);
    } catch (...) {
        delete q;
        throw;
    }
    delete q;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_knn_batch_host(gts_index *ix, const gts_query_batch *qb, const int64_t *ks,
                                  int64_t memory_units, int pruning, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!ix || !out) fail(GTS_EINVAL, "null argument");
    gts_queries *q = upload_queries(ix, qb, (cudaStream_t)stream);
    try {
        *out = run_search(ix, q, 1, nullptr, ks, memory_units, pruning, (cudaStream_t)stream);
    } catch (...) {
        delete q;
        throw;
    }
    delete q;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_batch_host(gts_index *ix, const gts_query_batch *qb, int mode, const double *radii,
                              const int64_t *ks, int64_t memory_units, int flags, void *stream, gts_result **out)
{
    ABI_BEGIN
    if (!ix || !out) fail(GTS_EINVAL, "null argument");
    if (mode != 0 && mode != 1) fail(GTS_EINVAL, "mode must be 0 (range) or 1 (knn)");
    gts_queries *q = upload_queries(ix, qb, (cudaStream_t)stream);
    try {
        *out = run_search(ix, q, mode, radii, ks, memory_units, (flags & GTS_FLAG_PRUNING) ? 1 : 0,
                          (cudaStream_t)stream, (flags & GTS_FLAG_CACHE) != 0);
    } catch (...) {
        delete q;
        throw;
    }
    delete q;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_index_cache_set(gts_index *ix, const gts_dataset *items, void *stream)
{
    ABI_BEGIN
    if (!ix || !items) fail(GTS_EINVAL, "null argument");
    CK(cudaSetDevice(ix->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = items->n;
    ix->cache_n = 0;
    ix->cache_max_len = 0;
    ix->cache_radius = 0.f;
    if (n == 0) return GTS_OK;
    if (n > (1 << 30)) fail(GTS_EINVAL, "cache too large");
    if (items->metric != ix->metric) fail(GTS_EMETRIC, "cache metric %d != index metric %d", items->metric, ix->metric);
    ix->cache_ids.alloc((size_t)n, st);
    h2d(ix->cache_ids.p, items->ids, (size_t)n, st);
    if (ix->metric == GTS_EDIT) {
        const auto &alpha = ix->h_alpha;
        bool missing = false;
        std::vector<uint32_t> words, wstart;
        std::vector<int32_t> lens;
        pack_words(n, items->offsets, [&](int64_t k) {
            auto it = std::lower_bound(alpha.begin(), alpha.end(), items->codes[k]);
            if (it == alpha.end() || *it != items->codes[k]) { missing = true; return 0u; }
            return (uint32_t)(it - alpha.begin());
        }, words, wstart, lens);
        if (missing) return set_error(GTS_EREBUILD, "cache holds a symbol outside the index alphabet");
        ix->cache_words.alloc(words.size(), st);
        h2d(ix->cache_words.p, words.data(), words.size(), st);
        ix->cache_sword.alloc(wstart.size(), st);
        h2d(ix->cache_sword.p, wstart.data(), wstart.size(), st);
        ix->cache_slen.alloc(lens.size(), st);
        h2d(ix->cache_slen.p, lens.data(), lens.size(), st);
        ix->cache_max_len = 0;
        for (auto l : lens) ix->cache_max_len = std::max<int>(ix->cache_max_len, l);
    } else {
        if (items->dim != ix->D) fail(GTS_EMETRIC, "cache dimensionality %lld != %d", (long long)items->dim, ix->D);
        ix->cache_vec64.alloc((size_t)(n * ix->D), st);
        h2d(ix->cache_vec64.p, items->vectors, (size_t)(n * ix->D), st);
        double cr = 0.0;
        if ((int64_t)ix->root_payload.size() == ix->D)
            for (int64_t i = 0; i < n; i++)
                cr = std::max(cr, host_metric(ix->metric, items->vectors + i * ix->D, ix->root_payload.data(), ix->D));
        else
            cr = INFINITY;
        ix->cache_radius = (float)(cr * (1.0 + 1e-6) + 1e-6);
    }
    CK(cudaStreamSynchronize(st));
    ix->cache_n = (int)n;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_result_info(const gts_result *r, int64_t *nq, int64_t *total, int64_t *peak, int64_t *limits)
{
    ABI_BEGIN
    if (!r) fail(GTS_EINVAL, "null result");
    if (nq) *nq = r->nq;
    if (total) *total = r->total;
    if (peak) *peak = r->peak;
    if (limits) std::memcpy(limits, r->limits, sizeof(r->limits));
    return GTS_OK;
    ABI_END
}

extern "C" int gts_result_copy(const gts_result *r, int64_t *offsets, int64_t *ids, double *dis, int64_t *verified,
                               int64_t *pruned, void *stream)
{
    ABI_BEGIN
    if (!r) fail(GTS_EINVAL, "null result");
    cudaStream_t st = (cudaStream_t)stream;
    if (offsets) CK(cudaMemcpyAsync(offsets, r->offsets.p, sizeof(int64_t) * (r->nq + 1), cudaMemcpyDefault, st));
    if (ids && r->total) CK(cudaMemcpyAsync(ids, r->ids.p, sizeof(int64_t) * r->total, cudaMemcpyDefault, st));
    if (dis && r->total) CK(cudaMemcpyAsync(dis, r->dis.p, sizeof(double) * r->total, cudaMemcpyDefault, st));
    if (verified && r->nq && r->verified.p)
        CK(cudaMemcpyAsync(verified, r->verified.p, sizeof(int64_t) * r->nq, cudaMemcpyDefault, st));
    if (pruned && r->nq && r->pruned.p)
        CK(cudaMemcpyAsync(pruned, r->pruned.p, sizeof(int64_t) * r->nq, cudaMemcpyDefault, st));
    if (verified && r->nq && !r->verified.p) std::memset(verified, 0, sizeof(int64_t) * r->nq);
    if (pruned && r->nq && !r->pruned.p) std::memset(pruned, 0, sizeof(int64_t) * r->nq);
    CK(cudaStreamSynchronize(st));
    return GTS_OK;
    ABI_END
}

extern "C" int gts_result_device(const gts_result *r, const int64_t **offsets, const int64_t **ids,
                                 const double **dis)
{
    ABI_BEGIN
    if (!r) fail(GTS_EINVAL, "null result");
    if (offsets) *offsets = r->offsets.p;
    if (ids) *ids = r->ids.p;
    if (dis) *dis = r->dis.p;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_result_free(gts_result *r)
{
    ABI_BEGIN
    delete r;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_pair_distances(int32_t metric, int64_t np, int64_t dim, const double *a_vec, const double *b_vec,
                                  const int32_t *a_codes, const int64_t *a_off, const int32_t *b_codes,
                                  const int64_t *b_off, double *out, void *stream)
{
    ABI_BEGIN
    cudaStream_t st = (cudaStream_t)stream;
    if (np == 0) return GTS_OK;
    if (metric == GTS_L1 || metric == GTS_L2 || metric == GTS_ANGULAR) {
        DBuf<double> a((size_t)(np * dim), st), b((size_t)(np * dim), st), o((size_t)np, st);
        h2d(a.p, a_vec, (size_t)(np * dim), st);
        h2d(b.p, b_vec, (size_t)(np * dim), st);
        k_pair_vec<<<grid_for(np, 128), 128, 0, st>>>(metric, np, (int)dim, a.p, b.p, o.p);
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(out, o.p, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return GTS_OK;
    }
    if (metric != GTS_EDIT) fail(GTS_EMETRIC, "metric %d not supported", metric);
    // shared dense alphabet of both sides
    const int64_t na = a_off[np], nb = b_off[np];
    std::vector<int32_t> alpha(a_codes, a_codes + na);
    alpha.insert(alpha.end(), b_codes, b_codes + nb);
    std::sort(alpha.begin(), alpha.end());
    alpha.erase(std::unique(alpha.begin(), alpha.end()), alpha.end());
    if (alpha.size() > 254) fail(GTS_EMETRIC, "alphabet too large");
    const int A = (int)alpha.size();
    std::vector<int64_t> peq_off((size_t)np + 1, 0);
    for (int64_t i = 0; i < np; i++) {
        int64_t m = a_off[i + 1] - a_off[i];
        if (m > 32 * kMaxWords && b_off[i + 1] - b_off[i] > 32 * kMaxWords)
            fail(GTS_EINVAL, "both strings of pair %lld longer than %d symbols", (long long)i, 32 * kMaxWords);
        peq_off[(size_t)i + 1] = peq_off[(size_t)i] + (int64_t)A * ((m + 31) / 32);
    }
    DBuf<int32_t> dalpha(std::max<size_t>(alpha.size(), 1), st);
    h2d(dalpha.p, alpha.data(), alpha.size(), st);
    DBuf<int32_t> ca((size_t)std::max<int64_t>(na, 1), st), cb((size_t)std::max<int64_t>(nb, 1), st);
    h2d(ca.p, a_codes, (size_t)na, st);
    h2d(cb.p, b_codes, (size_t)nb, st);
    DBuf<uint8_t> sa((size_t)std::max<int64_t>(na, 1), st);
    if (na) { k_map_symbols<<<grid_for(na, 256), 256, 0, st>>>(ca.p, na, dalpha.p, A, sa.p); LAUNCH_CHECK(); }
    std::vector<uint32_t> bw, bstart;
    std::vector<int32_t> blen;
    pack_words(np, b_off, [&](int64_t k) {
        return (uint32_t)(std::lower_bound(alpha.begin(), alpha.end(), b_codes[k]) - alpha.begin());
    }, bw, bstart, blen);
    DBuf<uint32_t> dbw(bw.size(), st), dbs(bstart.size(), st);
    DBuf<int32_t> dbl(blen.size(), st);
    h2d(dbw.p, bw.data(), bw.size(), st);
    h2d(dbs.p, bstart.data(), bstart.size(), st);
    h2d(dbl.p, blen.data(), blen.size(), st);
    DBuf<int64_t> aoff((size_t)np + 1, st), boff((size_t)np + 1, st), poff((size_t)np + 1, st);
    h2d(aoff.p, a_off, (size_t)np + 1, st);
    h2d(boff.p, b_off, (size_t)np + 1, st);
    h2d(poff.p, peq_off.data(), (size_t)np + 1, st);
    DBuf<uint32_t> peq((size_t)std::max<int64_t>(peq_off[(size_t)np], 1), st);
    CK(cudaMemsetAsync(peq.p, 0, sizeof(uint32_t) * peq.n, st));
    if (na) {
        k_build_peq<<<grid_for(na, 256), 256, 0, st>>>(sa.p, aoff.p, poff.p, (int)np, na, peq.p);
        LAUNCH_CHECK();
    }
    QueryView qa{};
    qa.soff = aoff.p;
    qa.str = sa.p;
    qa.peq = peq.p;
    qa.peq_off = poff.p;
    qa.A = A;
    DBuf<double> o((size_t)np, st);
    k_pair_edit<<<grid_for(np, 128), 128, 0, st>>>(np, dbw.p, dbs.p, dbl.p, qa, o.p);
    LAUNCH_CHECK();
    CK(cudaMemcpyAsync(out, o.p, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return GTS_OK;
    ABI_END
}

// multi-shard exchange + merge
#include "sharded.cuh"
// device bulk build
#include "devbuild.cuh"
// in-place inserts into leaf slack
#include "updates.cuh"
