// devbuild.cuh -- device bulk build of the flat pivot tree,
// included by engine.cu.
//
// Restates the reference construction (_Builder, tree.py:241-367) on the
// device and produces the same tree bit for bit as the host builder
// (builder.cpp) and the reference:
//   pivots ....... per node, the entry with the largest chain_min (running
//                  min of its distances to every ancestor pivot), smallest
//                  object id on ties (tree.py:293-310): one CUB segmented
//                  reduction per level over (chain bits, id, row)
//   map .......... float64 distance of every entry to its node's pivot in
//                  numpy's pairwise row-sum order (pw_sum64, as the search's
//                  exact recheck) or the exact edit distance (bit-parallel
//                  Myers/Hyyro, pattern = pivot): one thread per entry
//   sort ......... key = dis / (level max + 1) + node ordinal in float64
//                  (tree.py:122-135, 319-334), object id as the tie
//                  (runtime.py:149-185): two stable CUB radix sorts (id, then
//                  key bits -- the key is non-negative, so its IEEE bits
//                  order like its value)
//   split ........ children are fixed index ranges (size // N_c, the last
//                  child takes the rest, tree.py:336-354); their ranges are
//                  the first / last sorted distances (tree.py:361-367)
// Node positions and sizes depend only on n and N_c, so the host computes
// them; the device does everything that touches entries.

namespace {

struct PivCand {
    unsigned long long chain;   // float64 bits (chain_min >= 0)
    long long id;
    long long row;
};

struct PivMax {
    __device__ __forceinline__ PivCand operator()(const PivCand &a, const PivCand &b) const
    {
        if (a.chain != b.chain) return a.chain > b.chain ? a : b;
        return a.id <= b.id ? a : b;
    }
};

__global__ void k_b_iota(int32_t *rows, int64_t n)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) rows[i] = (int32_t)i;
}

__global__ void k_b_pivcand(const int32_t *__restrict__ rows, const double *__restrict__ chain,
                            const int64_t *__restrict__ ids, int64_t n, PivCand *out)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int32_t r = rows[e];
    out[e] = PivCand{(unsigned long long)__double_as_longlong(chain[e]), (long long)ids[r], (long long)r};
}

// entry -> ordinal of its node inside the level (segments tile [0, n))
__global__ void k_b_entry_node(const int64_t *__restrict__ seg_begin, int count, int64_t n, int32_t *node_of)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    int lo = 0, hi = count - 1;   // last segment with begin <= e (empty segments share a begin)
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (seg_begin[mid] <= e) lo = mid; else hi = mid - 1;
    }
    node_of[e] = lo;
}

// pivot payloads widened to float64 (the "query" side of pw_sum64)
__global__ void k_b_pivot_vec(const float *__restrict__ x32, const double *__restrict__ x64, int D,
                              const int32_t *__restrict__ prow, int count, double *p64)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= (int64_t)count * D) return;
    const int o = (int)(i / D), d = (int)(i - (int64_t)o * D);
    const int r = prow[o];
    p64[i] = r < 0 ? 0.0 : (x64 ? x64[(int64_t)r * D + d] : (double)x32[(int64_t)r * D + d]);
}

template <int MET>
__global__ void k_b_map_vec(const float *__restrict__ x32, const double *__restrict__ x64, int D,
                            const int32_t *__restrict__ rows, const int32_t *__restrict__ node_of,
                            const double *__restrict__ p64, int64_t n, double *dis)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int64_t r = rows[e];
    const double *q = p64 + (int64_t)node_of[e] * D;
    const double s = pw_sum64<MET>(x64 ? nullptr : x32 + r * D, x64 ? x64 + r * D : nullptr, q, 0, D);
    dis[e] = MET == kMetricL1 ? s : __dsqrt_rn(s);
}

// Myers masks of every pivot string: peq[o] = [A][W] words
__global__ void k_b_pivot_peq(const uint32_t *__restrict__ text, const uint32_t *__restrict__ sword,
                              const int32_t *__restrict__ slen, const int32_t *__restrict__ prow,
                              const int64_t *__restrict__ peq_off, int count, uint32_t *peq)
{
    const int o = blockIdx.x;
    if (o >= count) return;
    const int r = prow[o];
    if (r < 0) return;
    const int m = slen[r], W = (m + 31) >> 5;
    const uint32_t *t = text + sword[r];
    for (int j = threadIdx.x; j < m; j += blockDim.x) {
        const uint32_t c = (t[j >> 2] >> (8 * (j & 3))) & 0xffu;
        atomicOr(peq + peq_off[o] + (int64_t)c * W + (j >> 5), 1u << (j & 31));
    }
}

__global__ void k_b_map_edit(const uint32_t *__restrict__ text, const uint32_t *__restrict__ sword,
                             const int32_t *__restrict__ slen, const int32_t *__restrict__ rows,
                             const int32_t *__restrict__ node_of, const int32_t *__restrict__ prow,
                             const int64_t *__restrict__ peq_off, const uint32_t *__restrict__ peq, int64_t n,
                             double *dis)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int r = rows[e], o = node_of[e];
    dis[e] = (double)edit_peq(peq + peq_off[o], slen[prow[o]], text + sword[r], slen[r]);
}

__global__ void k_b_chain(const double *__restrict__ dis, int64_t n, int first, double *chain)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    chain[e] = first ? dis[e] : fmin(chain[e], dis[e]);
}

// sort keys: tie = object id, key = dis / denom + ordinal (float64, the
// reference's encode_keys, tree.py:130-135)
__global__ void k_b_keys(const double *__restrict__ dis, const int32_t *__restrict__ node_of,
                         const int32_t *__restrict__ rows, const int64_t *__restrict__ ids, double denom, int64_t n,
                         unsigned long long *key, unsigned long long *tie, int32_t *idx)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const double k = __dadd_rn(__ddiv_rn(dis[e], denom), (double)node_of[e]);
    key[e] = (unsigned long long)__double_as_longlong(k);
    tie[e] = (unsigned long long)ids[rows[e]];
    idx[e] = (int32_t)e;
}

__global__ void k_b_gather_key(const unsigned long long *__restrict__ key, const int32_t *__restrict__ idx,
                               int64_t n, unsigned long long *out)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) out[i] = key[idx[i]];
}

__global__ void k_b_permute(const int32_t *__restrict__ idx, const int32_t *__restrict__ rows,
                            const double *__restrict__ dis, const double *__restrict__ chain, int64_t n,
                            int32_t *rows2, double *dis2, double *chain2)
{
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int32_t j = idx[i];
    rows2[i] = rows[j];
    dis2[i] = dis[j];
    chain2[i] = chain[j];
}

// first / last distance of each (non-empty) segment
__global__ void k_b_ranges(const double *__restrict__ dis, const int64_t *__restrict__ pos,
                           const int64_t *__restrict__ size, int cnt, double *mn, double *mx)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cnt) return;
    if (size[i] > 0) {
        mn[i] = dis[pos[i]];
        mx[i] = dis[pos[i] + size[i] - 1];
    } else {
        mn[i] = 0.0;
        mx[i] = 0.0;
    }
}

// Device-resident build input.  Vectors: x32 ([n][D] float) or x64 ([n][D]
// double); strings: dense symbols 4 per word (text), word start and length
// per row.  ids: device [n].
struct BuildInput {
    int metric = 0;
    int64_t n = 0;
    int D = 0;
    const float *x32 = nullptr;
    const double *x64 = nullptr;
    const uint32_t *text = nullptr, *sword = nullptr;
    const int32_t *slen = nullptr;
    const int64_t *ids = nullptr;
    int A = 0;
    std::vector<int32_t> h_slen;   // host copy of the lengths (pattern sizes)
};

template <class T>
std::vector<T> d2h_vec(const T *p, size_t cnt, cudaStream_t st)
{
    std::vector<T> h(cnt);
    if (cnt) CK(cudaMemcpyAsync(h.data(), p, cnt * sizeof(T), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return h;
}

template <class T>
void h2d_vec(DBuf<T> &dst, const std::vector<T> &src, cudaStream_t st)
{
    dst.alloc(std::max<size_t>(src.size(), 1), st);
    h2d(dst.p, src.data(), src.size(), st);
}

// The build proper: fills the host tree arrays (t->nodes, nc set by the caller).
void device_build(const BuildInput &in, int64_t root_row, gts_tree *t, cudaStream_t st)
{
    const int64_t n = in.n, nc = t->nc;
    int64_t max_h, split;
    gts_tree_height(n, nc, &max_h, &split);
    t->split_rounds = split;
    t->levels = split + 1;
    const int64_t nodes = gts_node_count(t->levels, nc);
    if (t->nodes < nodes) fail(GTS_EINVAL, "tree arrays too small");
    for (int64_t i = 0; i <= nodes; i++) {
        t->pivot_id[i] = -1; t->pivot_row[i] = -1; t->min_dis[i] = 0; t->max_dis[i] = 0;
        t->pos[i] = 0; t->size[i] = 0;
    }
    t->size[1] = n;
    DBuf<int32_t> rows((size_t)n, st), rows2((size_t)n, st), node_of((size_t)n, st), idx((size_t)n, st),
        idx2((size_t)n, st);
    DBuf<double> dis((size_t)n, st), dis2((size_t)n, st), chain((size_t)n, st), chain2((size_t)n, st);
    DBuf<unsigned long long> key((size_t)n, st), key2((size_t)n, st), tie((size_t)n, st), tie2((size_t)n, st);
    const unsigned g = grid_for(n, 256);
    k_b_iota<<<g, 256, 0, st>>>(rows.p, n);
    LAUNCH_CHECK();
    size_t sort_bytes = 0, s2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, tie.p, tie2.p, idx.p, idx2.p, (int)n, 0, 64, st);
    cub::DeviceReduce::Max(nullptr, s2, dis.p, dis2.p, (int)n, st);
    DBuf<uint8_t> tmp(std::max(sort_bytes, s2), st);
    DBuf<double> dmax(1, st);
    for (int64_t level = 1; level <= t->levels; level++) {
        __int128 c = 1;
        for (int64_t l = 1; l < level; l++) c *= nc;
        const int count = (int)c;
        const int64_t first = (int64_t)((c - 1) / (nc - 1) + 1);
        std::vector<int64_t> hpos((size_t)count), hsize((size_t)count);
        for (int o = 0; o < count; o++) { hpos[(size_t)o] = t->pos[first + o]; hsize[(size_t)o] = t->size[first + o]; }
        DBuf<int64_t> dpos, dend;
        h2d_vec(dpos, hpos, st);
        k_b_entry_node<<<g, 256, 0, st>>>(dpos.p, count, n, node_of.p);
        LAUNCH_CHECK();
        // pivots
        std::vector<int32_t> hprow((size_t)count, -1);
        if (level == 1) {
            hprow[0] = (int32_t)root_row;   // rows are the identity at level 1
        } else {
            std::vector<int64_t> hend((size_t)count);
            for (int o = 0; o < count; o++) hend[(size_t)o] = hpos[(size_t)o] + hsize[(size_t)o];
            h2d_vec(dend, hend, st);
            DBuf<PivCand> cand((size_t)n, st), best((size_t)count, st);
            k_b_pivcand<<<g, 256, 0, st>>>(rows.p, chain.p, in.ids, n, cand.p);
            LAUNCH_CHECK();
            const PivCand ident{0ull, LLONG_MAX, -1};
            size_t rb = 0;
            cub::DeviceSegmentedReduce::Reduce(nullptr, rb, cand.p, best.p, count, dpos.p, dend.p, PivMax(), ident, st);
            DBuf<uint8_t> rt(rb, st);
            CK(cub::DeviceSegmentedReduce::Reduce(rt.p, rb, cand.p, best.p, count, dpos.p, dend.p, PivMax(), ident,
                                                  st));
            const std::vector<PivCand> hb = d2h_vec(best.p, (size_t)count, st);
            for (int o = 0; o < count; o++)
                if (hsize[(size_t)o] > 0) hprow[(size_t)o] = (int32_t)hb[(size_t)o].row;
        }
        DBuf<int32_t> dprow;
        h2d_vec(dprow, hprow, st);
        // map
        if (in.metric == GTS_EDIT) {
            std::vector<int64_t> poff((size_t)count + 1, 0);
            for (int o = 0; o < count; o++) {
                const int r = hprow[(size_t)o];
                const int64_t W = r >= 0 ? (in.h_slen[(size_t)r] + 31) / 32 : 0;
                poff[(size_t)o + 1] = poff[(size_t)o] + (int64_t)in.A * W;
            }
            DBuf<int64_t> dpoff;
            h2d_vec(dpoff, poff, st);
            DBuf<uint32_t> peq((size_t)std::max<int64_t>(poff[(size_t)count], 1), st);
            CK(cudaMemsetAsync(peq.p, 0, sizeof(uint32_t) * std::max<int64_t>(poff[(size_t)count], 1), st));
            k_b_pivot_peq<<<count, 128, 0, st>>>(in.text, in.sword, in.slen, dprow.p, dpoff.p, count, peq.p);
            LAUNCH_CHECK();
            k_b_map_edit<<<g, 256, 0, st>>>(in.text, in.sword, in.slen, rows.p, node_of.p, dprow.p, dpoff.p, peq.p, n,
                                            dis.p);
            LAUNCH_CHECK();
        } else {
            DBuf<double> p64((size_t)count * in.D, st);
            k_b_pivot_vec<<<grid_for((int64_t)count * in.D, 256), 256, 0, st>>>(in.x32, in.x64, in.D, dprow.p, count,
                                                                                p64.p);
            LAUNCH_CHECK();
            if (in.metric == GTS_L1)
                k_b_map_vec<kMetricL1><<<g, 256, 0, st>>>(in.x32, in.x64, in.D, rows.p, node_of.p, p64.p, n, dis.p);
            else
                k_b_map_vec<kMetricL2><<<g, 256, 0, st>>>(in.x32, in.x64, in.D, rows.p, node_of.p, p64.p, n, dis.p);
            LAUNCH_CHECK();
        }
        for (int o = 0; o < count; o++) {
            const int r = hprow[(size_t)o];
            if (r < 0) continue;
            t->pivot_row[first + o] = r;
        }
        k_b_chain<<<g, 256, 0, st>>>(dis.p, n, level == 1 ? 1 : 0, chain.p);
        LAUNCH_CHECK();
        // one global keyed sort over the level
        CK(cub::DeviceReduce::Max(tmp.p, s2, dis.p, dmax.p, (int)n, st));
        double lm = 0.0;
        CK(cudaMemcpyAsync(&lm, dmax.p, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double denom = lm + 1.0;
        k_b_keys<<<g, 256, 0, st>>>(dis.p, node_of.p, rows.p, in.ids, denom, n, key.p, tie.p, idx.p);
        LAUNCH_CHECK();
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, sort_bytes, tie.p, tie2.p, idx.p, idx2.p, (int)n, 0, 64, st));
        k_b_gather_key<<<g, 256, 0, st>>>(key.p, idx2.p, n, key2.p);
        LAUNCH_CHECK();
        CK(cub::DeviceRadixSort::SortPairs(tmp.p, sort_bytes, key2.p, key.p, idx2.p, idx.p, (int)n, 0, 64, st));
        k_b_permute<<<g, 256, 0, st>>>(idx.p, rows.p, dis.p, chain.p, n, rows2.p, dis2.p, chain2.p);
        LAUNCH_CHECK();
        std::swap(rows.p, rows2.p);
        std::swap(dis.p, dis2.p);
        std::swap(chain.p, chain2.p);
        // children (or, at the leaf level, the leaves themselves)
        std::vector<int64_t> cpos, csize;
        int64_t cfirst;
        if (level < t->levels) {
            cfirst = (first - 1) * nc + 2;
            cpos.resize((size_t)count * nc);
            csize.resize((size_t)count * nc);
            for (int o = 0; o < count; o++) {
                const int64_t sz = hsize[(size_t)o], p = hpos[(size_t)o], avg = sz / nc;
                for (int64_t j = 0; j < nc; j++) {
                    const size_t k = (size_t)(o * nc + j);
                    cpos[k] = p + j * avg;
                    csize[k] = (j == nc - 1) ? sz - avg * (nc - 1) : avg;
                    t->pos[cfirst + (int64_t)k] = cpos[k];
                    t->size[cfirst + (int64_t)k] = csize[k];
                }
            }
        } else {
            cfirst = first;
            cpos = hpos;
            csize = hsize;
        }
        const int cnt = (int)cpos.size();
        DBuf<int64_t> dcp, dcs;
        h2d_vec(dcp, cpos, st);
        h2d_vec(dcs, csize, st);
        DBuf<double> mn((size_t)cnt, st), mx((size_t)cnt, st);
        k_b_ranges<<<grid_for(cnt, 256), 256, 0, st>>>(dis.p, dcp.p, dcs.p, cnt, mn.p, mx.p);
        LAUNCH_CHECK();
        const std::vector<double> hmn = d2h_vec(mn.p, (size_t)cnt, st), hmx = d2h_vec(mx.p, (size_t)cnt, st);
        for (int k = 0; k < cnt; k++)
            if (csize[(size_t)k] > 0) {
                t->min_dis[cfirst + k] = hmn[(size_t)k];
                t->max_dis[cfirst + k] = hmx[(size_t)k];
            }
    }
    const std::vector<int32_t> hrows = d2h_vec(rows.p, (size_t)n, st);
    const std::vector<double> hdis = d2h_vec(dis.p, (size_t)n, st);
    for (int64_t e = 0; e < n; e++) {
        t->rows[e] = hrows[(size_t)e];
        t->dis[e] = hdis[(size_t)e];
        if (t->tombstone) t->tombstone[e] = 0;
    }
}

__global__ void k_b_ids_of_rows(const int64_t *__restrict__ ids, const int64_t *__restrict__ prow, int cnt,
                                int64_t *out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) out[i] = prow[i] >= 0 ? ids[prow[i]] : -1;
}

void fill_pivot_ids(const int64_t *ids_dev, gts_tree *t, int64_t nodes, cudaStream_t st)
{
    std::vector<int64_t> pr(t->pivot_row, t->pivot_row + nodes + 1);
    DBuf<int64_t> dpr, out((size_t)nodes + 1, st);
    h2d_vec(dpr, pr, st);
    k_b_ids_of_rows<<<grid_for(nodes + 1, 256), 256, 0, st>>>(ids_dev, dpr.p, (int)(nodes + 1), out.p);
    LAUNCH_CHECK();
    const std::vector<int64_t> h = d2h_vec(out.p, (size_t)nodes + 1, st);
    for (int64_t i = 0; i <= nodes; i++) t->pivot_id[i] = h[(size_t)i];
}

int64_t check_build_args(int64_t n, int64_t root_row, gts_tree *t)
{
    if (!t) fail(GTS_EINVAL, "null tree");
    if (t->nc < 2) fail(GTS_EINVAL, "node_capacity must be >= 2");
    if (n > (1ll << 31) - 64) fail(GTS_EINVAL, "device build limited to 2^31 entries; shard the collection");
    if (n > 0 && (root_row < 0 || root_row >= n)) fail(GTS_EINVAL, "root_row out of range");
    return n;
}

}  // namespace

// Device build from a host dataset (same arguments and result as
// gts_build_tree, tree.py:370-385).
extern "C" int gts_build_tree_device(const gts_dataset *ds, int64_t root_row, int device, gts_tree *t)
{
    ABI_BEGIN
    if (!ds) fail(GTS_EINVAL, "null dataset");
    const int64_t n = check_build_args(ds->n, root_row, t);
    if (n == 0) { t->levels = 0; t->split_rounds = 0; return GTS_OK; }
    if (ds->metric != GTS_EDIT && ds->metric != GTS_L1 && ds->metric != GTS_L2)
        fail(GTS_EMETRIC, "device build supports edit, l1, l2 (angular: gts_build_tree)");
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
    BuildInput in;
    in.metric = ds->metric;
    in.n = n;
    DBuf<int64_t> ids((size_t)n, st);
    h2d(ids.p, ds->ids, (size_t)n, st);
    in.ids = ids.p;
    DBuf<double> x64;
    DBuf<uint32_t> text, sword;
    DBuf<int32_t> slen;
    if (ds->metric == GTS_EDIT) {
        std::vector<int32_t> alpha;
        dense_alphabet(ds->codes, ds->offsets[n], alpha);
        if (alpha.size() > 254) fail(GTS_EMETRIC, "device build: alphabet of %zu symbols exceeds 254", alpha.size());
        in.A = (int)alpha.size();
        std::vector<uint32_t> words, wstart;
        std::vector<int32_t> lens;
        const SymMap smap(alpha);
        pack_words(n, ds->offsets, [&](int64_t k) { return smap(ds->codes[k]); }, words, wstart, lens);
        for (auto l : lens)
            if (l > kMaxWords * 32) fail(GTS_EINVAL, "device build: strings longer than %d symbols", kMaxWords * 32);
        text.alloc(words.size(), st);
        h2d(text.p, words.data(), words.size(), st);
        sword.alloc(wstart.size(), st);
        h2d(sword.p, wstart.data(), wstart.size(), st);
        slen.alloc(lens.size(), st);
        h2d(slen.p, lens.data(), lens.size(), st);
        in.text = text.p;
        in.sword = sword.p;
        in.slen = slen.p;
        in.h_slen = std::move(lens);
    } else {
        in.D = (int)ds->dim;
        x64.alloc((size_t)(n * in.D), st);
        h2d(x64.p, ds->vectors, (size_t)(n * in.D), st);
        in.x64 = x64.p;
    }
    device_build(in, root_row, t, st);
    fill_pivot_ids(ids.p, t, gts_node_count(t->levels, t->nc), st);
    CK(cudaStreamSynchronize(st));
    return GTS_OK;
    ABI_END
}

// Device build over device-resident float32 vectors (x: [n][dim] on
// `device`, e.g. from gts_generate_clustered); ids: host [n].
extern "C" int gts_build_tree_device_f32(int32_t metric, int64_t n, int64_t dim, const float *x, const int64_t *ids,
                                         int64_t root_row, int device, gts_tree *t)
{
    ABI_BEGIN
    check_build_args(n, root_row, t);
    if (n == 0) { t->levels = 0; t->split_rounds = 0; return GTS_OK; }
    if (metric != GTS_L1 && metric != GTS_L2) fail(GTS_EMETRIC, "device f32 build supports l1, l2");
    if (!x || !ids) fail(GTS_EINVAL, "null argument");
    CK(cudaSetDevice(device));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};
    BuildInput in;
    in.metric = metric;
    in.n = n;
    in.D = (int)dim;
    in.x32 = x;
    DBuf<int64_t> dids((size_t)n, st);
    h2d(dids.p, ids, (size_t)n, st);
    in.ids = dids.p;
    device_build(in, root_row, t, st);
    fill_pivot_ids(dids.p, t, gts_node_count(t->levels, t->nc), st);
    CK(cudaStreamSynchronize(st));
    return GTS_OK;
    ABI_END
}

// ---------------------------------------------------------------------------
// Device-side synthetic data (a generate_clustered-
// equivalent collection produced on the device with a counter-based RNG, so
// a 100M x 32 collection never exists as a host array) and an index over
// device-resident float32 vectors.
// ---------------------------------------------------------------------------
namespace {

// Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11): counter-based, so any
// object of the collection is generated independently from its index.
__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k)
{
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
        k.x += 0x9E3779B9u;
        k.y += 0xBB67AE85u;
    }
    return c;
}

__device__ __forceinline__ float u01(uint32_t x) { return (float)((x >> 8) + 1u) * 0x1p-24f; }   // (0, 1]

__device__ __forceinline__ void normals4(uint4 r, float *z)
{
    const float a = sqrtf(-2.f * logf(u01(r.x))), b = sqrtf(-2.f * logf(u01(r.z)));
    float s0, c0, s1, c1;
    sincospif(2.f * u01(r.y), &s0, &c0);
    sincospif(2.f * u01(r.w), &s1, &c1);
    z[0] = a * c0;
    z[1] = a * s0;
    z[2] = b * c1;
    z[3] = b * s1;
}

// out[i] = object first+i (query_seed == 0): cluster c uniform in
// [0, clusters), centre U(0,1]^D, member = centre + N(0, spread);
// or query first+i (query_seed != 0): a uniformly drawn object + N(0, noise).
__global__ void k_gen_clustered(uint2 key, int64_t n_total, int D, int64_t clusters, float spread, int64_t first,
                                int64_t count, uint2 qkey, int query, float noise, float *out)
{
    const int g4 = (D + 3) >> 2;
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= count * g4) return;
    const int64_t i = t / g4;
    const int d4 = (int)(t - i * g4);
    const uint64_t j = (uint64_t)(first + i);
    uint64_t row = j;
    if (query) {
        const uint4 r = philox4x32(make_uint4((uint32_t)j, (uint32_t)(j >> 32), 0xA5A5A5A5u, 0u), qkey);
        row = (((uint64_t)r.x << 32) | r.y) % (uint64_t)n_total;
    }
    const uint4 a = philox4x32(make_uint4((uint32_t)row, (uint32_t)(row >> 32), 0xC1u, 0u), key);
    const uint64_t c = (((uint64_t)a.x << 32) | a.y) % (uint64_t)clusters;
    const uint4 cu = philox4x32(make_uint4((uint32_t)c, (uint32_t)(c >> 32), (uint32_t)d4, 0xCEu), key);
    float z[4], w[4] = {0.f, 0.f, 0.f, 0.f};
    normals4(philox4x32(make_uint4((uint32_t)row, (uint32_t)(row >> 32), (uint32_t)d4, 0x4Eu), key), z);
    if (query) normals4(philox4x32(make_uint4((uint32_t)j, (uint32_t)(j >> 32), (uint32_t)d4, 0x51u), qkey), w);
    const float cen[4] = {u01(cu.x), u01(cu.y), u01(cu.z), u01(cu.w)};
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const int d = d4 * 4 + k;
        if (d < D) {
            float v = __fadd_rn(cen[k], __fmul_rn(spread, z[k]));
            if (query) v = __fadd_rn(v, __fmul_rn(noise, w[k]));
            out[i * D + d] = v;
        }
    }
}

__global__ void k_gather_rows_f32(const float *__restrict__ x, int D, int Dp, const int32_t *__restrict__ drow,
                                  int64_t n, float *v32)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * Dp) return;
    const int64_t e = t / Dp;
    const int d = (int)(t - e * Dp);
    v32[t] = (d < D && drow[e] >= 0) ? x[(int64_t)drow[e] * D + d] : 0.f;
}

// tensor-core copy (k_leafgroup_mma2): bf16(o - leaf pivot), K padded to Dk
__global__ void k_vcent(const float *__restrict__ v32, int D, int Dp, int Dk, const int32_t *__restrict__ epiv,
                        int64_t n, __nv_bfloat16 *vc)
{
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n * Dk) return;
    const int64_t e = t / Dk;
    const int d = (int)(t - e * Dk);
    const int p = epiv[e];
    vc[t] = __float2bfloat16(d < D && p >= 0 ? v32[e * Dp + d] - v32[(int64_t)p * Dp + d] : 0.f);
}

// se_e = c . bf16(o_e - c) accumulated in float64 in index order (the
// host's loop, gts_index_create)
__global__ void k_vse(const float *__restrict__ v32, int D, int Dp, int Dk, const int32_t *__restrict__ epiv,
                      const __nv_bfloat16 *__restrict__ vc, int64_t n, float *se)
{
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= n) return;
    const int p = epiv[e];
    double acc = 0.0;
    if (p >= 0)
        for (int d = 0; d < D; d++)
            acc = __dadd_rn(acc, __dmul_rn((double)v32[(int64_t)p * Dp + d], (double)__bfloat162float(vc[e * Dk + d])));
    se[e] = (float)acc;
}

}  // namespace

extern "C" int gts_generate_clustered(uint64_t seed, int64_t n_total, int64_t dim, int64_t clusters, float spread,
                                      int64_t first, int64_t count, uint64_t query_seed, float noise, float *out,
                                      void *stream)
{
    ABI_BEGIN
    if (!out || dim < 1 || clusters < 1 || n_total < 1 || first < 0 || count < 0) fail(GTS_EINVAL, "invalid arguments");
    if (count == 0) return GTS_OK;
    const int64_t work = count * ((dim + 3) / 4);
    k_gen_clustered<<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(
        make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)), n_total, (int)dim, clusters, spread, first, count,
        make_uint2((uint32_t)query_seed, (uint32_t)(query_seed >> 32)), query_seed != 0, noise, out);
    LAUNCH_CHECK();
    return GTS_OK;
    ABI_END
}

// Index over device-resident float32 vectors x[n][dim] (dataset row order,
// on `device`); tree: host arrays of the collection's tree; ids: host [n].
extern "C" int gts_index_create_f32dev(const gts_tree *t, int32_t metric, int64_t dim, const float *x,
                                       const int64_t *ids, int device, gts_index **out)
{
    ABI_BEGIN
    if (!t || !x || !ids || !out) fail(GTS_EINVAL, "null argument");
    if (metric != GTS_L1 && metric != GTS_L2) fail(GTS_EMETRIC, "device-resident vectors: l1 or l2");
    if (t->n > (1ll << 31) - 64) fail(GTS_EINVAL, "index larger than 2^31 entries; shard it");
    prime_pool(device);
    CK(cudaSetDevice(device));
    auto *ix = new gts_index();
    try {
        cudaStream_t st = 0;
        ix->device = device;
        ix->metric = metric;
        ix->n = t->n;
        ix->nc = (int)t->nc;
        ix->levels = (int)t->levels;
        ix->split_rounds = (int)t->split_rounds;
        ix->nodes = t->nodes;
        ix->D = (int)dim;
        ix->Dp = (ix->D + 3) & ~3;
        const int64_t n = t->n;
        if (n == 0 || t->levels == 0) { *out = ix; return GTS_OK; }
        std::vector<int64_t> ord((size_t)n), drow;
        for (int64_t e = 0; e < n; e++) ord[(size_t)e] = e;
        const SlotLayout lay = slot_layout(t);
        ord = slot_order(t, lay, ord);
        std::vector<NodeRec> nodes;
        upload_tables(ix, t, ord, ids, st, drow, nodes, lay);
        const int64_t ns = lay.n_slots;
        ix->data_exact = true;   // float32 payloads: the fp32 copy is exact
        ix->vec32.alloc((size_t)(ns * ix->Dp), st);
        k_gather_rows_f32<<<grid_for(ns * ix->Dp, 256), 256, 0, st>>>(x, ix->D, ix->Dp, ix->row.p, ns, ix->vec32.p);
        LAUNCH_CHECK();
        if (metric == GTS_L2 && ix->D >= 32 && ix->D <= 128 && ix->max_leaf <= 256 &&
            std::getenv("GTS_NO_MMA") == nullptr) {
            ix->Dk = (ix->D + 63) & ~63;
            std::vector<int32_t> epiv((size_t)ns, -1);
            for (int64_t i = ix->leaf_first; i < (int64_t)ix->leaf_first + ix->leaf_count; i++)
                for (int64_t e = lay.dpos[(size_t)i]; e < lay.dpos[(size_t)i] + t->size[i]; e++)
                    epiv[(size_t)e] = nodes[(size_t)i].piv;
            DBuf<int32_t> dep;
            h2d_vec(dep, epiv, st);
            const size_t tail = (size_t)16 * ix->Dk / 8;
            ix->vcent.alloc((size_t)ns * ix->Dk / 8 + tail, st);
            CK(cudaMemsetAsync(ix->vcent.p, 0, ((size_t)ns * ix->Dk / 8 + tail) * sizeof(uint4), st));
            auto *vc = reinterpret_cast<__nv_bfloat16 *>(ix->vcent.p);
            k_vcent<<<grid_for(ns * ix->Dk, 256), 256, 0, st>>>(ix->vec32.p, ix->D, ix->Dp, ix->Dk, dep.p, ns, vc);
            LAUNCH_CHECK();
            ix->vse.alloc((size_t)ns, st);
            k_vse<<<grid_for(ns, 256), 256, 0, st>>>(ix->vec32.p, ix->D, ix->Dp, ix->Dk, dep.p, vc, ns, ix->vse.p);
            LAUNCH_CHECK();
            build_vtile(ix, st);
        }
        CK(cudaStreamSynchronize(st));
        // max |x| (used only by inexact data's slack; kept for completeness)
        ix->data_maxabs = 0.f;
        const int64_t prow = t->pivot_row[1];
        if (prow >= 0 && prow < n) {
            std::vector<float> r32((size_t)ix->D);
            CK(cudaMemcpy(r32.data(), x + prow * ix->D, sizeof(float) * ix->D, cudaMemcpyDeviceToHost));
            root_radius_of(ix, std::vector<double>(r32.begin(), r32.end()), st);
        }
        *out = ix;
        return GTS_OK;
    } catch (...) {
        delete ix;
        throw;
    }
    ABI_END
}
