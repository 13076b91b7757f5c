// sharded.cuh -- the multi-shard exchange step, included
// at the end of engine.cu (it uses the engine's index / result types).
//
// A collection split into shards has one GTS tree per shard; exact search
// over the union is the union of exact per-shard answers (PAPER.md:213-222,
// Def. 1/2).  The reference has a single index, so its anchors are the
// per-query merge it does inside one index: _KnnPool.merge (search.py:116-144)
// keeps the k smallest (distance, id), and _collect (search.py:298-314)
// orders range answers by (distance, id).
//
// k_merge_rank is that merge for S sorted per-shard lists at once: every
// answer's output slot is its rank inside its own (shard, query) list plus,
// for every other shard, the number of that shard's answers of the same
// query that order before it -- a binary search per other shard.  No sort,
// one pass, and kNN truncation is "slot < k".
//
// Two drivers sit on it:
//  * gts_merge_results: the owner-side merge after an all-to-all exchange
//    (the torch.distributed / NCCL path of paper_2404_00966_b200/sharded.py);
//  * gts_multi_*: one process driving every shard of a collection, one host
//    thread per shard (each on its own device and stream), the kNN bound
//    exchange as a device MIN, and the merge on the first shard's device.

namespace {

__device__ __forceinline__ bool ans_before(double da, long long ia, int sa, double db, long long ib, int sb)
{
    return da < db || (da == db && (ia < ib || (ia == ib && sa < sb)));
}

// counts[s*nq + q] -> per-query output sizes (kNN: min(total, k))
__global__ void k_merge_totals(const int64_t *__restrict__ counts, int nsrc, int64_t nq,
                               const int64_t *__restrict__ ks, long long *tot)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q > nq) return;
    if (q == nq) { tot[q] = 0; return; }
    long long t = 0;
    for (int s = 0; s < nsrc; s++) t += counts[(int64_t)s * nq + q];
    if (ks) t = min(t, (long long)ks[q]);
    tot[q] = t;
}

__global__ void k_merge_rank(const int64_t *__restrict__ counts, const long long *__restrict__ seg_off, int nsrc,
                             int64_t nq, const int64_t *__restrict__ ids, const double *__restrict__ dis,
                             int64_t total_in, const long long *__restrict__ out_off, int64_t *oids, double *odis)
{
    const int64_t nseg = (int64_t)nsrc * nq;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total_in;
         e += (int64_t)gridDim.x * blockDim.x) {
        // segment holding e: last seg with seg_off[seg] <= e (skips empty ones)
        int64_t lo = 0, hi = nseg - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (seg_off[mid] <= e) lo = mid; else hi = mid - 1;
        }
        const int s = (int)(lo / nq);
        const int64_t q = lo - (int64_t)s * nq;
        const double d = dis[e];
        const long long id = ids[e];
        long long pos = e - seg_off[lo];
        const long long lim = out_off[q + 1] - out_off[q];
        if (pos >= lim) continue;   // already past k inside its own list
        for (int s2 = 0; s2 < nsrc && pos < lim; s2++) {
            if (s2 == s) continue;
            const long long b = seg_off[(int64_t)s2 * nq + q];
            long long a = 0, c = counts[(int64_t)s2 * nq + q];
            while (a < c) {   // count of s2's answers ordering before (d, id, s)
                const long long m = (a + c) >> 1;
                if (ans_before(dis[b + m], ids[b + m], s2, d, id, s)) a = m + 1; else c = m;
            }
            pos += a;
        }
        if (pos < lim) {
            oids[out_off[q] + pos] = id;
            odis[out_off[q] + pos] = d;
        }
    }
}

__global__ void k_sum_stats(const int64_t *__restrict__ v, int nsrc, int64_t nq, unsigned long long *out)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long t = 0;
    for (int s = 0; s < nsrc; s++) t += (unsigned long long)v[(int64_t)s * nq + q];
    out[q] = t;
}

__global__ void k_offsets_to_counts(const int64_t *__restrict__ off, int64_t nq, int64_t *counts)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q < nq) counts[q] = off[q + 1] - off[q];
}

__global__ void k_min_radius(const float *__restrict__ all, int nsrc, int64_t nq, float *out)
{
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= nq) return;
    float m = INFINITY;
    for (int s = 0; s < nsrc; s++) m = fminf(m, all[(int64_t)s * nq + q]);
    out[q] = m;
}

// Merge S per-source CSR lists (source-major: counts[s][q], then every
// source's answers query by query) into one result on the current device.
gts_result *merge_results(int nsrc, int64_t nq, const int64_t *counts, const int64_t *ids, const double *dis,
                          const int64_t *ks, const int64_t *verified, const int64_t *pruned, cudaStream_t st)
{
    auto *res = new gts_result();
    try {
        res->nq = nq;
        res->stream = st;
        res->offsets.alloc((size_t)nq + 1, st);
        const int64_t nseg = (int64_t)nsrc * nq;
        DBuf<long long> seg_off((size_t)nseg + 1, st), tot((size_t)nq + 1, st), out_off((size_t)nq + 1, st);
        // exclusive scan of the source-major counts = every segment's start
        {
            DBuf<long long> cnt((size_t)nseg + 1, st);
            CK(cudaMemsetAsync(cnt.p, 0, sizeof(long long) * (nseg + 1), st));
            if (nseg) CK(cudaMemcpyAsync(cnt.p, counts, sizeof(int64_t) * nseg, cudaMemcpyDeviceToDevice, st));
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, seg_off.p, nseg + 1, st);
            DBuf<uint8_t> tmp(tb, st);
            CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, seg_off.p, nseg + 1, st));
        }
        k_merge_totals<<<grid_for(nq + 1, 256), 256, 0, st>>>(counts, nsrc, nq, ks, tot.p);
        LAUNCH_CHECK();
        {
            size_t tb = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb, tot.p, out_off.p, nq + 1, st);
            DBuf<uint8_t> tmp(tb, st);
            CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, tot.p, out_off.p, nq + 1, st));
        }
        long long h[2] = {0, 0};
        CK(cudaMemcpyAsync(&h[0], seg_off.p + nseg, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&h[1], out_off.p + nq, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const int64_t total_in = h[0], total_out = h[1];
        res->total = total_out;
        res->ids.alloc((size_t)std::max<int64_t>(total_out, 1), st);
        res->dis.alloc((size_t)std::max<int64_t>(total_out, 1), st);
        if (total_in)
            k_merge_rank<<<grid_for(total_in, 256, 148u * 64u), 256, 0, st>>>(counts, seg_off.p, nsrc, nq, ids, dis,
                                                                              total_in, out_off.p, res->ids.p,
                                                                              res->dis.p);
        LAUNCH_CHECK();
        CK(cudaMemcpyAsync(res->offsets.p, out_off.p, sizeof(int64_t) * (nq + 1), cudaMemcpyDeviceToDevice, st));
        if (verified) {
            res->verified.alloc((size_t)std::max<int64_t>(nq, 1), st);
            k_sum_stats<<<grid_for(nq, 256), 256, 0, st>>>(verified, nsrc, nq, res->verified.p);
            LAUNCH_CHECK();
        }
        if (pruned) {
            res->pruned.alloc((size_t)std::max<int64_t>(nq, 1), st);
            k_sum_stats<<<grid_for(nq, 256), 256, 0, st>>>(pruned, nsrc, nq, res->pruned.p);
            LAUNCH_CHECK();
        }
        CK(cudaStreamSynchronize(st));
    } catch (...) {
        delete res;
        throw;
    }
    return res;
}

}  // namespace

// A collection served by several shard indexes (one GTS tree each), each on
// the device it was created on.  Answers are merged on shards[0]'s device.
struct gts_multi {
    std::vector<gts_index *> shards;
    std::vector<cudaStream_t> streams;
    int merge_device = 0;
};

extern "C" int gts_merge_results(int nsrc, int64_t nq, const int64_t *counts, const int64_t *ids, const double *dis,
                                 const int64_t *ks, const int64_t *verified, const int64_t *pruned, void *stream,
                                 gts_result **out)
{
    ABI_BEGIN
    if (!out || nsrc < 1 || nq < 0 || (nq && !counts)) fail(GTS_EINVAL, "invalid merge arguments");
    *out = merge_results(nsrc, nq, counts, ids, dis, ks, verified, pruned, (cudaStream_t)stream);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_multi_create(int nshards, gts_index *const *shards, gts_multi **out)
{
    ABI_BEGIN
    if (!out || nshards < 1 || !shards) fail(GTS_EINVAL, "need at least one shard");
    auto *m = new gts_multi();
    try {
        for (int i = 0; i < nshards; i++) {
            if (!shards[i]) fail(GTS_EINVAL, "null shard %d", i);
            if (shards[i]->metric != shards[0]->metric || shards[i]->D != shards[0]->D)
                fail(GTS_EMETRIC, "shard %d metric/dimension differs from shard 0", i);
            m->shards.push_back(shards[i]);
            CK(cudaSetDevice(shards[i]->device));
            cudaStream_t s;
            CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
            m->streams.push_back(s);
        }
        m->merge_device = shards[0]->device;
        // NVLink peer access between every pair of distinct shard devices
        for (int i = 0; i < nshards; i++)
            for (int j = 0; j < nshards; j++) {
                const int a = shards[i]->device, b = shards[j]->device;
                int ok = 0;
                if (a != b && cudaDeviceCanAccessPeer(&ok, a, b) == cudaSuccess && ok) {
                    CK(cudaSetDevice(a));
                    if (cudaDeviceEnablePeerAccess(b, 0) != cudaSuccess) cudaGetLastError();
                }
            }
    } catch (...) {
        for (auto s : m->streams) cudaStreamDestroy(s);
        delete m;
        throw;
    }
    *out = m;
    return GTS_OK;
    ABI_END
}

extern "C" int gts_multi_destroy(gts_multi *m)
{
    ABI_BEGIN
    if (!m) return GTS_OK;
    for (size_t i = 0; i < m->streams.size(); i++) {
        cudaSetDevice(m->shards[i]->device);
        cudaStreamDestroy(m->streams[i]);
    }
    delete m;
    return GTS_OK;
    ABI_END
}

namespace {

// run fn(i) for every shard on its own host thread; the first error wins
template <class F>
void per_shard(gts_multi *m, F &&fn)
{
    const int S = (int)m->shards.size();
    std::vector<int> codes((size_t)S, GTS_OK);
    std::vector<std::string> msgs((size_t)S);
    std::vector<std::thread> th;
    for (int i = 0; i < S; i++)
        th.emplace_back([&, i] {
            try {
                CK(cudaSetDevice(m->shards[(size_t)i]->device));
                fn(i);
            } catch (const Error &e) {
                codes[(size_t)i] = e.code;
                msgs[(size_t)i] = g_err;
            } catch (const std::bad_alloc &) {
                codes[(size_t)i] = GTS_EOOM;
                msgs[(size_t)i] = "host allocation failed";
            } catch (...) {
                codes[(size_t)i] = GTS_EINVAL;
                msgs[(size_t)i] = "unexpected C++ exception";
            }
        });
    for (auto &t : th) t.join();
    for (int i = 0; i < S; i++)
        if (codes[(size_t)i] != GTS_OK) fail(codes[(size_t)i], "shard %d: %s", i, msgs[(size_t)i].c_str());
}

}  // namespace

// StreamingIndex-free sharded batch (BatchSearcher.range_batch / knn_batch
// semantics over the union of the shards): upload the batch to every shard,
// kNN: probe on every shard -> MIN of the radii -> bounded search; range:
// search; then gather every shard's CSR to the merge device and merge.
extern "C" int gts_multi_batch_host(gts_multi *m, const gts_query_batch *qb, int mode, const double *radii,
                                    const int64_t *ks, int64_t memory_units, int flags, gts_result **out)
{
    ABI_BEGIN
    if (!m || !qb || !out) fail(GTS_EINVAL, "null argument");
    if (mode != 0 && mode != 1) fail(GTS_EINVAL, "mode must be 0 (range) or 1 (knn)");
    const int S = (int)m->shards.size();
    const int64_t nq = qb->nq;
    const int pruning = (flags & GTS_FLAG_PRUNING) ? 1 : 0;
    std::vector<gts_queries *> qs((size_t)S, nullptr);
    std::vector<gts_result *> rs((size_t)S, nullptr);
    std::vector<DBuf<float>> rad((size_t)S);
    auto cleanup = [&] {
        for (int i = 0; i < S; i++) {
            cudaSetDevice(m->shards[(size_t)i]->device);
            delete rs[(size_t)i];
            delete qs[(size_t)i];
            rad[(size_t)i].release();
        }
    };
    try {
        per_shard(m, [&](int i) {
            cudaStream_t st = m->streams[(size_t)i];
            qs[(size_t)i] = upload_queries(m->shards[(size_t)i], qb, st);
            if (mode == 1 && pruning) {
                rad[(size_t)i].alloc((size_t)std::max<int64_t>(nq, 1), st);
                run_search(m->shards[(size_t)i], qs[(size_t)i], 1, nullptr, ks, 0, 1, st, false, nullptr,
                           rad[(size_t)i].p);
            }
        });
        if (mode == 1 && pruning && S > 1 && nq > 0) {
            // the one kNN exchange: every shard searches with the MIN radius
            CK(cudaSetDevice(m->merge_device));
            cudaStream_t st = m->streams[0];
            DBuf<float> all((size_t)S * nq, st), mn((size_t)nq, st);
            for (int i = 0; i < S; i++)
                CK(cudaMemcpyPeerAsync(all.p + (size_t)i * nq, m->merge_device, rad[(size_t)i].p,
                                       m->shards[(size_t)i]->device, sizeof(float) * nq, st));
            k_min_radius<<<grid_for(nq, 256), 256, 0, st>>>(all.p, S, nq, mn.p);
            LAUNCH_CHECK();
            for (int i = 0; i < S; i++)
                CK(cudaMemcpyPeerAsync(rad[(size_t)i].p, m->shards[(size_t)i]->device, mn.p, m->merge_device,
                                       sizeof(float) * nq, st));
            CK(cudaStreamSynchronize(st));
        }
        per_shard(m, [&](int i) {
            cudaStream_t st = m->streams[(size_t)i];
            rs[(size_t)i] = run_search(m->shards[(size_t)i], qs[(size_t)i], mode, radii, ks, memory_units, pruning,
                                       st, (flags & GTS_FLAG_CACHE) != 0,
                                       (mode == 1 && pruning) ? rad[(size_t)i].p : nullptr, nullptr);
            CK(cudaStreamSynchronize(st));
        });
        // gather to the merge device: [S][nq] counts, answers source-major
        CK(cudaSetDevice(m->merge_device));
        cudaStream_t st = m->streams[0];
        int64_t tot = 0;
        std::vector<int64_t> base((size_t)S);
        for (int i = 0; i < S; i++) { base[(size_t)i] = tot; tot += rs[(size_t)i]->total; }
        DBuf<int64_t> offs((size_t)S * (nq + 1), st), cnt((size_t)std::max<int64_t>(S * nq, 1), st);
        DBuf<int64_t> ids((size_t)std::max<int64_t>(tot, 1), st), ver((size_t)std::max<int64_t>(S * nq, 1), st),
            prn((size_t)std::max<int64_t>(S * nq, 1), st);
        DBuf<double> dis((size_t)std::max<int64_t>(tot, 1), st);
        int64_t peak = 0;
        int64_t limits[64] = {0};
        for (int i = 0; i < S; i++) {
            gts_result *r = rs[(size_t)i];
            const int dev = m->shards[(size_t)i]->device;
            CK(cudaMemcpyPeerAsync(offs.p + (size_t)i * (nq + 1), m->merge_device, r->offsets.p, dev,
                                   sizeof(int64_t) * (nq + 1), st));
            if (r->total) {
                CK(cudaMemcpyPeerAsync(ids.p + base[(size_t)i], m->merge_device, r->ids.p, dev,
                                       sizeof(int64_t) * r->total, st));
                CK(cudaMemcpyPeerAsync(dis.p + base[(size_t)i], m->merge_device, r->dis.p, dev,
                                       sizeof(double) * r->total, st));
            }
            if (nq && r->verified.p)
                CK(cudaMemcpyPeerAsync(ver.p + (size_t)i * nq, m->merge_device, r->verified.p, dev,
                                       sizeof(int64_t) * nq, st));
            else if (nq)
                CK(cudaMemsetAsync(ver.p + (size_t)i * nq, 0, sizeof(int64_t) * nq, st));
            if (nq && r->pruned.p)
                CK(cudaMemcpyPeerAsync(prn.p + (size_t)i * nq, m->merge_device, r->pruned.p, dev,
                                       sizeof(int64_t) * nq, st));
            else if (nq)
                CK(cudaMemsetAsync(prn.p + (size_t)i * nq, 0, sizeof(int64_t) * nq, st));
            peak = std::max(peak, r->peak);
            for (int l = 0; l < 64; l++) limits[l] = std::max(limits[l], r->limits[l]);
        }
        for (int i = 0; i < S; i++) {
            // the answer offsets become per-query counts (answers are already
            // contiguous per source and query in the gathered buffer)
            k_offsets_to_counts<<<grid_for(nq, 256), 256, 0, st>>>(offs.p + (size_t)i * (nq + 1), nq,
                                                                  cnt.p + (size_t)i * nq);
            LAUNCH_CHECK();
        }
        int64_t *dks = nullptr;
        DBuf<int64_t> kbuf;
        if (mode == 1) {
            kbuf.alloc((size_t)std::max<int64_t>(nq, 1), st);
            h2d(kbuf.p, ks, (size_t)nq, st);
            dks = kbuf.p;
        }
        gts_result *res = merge_results(S, nq, cnt.p, ids.p, dis.p, dks, ver.p, prn.p, st);
        res->peak = peak;
        std::memcpy(res->limits, limits, sizeof(limits));
        cleanup();
        *out = res;
    } catch (...) {
        cleanup();
        throw;
    }
    return GTS_OK;
    ABI_END
}
