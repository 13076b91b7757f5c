// updates.cuh -- in-place inserts into leaf slack,
// included by engine.cu.
//
// The reference buffers inserts in a pending list that every query scans by
// brute force, and rebuilds the whole tree when the list overflows
// (updates.py:109-158).  Here an insert goes into the
// tree itself: the device slot layout leaves free slots after every leaf
// (slot_layout), and an inserted object
//   * descends from the root: at each internal node it takes the child whose
//     [min, max] ring (distances to that node's pivot) contains its own
//     distance to the pivot, else the nearest ring; at the last split it
//     takes, among the leaves with a free slot, the one whose own-pivot
//     range it is nearest to (k_insert_path, float64 distances -- numpy
//     order / exact edit distance, as the build);
//   * is written into that leaf's next free slot (payload, pivot distance,
//     id, alive bit), and
//   * widens the chosen leaf's own-pivot range and every chosen internal
//     node's parent-pivot range to include it (fp32 bounds rounded
//     outward),
// so every pruning bound of search.py:28-57 stays valid and the answers stay
// exact.  Objects that cannot be placed (leaf full, string longer than a
// slot or with a symbol outside the index alphabet, payload that is not
// float32-exact over float32-exact data, angular metric) are reported back
// (slot -1); the caller keeps them in the pending cache that the same batch
// call scans (gts_index_cache_set).  The rebuild trigger stays the
// reference's (pending count over capacity) and the rebuild runs on the
// device (gts_build_tree_device).

namespace {

template <int MET>
__device__ __forceinline__ double exact_dist(const IndexView &ix, const QueryView &qv, int q, int e)
{
    if (MET == kMetricEdit) return (double)dist32<MET>(ix, qv, q, e);
    return vdist64<MET>(ix, qv, q, e);
}

// One thread per item: the descent, the float64 distance to every pivot on
// the path (dpath[t * levels + l], l = 0 is the root), the leaf reached
// (-1: the tree has no free slot).  Item t of this launch is query qidx[t]
// of the uploaded batch; node_free[v] = free slots in the leaves under node
// v, so the descent only enters subtrees that can still take the item.
template <int MET>
__global__ void k_insert_path(IndexView ix, QueryView qv, int nitems, const int32_t *__restrict__ qidx,
                              const int32_t *__restrict__ node_free, int32_t *out_leaf, double *dpath)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= nitems) return;
    const int q = qidx[t];
    const int nc = ix.nc, L = ix.levels;
    int node = 1;
    for (int l = 0; l + 1 < L; l++) {
        const double dv = exact_dist<MET>(ix, qv, q, ix.node[node].piv);
        dpath[(size_t)t * L + l] = dv;
        const int c0 = (node - 1) * nc + 2;
        // nearest ring first; among rings at the same gap (often many hold
        // d: edit distances to a pivot concentrate), the one whose centre is
        // nearest, so a batch spreads over the children instead of piling
        // into the first one
        int best = -1;
        double bgap = INFINITY, bctr = INFINITY;
        if (l + 2 < L) {
            // internal children: rings of distances to this node's pivot
            for (int j = 0; j < nc; j++) {
                const NodeRec c = ix.node[c0 + j];
                if (c.size <= 0 || node_free[c0 + j] <= 0) continue;
                const double gap = fmax(0.0, fmax((double)c.mn - dv, dv - (double)c.mx));
                const double ctr = fabs(dv - 0.5 * ((double)c.mn + (double)c.mx));
                if (gap < bgap || (gap == bgap && ctr < bctr)) { bgap = gap; bctr = ctr; best = c0 + j; }
            }
        } else {
            // leaf children: own-pivot ranges, only leaves with a free slot
            for (int j = 0; j < nc; j++) {
                const NodeRec c = ix.node[c0 + j];
                if (c.size <= 0 || node_free[c0 + j] <= 0) continue;
                const double dl = exact_dist<MET>(ix, qv, q, c.piv);
                const double gap = fmax(0.0, fmax((double)c.mn - dl, dl - (double)c.mx));
                const double ctr = fabs(dl - 0.5 * ((double)c.mn + (double)c.mx));
                if (gap < bgap || (gap == bgap && ctr < bctr)) { bgap = gap; bctr = ctr; best = c0 + j; }
            }
        }
        node = best;
        if (node < 0) break;
    }
    if (node >= 0 && L >= 1) {
        if (L == 1 && node_free[1] <= 0) node = -1;
        if (node >= 0) dpath[(size_t)t * L + (L - 1)] = exact_dist<MET>(ix, qv, q, ix.node[node].piv);
    }
    out_leaf[t] = node;
}

// Scatter the placed items into their slots.  Vectors: the uploaded
// float32 / float64 rows; strings: host-packed text words and scan records.
__global__ void k_insert_write(int nitems, const int32_t *__restrict__ slot, const float *__restrict__ dis,
                               const int64_t *__restrict__ ids, float *ix_dis, int64_t *ix_ids, int32_t *ix_row,
                               const float *__restrict__ q32, const double *__restrict__ q64, int D, int Dp,
                               float *vec32, double *vec64)
{
    const int i = blockIdx.x;
    if (i >= nitems) return;
    const int s = slot[i];
    if (s < 0) return;
    if (threadIdx.x == 0) {
        ix_dis[s] = dis[i];
        ix_ids[s] = ids[i];
        ix_row[s] = -1;
    }
    if (vec32)
        for (int d = threadIdx.x; d < Dp; d += blockDim.x) vec32[(size_t)s * Dp + d] = q32[(size_t)i * Dp + d];
    if (vec64)
        for (int d = threadIdx.x; d < D; d += blockDim.x) vec64[(size_t)s * D + d] = q64[(size_t)i * D + d];
}

// tensor-core copy of the placed vectors: bf16(o - leaf pivot) and
// se = c . bf16(o - c) in float64 index order (as gts_index_create)
__global__ void k_insert_vcent(int nitems, const int32_t *__restrict__ slot, const int32_t *__restrict__ piv,
                               const float *__restrict__ vec32, int D, int Dp, int Dk, __nv_bfloat16 *vc, float *se)
{
    const int i = blockIdx.x;
    if (i >= nitems || slot[i] < 0) return;
    const int64_t s = slot[i], p = piv[i];
    for (int d = threadIdx.x; d < Dk; d += blockDim.x)
        vc[s * Dk + d] = __float2bfloat16(d < D ? vec32[s * Dp + d] - vec32[p * Dp + d] : 0.f);
    __syncthreads();
    if (threadIdx.x == 0) {
        double acc = 0.0;
        for (int d = 0; d < D; d++)
            acc = __dadd_rn(acc, __dmul_rn((double)vec32[p * Dp + d], (double)__bfloat162float(vc[s * Dk + d])));
        se[s] = (float)acc;
    }
}

__global__ void k_insert_text(int nitems, const int32_t *__restrict__ slot, const uint32_t *__restrict__ sword,
                              const uint32_t *__restrict__ words, const int64_t *__restrict__ woff,
                              const uint4 *__restrict__ rec, const uint4 *__restrict__ hist, uint32_t *str,
                              int32_t *slen, uint4 *erec, uint4 *ehist)
{
    const int i = blockIdx.x;
    if (i >= nitems || slot[i] < 0) return;
    const int64_t s = slot[i];
    const int64_t a = woff[i], b = woff[i + 1];
    for (int64_t w = a + threadIdx.x; w < b; w += blockDim.x) str[sword[s] + (w - a)] = words[w];
    if (threadIdx.x == 0) {
        uint4 r = rec[i];
        r.z = sword[s];
        erec[s] = r;
        slen[s] = (int32_t)r.y;
        if (ehist) {
            ehist[2 * s] = hist[2 * i];
            ehist[2 * s + 1] = hist[2 * i + 1];
        }
    }
}

__global__ void k_set_alive_words(const int32_t *__restrict__ widx, const uint32_t *__restrict__ wval, int n,
                                  uint32_t *alive)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) alive[widx[i]] = wval[i];
}

__global__ void k_erec_slots(const int32_t *__restrict__ slots, int n, uint4 *erec, const float *dis,
                             const uint32_t *alive)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || slots[i] < 0) return;
    const int e = slots[i];
    const bool al = (alive[e >> 5] >> (e & 31)) & 1u;
    erec[e].x = al ? __float_as_uint(dis[e]) : 0x7fc00000u;
}

float round_down_f32(double v)
{
    float f = (float)v;
    if ((double)f > v) f = std::nextafter(f, -INFINITY);
    return f;
}

float round_up_f32_h(double v)
{
    float f = (float)v;
    if ((double)f < v) f = std::nextafter(f, INFINITY);
    return f;
}

// push changed alive words (and the scan records of the touched slots)
void sync_alive(gts_index *ix, const std::vector<int32_t> &slots, cudaStream_t st)
{
    std::vector<int32_t> widx;
    std::vector<uint32_t> wval;
    for (int32_t s : slots) {
        if (s < 0) continue;
        const int32_t w = s >> 5;
        if (std::find(widx.begin(), widx.end(), w) == widx.end()) widx.push_back(w);
    }
    if (widx.empty()) return;
    for (int32_t w : widx) wval.push_back(ix->h_alive[(size_t)w]);
    DBuf<int32_t> dw;
    DBuf<uint32_t> dv;
    h2d_vec(dw, widx, st);
    h2d_vec(dv, wval, st);
    k_set_alive_words<<<grid_for((int64_t)widx.size(), 256), 256, 0, st>>>(dw.p, dv.p, (int)widx.size(),
                                                                         ix->alive.p);
    LAUNCH_CHECK();
    if (ix->erec.p) {
        DBuf<int32_t> ds;
        h2d_vec(ds, slots, st);
        k_erec_slots<<<grid_for((int64_t)slots.size(), 256), 256, 0, st>>>(ds.p, (int)slots.size(), ix->erec.p,
                                                                         ix->dis.p, ix->alive.p);
        LAUNCH_CHECK();
    }
    CK(cudaStreamSynchronize(st));
}

}  // namespace

extern "C" int gts_index_insert(gts_index *ix, const gts_dataset *items, int32_t *slots, void *stream)
{
    ABI_BEGIN
    if (!ix || !items || !slots) fail(GTS_EINVAL, "null argument");
    const int64_t n = items->n;
    for (int64_t i = 0; i < n; i++) slots[i] = -1;
    if (n == 0 || ix->levels == 0 || ix->n_ref == 0) return GTS_OK;
    if (items->metric != ix->metric) fail(GTS_EMETRIC, "insert metric %d != index metric %d", items->metric, ix->metric);
    if (ix->metric == GTS_ANGULAR) return GTS_OK;   // angular inserts stay in the pending cache
    if (ix->metric != GTS_EDIT && items->dim != ix->D)
        fail(GTS_EMETRIC, "insert dimensionality %lld != %d", (long long)items->dim, ix->D);
    if (n > (1 << 24)) fail(GTS_EINVAL, "insert batch too large");
    CK(cudaSetDevice(ix->device));
    cudaStream_t st = (cudaStream_t)stream;
    const bool edit = ix->metric == GTS_EDIT;
    // host-side eligibility
    std::vector<uint8_t> ok((size_t)n, 1);
    std::vector<uint32_t> words;
    std::vector<int64_t> woff((size_t)n + 1, 0);
    std::vector<uint4> rec((size_t)n), hist;
    std::vector<int32_t> lens((size_t)n, 0);
    if (edit) {
        const SymMap smap(ix->h_alpha);
        if (ix->ehist.p) hist.assign((size_t)n * 2, make_uint4(0, 0, 0, 0));
        for (int64_t i = 0; i < n; i++) {
            const int64_t a = items->offsets[i], b = items->offsets[i + 1], l = b - a;
            lens[(size_t)i] = (int32_t)l;
            const int64_t nw = ((l + 15) / 16) * 4;
            bool good = nw <= ix->slot_words && l <= kMaxWords * 32;
            std::vector<uint32_t> w((size_t)std::max<int64_t>(nw, 1), 0u);
            uint8_t h[32] = {0};
            for (int64_t k = a; k < b && good; k++) {
                const uint32_t c = smap(items->codes[k]);
                if (c >= (uint32_t)ix->A) { good = false; break; }
                w[(size_t)((k - a) >> 2)] |= c << (8 * ((k - a) & 3));
                if (h[c & 31] < 255) h[c & 31]++;
            }
            ok[(size_t)i] = good;
            if (good) words.insert(words.end(), w.begin(), w.begin() + nw);
            woff[(size_t)i + 1] = (int64_t)words.size();
            if (good && ix->ehist.p) std::memcpy(&hist[(size_t)2 * i], h, 32);
        }
    } else if (ix->data_exact) {
        for (int64_t i = 0; i < n; i++)
            for (int64_t d = 0; d < ix->D; d++) {
                const double v = items->vectors[i * ix->D + d];
                if ((double)(float)v != v) { ok[(size_t)i] = 0; break; }
            }
    }
    // the eligible items as a query batch (descent distances use the
    // search's distance code, query = item)
    std::vector<int64_t> sel;
    for (int64_t i = 0; i < n; i++)
        if (ok[(size_t)i]) sel.push_back(i);
    const int64_t m = (int64_t)sel.size();
    if (m == 0) return GTS_OK;
    std::vector<double> cvec;
    std::vector<int32_t> ccodes;
    std::vector<int64_t> coff(1, 0);
    if (edit) {
        for (int64_t i : sel) {
            ccodes.insert(ccodes.end(), items->codes + items->offsets[i], items->codes + items->offsets[i + 1]);
            coff.push_back((int64_t)ccodes.size());
        }
        if (ccodes.empty()) ccodes.push_back(0);
    } else {
        cvec.resize((size_t)(m * ix->D));
        for (int64_t j = 0; j < m; j++)
            std::memcpy(cvec.data() + j * ix->D, items->vectors + sel[(size_t)j] * ix->D, sizeof(double) * ix->D);
    }
    gts_query_batch qb{items->metric, m, edit ? 0 : ix->D, edit ? nullptr : cvec.data(),
                       edit ? ccodes.data() : nullptr, edit ? coff.data() : nullptr};
    gts_queries *q = upload_queries(ix, &qb, st);
    struct QGuard { gts_queries *q; ~QGuard() { delete q; } } qg{q};
    const IndexView iv = make_view(ix, q);
    const QueryView qv = make_qview(ix, q);
    // Descent rounds: every item of a round descends against the free-slot
    // counts at the start of the round, so items racing for the same leaf
    // can overfill it; those are descended again, with the leaves filled by
    // this batch excluded, for up to eight rounds.
    const int L = ix->levels, nc = ix->nc;
    std::vector<int32_t> leaf((size_t)m, -1);
    std::vector<double> path((size_t)m * L, 0.0);
    std::vector<int32_t> free_((size_t)ix->leaf_count);
    for (int64_t l = 0; l < ix->leaf_count; l++)
        free_[(size_t)l] = (int32_t)(ix->leaf_cap[(size_t)l] - ix->leaf_size[(size_t)l]);
    std::vector<int32_t> todo((size_t)m);
    for (int64_t j = 0; j < m; j++) todo[(size_t)j] = (int32_t)j;
    for (int round = 0; round < 8 && !todo.empty(); round++) {
        const int nt = (int)todo.size();
        // free slots per node (leaves, then summed up the tree; Eq. 1 parent)
        std::vector<int32_t> nfree((size_t)ix->nodes + 1, 0);
        for (int64_t l = 0; l < ix->leaf_count; l++) nfree[(size_t)(ix->leaf_first + l)] = free_[(size_t)l];
        for (int64_t v = ix->nodes; v >= 2; v--) nfree[(size_t)((v - 2) / nc + 1)] += nfree[(size_t)v];
        DBuf<int32_t> dfree, dq, dleaf((size_t)nt, st);
        h2d_vec(dfree, nfree, st);
        h2d_vec(dq, todo, st);
        DBuf<double> dpath((size_t)nt * L, st);
        const unsigned g = grid_for(nt, 128);
        switch (ix->metric) {
        case GTS_EDIT: k_insert_path<kMetricEdit><<<g, 128, 0, st>>>(iv, qv, nt, dq.p, dfree.p, dleaf.p, dpath.p); break;
        case GTS_L1: k_insert_path<kMetricL1><<<g, 128, 0, st>>>(iv, qv, nt, dq.p, dfree.p, dleaf.p, dpath.p); break;
        default: k_insert_path<kMetricL2><<<g, 128, 0, st>>>(iv, qv, nt, dq.p, dfree.p, dleaf.p, dpath.p); break;
        }
        LAUNCH_CHECK();
        const std::vector<int32_t> rl = d2h_vec(dleaf.p, (size_t)nt, st);
        const std::vector<double> rp = d2h_vec(dpath.p, (size_t)nt * L, st);
        std::vector<int32_t> again;
        for (int t = 0; t < nt; t++) {
            const int32_t j = todo[(size_t)t], lf = rl[(size_t)t];
            if (lf < 0) continue;                                   // no free leaf under its path
            int32_t &fr = free_[(size_t)(lf - ix->leaf_first)];
            if (fr <= 0) { again.push_back(j); continue; }          // filled by an earlier item of this round
            fr--;
            leaf[(size_t)j] = lf;
            std::copy(rp.begin() + (size_t)t * L, rp.begin() + (size_t)(t + 1) * L, path.begin() + (size_t)j * L);
        }
        static const bool trace = std::getenv("GTS_TRACE") != nullptr;
        if (trace) {
            int none = 0;
            for (int t = 0; t < nt; t++) none += rl[(size_t)t] < 0;
            int64_t tf = 0;
            for (auto f : free_) tf += f;
            fprintf(stderr, "[gts] insert round %d: %d items, %d without a leaf, %zu collided, %lld free slots left, "
                            "levels %d, leaves %d\n", round, nt, none, again.size(), (long long)tf, L, ix->leaf_count);
        }
        todo.swap(again);
    }
    // slots, in item order; ranges of every node on the path widen
    std::vector<float> hdis((size_t)m, 0.f);
    std::vector<int32_t> hpiv((size_t)m, 0), cslot((size_t)m, -1);
    std::vector<int64_t> cids((size_t)m);
    std::vector<uint4> crec((size_t)m), chist(ix->ehist.p ? (size_t)m * 2 : 0);
    std::vector<uint32_t> cwords;
    std::vector<int64_t> cwoff((size_t)m + 1, 0);
    int64_t placed = 0;
    for (int64_t j = 0; j < m; j++) {
        const int64_t i = sel[(size_t)j];
        cids[(size_t)j] = items->ids[i];
        if (edit) {
            cwords.insert(cwords.end(), words.begin() + woff[(size_t)i], words.begin() + woff[(size_t)i + 1]);
            if (ix->ehist.p) { chist[(size_t)2 * j] = hist[(size_t)2 * i]; chist[(size_t)2 * j + 1] = hist[(size_t)2 * i + 1]; }
        }
        cwoff[(size_t)j + 1] = (int64_t)cwords.size();
        const int lf = leaf[(size_t)j];
        if (lf < 0) continue;
        const int64_t li = lf - ix->leaf_first;
        if (ix->leaf_size[(size_t)li] >= ix->leaf_cap[(size_t)li]) continue;
        const int64_t s = ix->leaf_dpos[(size_t)li] + ix->leaf_size[(size_t)li];
        ix->leaf_size[(size_t)li]++;
        slots[i] = (int32_t)s;
        cslot[(size_t)j] = (int32_t)s;
        placed++;
        // the path: the node at depth l (l >= 1) was chosen with the distance
        // to its parent's pivot (depth l - 1); the leaf's range is own-pivot
        int node = lf;
        std::vector<int> chain((size_t)L);
        for (int l = L - 1; l >= 0; l--) { chain[(size_t)l] = node; node = (node - 2) / nc + 1; }
        for (int l = (L == 1 ? 0 : 1); l < L; l++) {
            NodeRec &r = ix->h_nodes[(size_t)chain[(size_t)l]];
            const double d = (l == L - 1) ? path[(size_t)j * L + (L - 1)] : path[(size_t)j * L + (l - 1)];
            r.mn = std::min(r.mn, round_down_f32(d));
            r.mx = std::max(r.mx, round_up_f32_h(d));
        }
        ix->h_nodes[(size_t)lf].size = (int32_t)ix->leaf_size[(size_t)li];
        const double dl = path[(size_t)j * L + (L - 1)];
        hdis[(size_t)j] = (float)dl;
        hpiv[(size_t)j] = ix->h_nodes[(size_t)lf].piv;
        ix->h_alive[(size_t)(s >> 5)] |= 1u << (s & 31);
        if (!edit) ix->root_radius = std::max(ix->root_radius, round_up_f32_h(path[(size_t)j * L]));
        if (edit) {
            ix->h_slen[(size_t)s] = lens[(size_t)i];
            ix->max_len = std::max(ix->max_len, lens[(size_t)i]);
            const float lf32 = (float)lens[(size_t)i];
            uint32_t db, lb;
            std::memcpy(&db, &hdis[(size_t)j], 4);
            std::memcpy(&lb, &lf32, 4);
            crec[(size_t)j] = make_uint4(db, (uint32_t)lens[(size_t)i], 0u, lb);
        }
    }
    if (placed == 0) return GTS_OK;
    ix->n_inserted += placed;
    // device writes: payloads, records, node ranges and sizes, alive bits
    DBuf<int32_t> dsl, dpv;
    DBuf<float> ddis;
    DBuf<int64_t> dids;
    h2d_vec(dsl, cslot, st);
    h2d_vec(ddis, hdis, st);
    h2d_vec(dids, cids, st);
    h2d_vec(dpv, hpiv, st);
    k_insert_write<<<(unsigned)m, 128, 0, st>>>((int)m, dsl.p, ddis.p, dids.p, ix->dis.p, ix->ids.p, ix->row.p,
                                                q->vec32.p, q->vec64.p, ix->D, ix->Dp, edit ? nullptr : ix->vec32.p,
                                                edit ? nullptr : ix->vec64.p);
    LAUNCH_CHECK();
    if (!edit && ix->vcent.p) {
        k_insert_vcent<<<(unsigned)m, 128, 0, st>>>((int)m, dsl.p, dpv.p, ix->vec32.p, ix->D, ix->Dp, ix->Dk,
                                                    reinterpret_cast<__nv_bfloat16 *>(ix->vcent.p), ix->vse.p);
        LAUNCH_CHECK();
        build_vtile(ix, st);   // the leaf images follow vcent
    }
    if (edit) {
        DBuf<uint32_t> dw;
        DBuf<int64_t> dwo;
        DBuf<uint4> drec, dh;
        if (cwords.empty()) cwords.push_back(0u);
        h2d_vec(dw, cwords, st);
        h2d_vec(dwo, cwoff, st);
        h2d_vec(drec, crec, st);
        if (ix->ehist.p) h2d_vec(dh, chist, st);
        k_insert_text<<<(unsigned)m, 64, 0, st>>>((int)m, dsl.p, ix->sword.p, dw.p, dwo.p, drec.p,
                                                  ix->ehist.p ? dh.p : nullptr, ix->str.p, ix->slen.p, ix->erec.p,
                                                  ix->ehist.p);
        LAUNCH_CHECK();
        if (ix->esig.p) {
            k_slot_sig<<<grid_for(m, 128), 128, 0, st>>>(ix->str.p, ix->sword.p, ix->slen.p, dsl.p, m, ix->A,
                                                         ix->esig.p);
            LAUNCH_CHECK();
        }
    }
    CK(cudaStreamSynchronize(st));
    std::vector<int32_t> vslots(slots, slots + n);
    h2d(ix->node.p, ix->h_nodes.data(), ix->h_nodes.size(), st);
    sync_alive(ix, vslots, st);
    return GTS_OK;
    ABI_END
}

extern "C" int gts_index_erase(gts_index *ix, const int32_t *slots, int64_t n, void *stream)
{
    ABI_BEGIN
    if (!ix || (n && !slots)) fail(GTS_EINVAL, "null argument");
    if (n == 0) return GTS_OK;
    CK(cudaSetDevice(ix->device));
    std::vector<int32_t> v(slots, slots + n);
    for (int32_t s : v) {
        if (s < 0 || s >= ix->n || ix->ord[(size_t)s] >= 0) fail(GTS_EINVAL, "slot %d was not filled by an insert", s);
        ix->h_alive[(size_t)(s >> 5)] &= ~(1u << (s & 31));
    }
    sync_alive(ix, v, (cudaStream_t)stream);
    return GTS_OK;
    ABI_END
}
