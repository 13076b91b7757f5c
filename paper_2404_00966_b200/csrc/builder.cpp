// builder.cpp -- host-side bulk builder of the flat pivot tree.
//
// Restates the reference construction (tree.py:241-367, _Builder) so the
// device tables index exactly the tree the reference would build:
//   * height / addressing ...... tree.py:60-108
//   * farthest-first pivots .... tree.py:293-310 (max chain_min, min id tie)
//   * level map ................ tree.py:311-317 (row_to_row distances, f64)
//   * one global keyed sort .... tree.py:319-334 (key dis/(max+1)+ordinal,
//                                object id as tie; runtime.py:149-185)
//   * child split + ranges ..... tree.py:336-367
// Distances are computed in float64 with numpy's row-sum order (vectors)
// or exactly (edit distance, via a bit-parallel Myers/Hyyro recurrence that
// returns the same integer as the reference DP, metrics.py:54-84).
// Compile with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>
#include <parallel/algorithm>
#include <omp.h>

#include "../../include/gts.h"
#include "common.h"

namespace gts {

// numpy pairwise_sum order (see oracle/gts_oracle.c for the derivation).
static double pw_sum(const double *a, int64_t n)
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
    return pw_sum(a, n2) + pw_sum(a + n2, n - n2);
}

// angular_row_pairs (metrics.py:175-193) with the dataset's pairwise norms
// (data.py:81-84): arccos(clip(dot / (|x| |q|))), zero-vector rules, and
// identical vectors forced to 0.  libm's acos: the reference's numpy arccos
// may differ in the last bits (see tests/test_angular.py).
static double host_angular(const double *x, const double *q, int64_t D, double *tmp)
{
    for (int64_t d = 0; d < D; d++) tmp[d] = x[d] * x[d];
    const double nx = std::sqrt(pw_sum(tmp, D));
    for (int64_t d = 0; d < D; d++) tmp[d] = q[d] * q[d];
    const double nq = std::sqrt(pw_sum(tmp, D));
    if (nx == 0.0 || nq == 0.0) return (nx == 0.0 && nq == 0.0) ? 0.0 : M_PI;
    for (int64_t d = 0; d < D; d++) tmp[d] = x[d] * q[d];
    double c = pw_sum(tmp, D) / (nx * nq);
    c = std::min(1.0, std::max(-1.0, c));
    double r = std::acos(c);
    if (r < 1e-6) {
        bool eq = true;
        for (int64_t d = 0; d < D && eq; d++) eq = x[d] == q[d];
        if (eq) r = 0.0;
    }
    return r;
}

double host_vec_dist(int metric, const double *x, const double *q, int64_t D, double *tmp)
{
    if (metric == GTS_ANGULAR) return host_angular(x, q, D, tmp);
    for (int64_t d = 0; d < D; d++) {
        double diff = x[d] - q[d];
        tmp[d] = (metric == GTS_L1) ? std::fabs(diff) : diff * diff;
    }
    double s = pw_sum(tmp, D);
    return metric == GTS_L1 ? s : std::sqrt(s);
}

// Myers/Hyyro block bit-vector edit distance, pattern p (dense symbols
// with precomputed peq[A][W]), text t.  Same integer as the DP.
struct HostPattern {
    int64_t m = 0, W = 0;
    std::vector<uint64_t> peq;  // [A*W]
};

static void make_pattern(const int32_t *p, int64_t m, int64_t A, HostPattern &hp)
{
    hp.m = m;
    hp.W = (m + 63) / 64;
    hp.peq.assign((size_t)(A * hp.W), 0);
    for (int64_t i = 0; i < m; i++) hp.peq[(size_t)(p[i] * hp.W + i / 64)] |= 1ull << (i % 64);
}

static int64_t myers_host(const HostPattern &hp, const int32_t *t, int64_t n,
                          std::vector<uint64_t> &P, std::vector<uint64_t> &M)
{
    const int64_t m = hp.m, W = hp.W;
    if (m == 0) return n;
    if (n == 0) return m;
    P.assign((size_t)W, ~0ull);
    M.assign((size_t)W, 0ull);
    const uint64_t last = 1ull << ((m - 1) % 64);
    int64_t score = m;
    for (int64_t j = 0; j < n; j++) {
        const uint64_t *eqrow = hp.peq.data() + (size_t)(t[j] * W);
        int hin = 1;  // top row D[0][j] = j: +1 per column
        for (int64_t b = 0; b < W; b++) {
            uint64_t Eq = eqrow[b], Pv = P[b], Mv = M[b];
            uint64_t Xv = Eq | Mv;
            if (hin < 0) Eq |= 1ull;
            uint64_t Xh = (((Eq & Pv) + Pv) ^ Pv) | Eq;
            uint64_t Ph = Mv | ~(Xh | Pv);
            uint64_t Mh = Pv & Xh;
            uint64_t hb = (b == W - 1) ? last : (1ull << 63);
            int hout = (Ph & hb) ? 1 : ((Mh & hb) ? -1 : 0);
            Ph <<= 1;
            Mh <<= 1;
            if (hin < 0) Mh |= 1ull;
            else if (hin > 0) Ph |= 1ull;
            P[b] = Mh | ~(Xv | Ph);
            M[b] = Ph & Xv;
            hin = hout;
        }
        score += hin;
    }
    return score;
}

// dense alphabet: sorted unique code points -> [0, A)
// sorted distinct code points: a presence table for code points < 2^16 (one
// pass, no sort of all n*len codes), a sort of the rest
void dense_alphabet(const int32_t *codes, int64_t ncodes, std::vector<int32_t> &alpha)
{
    std::vector<uint8_t> seen((size_t)1 << 16, 0);
    std::vector<int32_t> big;
    for (int64_t i = 0; i < ncodes; i++) {
        const int32_t c = codes[i];
        if (c >= 0 && c < (1 << 16)) seen[(size_t)c] = 1;
        else big.push_back(c);
    }
    std::sort(big.begin(), big.end());
    big.erase(std::unique(big.begin(), big.end()), big.end());
    alpha.clear();
    for (auto c : big) if (c < 0) alpha.push_back(c);
    for (int32_t c = 0; c < (1 << 16); c++) if (seen[(size_t)c]) alpha.push_back(c);
    for (auto c : big) if (c >= (1 << 16)) alpha.push_back(c);
}

}  // namespace gts

using namespace gts;

extern "C" int gts_tree_height(int64_t n, int64_t nc, int64_t *max_h, int64_t *split_rounds)
{
    if (nc < 2) return set_error(GTS_EINVAL, "node_capacity must be >= 2");
    if (n < 1) return set_error(GTS_EINVAL, "tree_height requires n >= 1");
    int64_t t = 0;
    __int128 power = 1;
    while (power < (__int128)n + 1) { power *= nc; t++; }
    *max_h = t - 1;
    *split_rounds = std::max<int64_t>(t - 2, 0);
    return GTS_OK;
}

extern "C" int64_t gts_node_count(int64_t levels, int64_t nc)
{
    __int128 p = 1;
    for (int64_t i = 0; i < levels; i++) p *= nc;
    return (int64_t)((p - 1) / (nc - 1));
}

static void level_range(int64_t level, int64_t nc, int64_t &first, int64_t &count)
{
    __int128 c = 1;
    for (int64_t i = 1; i < level; i++) c *= nc;
    count = (int64_t)c;
    first = (int64_t)((c - 1) / (nc - 1) + 1);
}

namespace {
struct KeyRec {
    double key;
    int64_t tie;
    int64_t idx;
    bool operator<(const KeyRec &o) const
    {
        if (key != o.key) return key < o.key;
        return tie < o.tie;
    }
};
}  // namespace

extern "C" int gts_build_tree(const gts_dataset *ds, int64_t root_row, int nthreads, gts_tree *t)
{
    try {
        if (!ds || !t) return set_error(GTS_EINVAL, "null argument");
        const int64_t n = ds->n, nc = t->nc;
        if (nc < 2) return set_error(GTS_EINVAL, "node_capacity must be >= 2");
        if (n == 0) { t->levels = 0; t->split_rounds = 0; return GTS_OK; }
        if (root_row < 0 || root_row >= n) return set_error(GTS_EINVAL, "root_row out of range");
        const bool edit = ds->metric == GTS_EDIT;
        if (!edit && ds->metric != GTS_L1 && ds->metric != GTS_L2 && ds->metric != GTS_ANGULAR)
            return set_error(GTS_EMETRIC, "builder supports edit, l1, l2, angular");
        if (nthreads > 0) omp_set_num_threads(nthreads);
        int64_t max_h, split;
        gts_tree_height(n, nc, &max_h, &split);
        t->split_rounds = split;
        t->levels = split + 1;
        const int64_t nodes = gts_node_count(t->levels, nc);
        if (t->nodes < nodes) return set_error(GTS_EINVAL, "tree arrays too small");
        for (int64_t i = 0; i <= nodes; i++) {
            t->pivot_id[i] = -1; t->pivot_row[i] = -1; t->min_dis[i] = 0; t->max_dis[i] = 0;
            t->pos[i] = 0; t->size[i] = 0;
        }
        t->size[1] = n;
        for (int64_t i = 0; i < n; i++) { t->rows[i] = i; t->dis[i] = 0; if (t->tombstone) t->tombstone[i] = 0; }

        // dense string symbols for the bit-parallel edit distance
        std::vector<int32_t> alpha, dense;
        int64_t A = 0;
        if (edit) {
            int64_t nc_codes = ds->offsets[n];
            dense_alphabet(ds->codes, nc_codes, alpha);
            A = (int64_t)alpha.size();
            dense.resize((size_t)std::max<int64_t>(nc_codes, 1));
            #pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < nc_codes; i++)
                dense[(size_t)i] = (int32_t)(std::lower_bound(alpha.begin(), alpha.end(), ds->codes[i]) - alpha.begin());
        }
        const int64_t D = ds->dim;
        std::vector<double> chain((size_t)n), tmpd((size_t)n);
        std::vector<int64_t> tmpr((size_t)n);
        std::vector<KeyRec> keys((size_t)n);
        bool have_chain = false;

        for (int64_t level = 1; level <= t->levels; level++) {
            int64_t first, count;
            level_range(level, nc, first, count);
            if (level == 1) {
                int64_t prow = t->rows[root_row];
                t->pivot_row[1] = prow;
                t->pivot_id[1] = ds->ids[prow];
            } else {
                #pragma omp parallel for schedule(dynamic, 16)
                for (int64_t node = first; node < first + count; node++) {
                    int64_t sz = t->size[node];
                    if (sz <= 0) continue;
                    int64_t p = t->pos[node];
                    double best = chain[(size_t)p];
                    for (int64_t e = p + 1; e < p + sz; e++) best = std::max(best, chain[(size_t)e]);
                    int64_t prow = -1, pid = 0;
                    for (int64_t e = p; e < p + sz; e++) {
                        if (chain[(size_t)e] == best) {
                            int64_t r = t->rows[e];
                            if (prow < 0 || ds->ids[r] < pid) { prow = r; pid = ds->ids[r]; }
                        }
                    }
                    t->pivot_row[node] = prow;
                    t->pivot_id[node] = pid;
                }
            }
            // map: every entry against its node's pivot.  Patterns are built
            // per node first, then the distances run in parallel over ENTRIES
            // (parallelising over nodes left the root level -- n distances of
            // one node -- on a single thread)
            std::vector<HostPattern> pats(edit ? (size_t)count : 0);
            #pragma omp parallel for schedule(dynamic, 16)
            for (int64_t o = 0; o < count; o++) {
                const int64_t node = first + o;
                const int64_t sz = t->size[node];
                if (sz > 0) {
                    if (edit) {
                        const int64_t pv = t->pivot_row[node];
                        make_pattern(dense.data() + ds->offsets[pv], ds->offsets[pv + 1] - ds->offsets[pv], A,
                                     pats[(size_t)o]);
                    }
                    for (int64_t e = t->pos[node]; e < t->pos[node] + sz; e++) tmpr[(size_t)e] = o;   // entry -> node
                }
            }
            #pragma omp parallel
            {
                std::vector<double> tmp((size_t)D + 1);
                std::vector<uint64_t> P, M;
                #pragma omp for schedule(dynamic, 2048)
                for (int64_t e = 0; e < n; e++) {
                    const int64_t o = tmpr[(size_t)e], r = t->rows[e];
                    if (edit) {
                        t->dis[e] = (double)myers_host(pats[(size_t)o], dense.data() + ds->offsets[r],
                                                       ds->offsets[r + 1] - ds->offsets[r], P, M);
                    } else {
                        const double *pvec = ds->vectors + t->pivot_row[first + o] * D;
                        t->dis[e] = host_vec_dist(ds->metric, ds->vectors + r * D, pvec, D, tmp.data());
                    }
                }
            }
            if (!have_chain) { std::copy(t->dis, t->dis + n, chain.begin()); have_chain = true; }
            else {
                #pragma omp parallel for schedule(static)
                for (int64_t e = 0; e < n; e++) chain[(size_t)e] = std::min(chain[(size_t)e], t->dis[e]);
            }
            // one global keyed sort over the whole level
            double lm = t->dis[0];
            for (int64_t e = 1; e < n; e++) lm = std::max(lm, t->dis[e]);
            const double denom = lm + 1.0;
            #pragma omp parallel for schedule(dynamic, 16)
            for (int64_t o = 0; o < count; o++) {
                int64_t node = first + o, p = t->pos[node];
                for (int64_t e = p; e < p + t->size[node]; e++) {
                    keys[(size_t)e].key = t->dis[e] / denom + (double)o;
                    keys[(size_t)e].tie = ds->ids[t->rows[e]];
                    keys[(size_t)e].idx = e;
                }
            }
            __gnu_parallel::sort(keys.begin(), keys.end());
            #pragma omp parallel for schedule(static)
            for (int64_t e = 0; e < n; e++) {
                tmpr[(size_t)e] = t->rows[keys[(size_t)e].idx];
                tmpd[(size_t)e] = t->dis[keys[(size_t)e].idx];
            }
            std::copy(tmpr.begin(), tmpr.end(), t->rows);
            std::copy(tmpd.begin(), tmpd.end(), t->dis);
            if (level < t->levels) {
                #pragma omp parallel for schedule(static)
                for (int64_t e = 0; e < n; e++) tmpd[(size_t)e] = chain[(size_t)keys[(size_t)e].idx];
                chain.swap(tmpd);
                const int64_t cfirst = (first - 1) * nc + 2;
                for (int64_t o = 0; o < count; o++) {
                    int64_t node = first + o, sz = t->size[node], p = t->pos[node];
                    int64_t avg = sz / nc;
                    for (int64_t j = 0; j < nc; j++) {
                        int64_t c = cfirst + o * nc + j;
                        t->pos[c] = p + j * avg;
                        t->size[c] = (j == nc - 1) ? sz - avg * (nc - 1) : avg;
                        if (t->size[c] > 0) {
                            t->min_dis[c] = t->dis[t->pos[c]];
                            t->max_dis[c] = t->dis[t->pos[c] + t->size[c] - 1];
                        }
                    }
                }
            } else {
                for (int64_t o = 0; o < count; o++) {
                    int64_t c = first + o;
                    if (t->size[c] > 0) {
                        t->min_dis[c] = t->dis[t->pos[c]];
                        t->max_dis[c] = t->dis[t->pos[c] + t->size[c] - 1];
                    }
                }
            }
        }
        return GTS_OK;
    } catch (const std::bad_alloc &) {
        return set_error(GTS_EOOM, "host allocation failed in gts_build_tree");
    } catch (...) {
        return set_error(GTS_EINVAL, "unexpected failure in gts_build_tree");
    }
}
