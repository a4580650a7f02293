// Native index build: a bit-identical restatement of tree.build_index
// (tree.py:164-189) and _try_split (tree.py:125-161), host C++.
//
// Series are inserted one by one in id order; every node on the path widens
// its envelope (summarize.py:90-94); a leaf above max_leaf_size splits on the
// segment with the widest envelope (first maximum, np.argmax) at the member
// median (np.median: middle order statistic, or the mean of the two middle
// ones), falling back to the mid-range, and is flagged oversized when neither
// separates its members.  Segment means use numpy's reduceat order
// (common.cuh: segment_mean), so every envelope and threshold is bit-equal to
// the reference and the node table is identical.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <thread>
#include <vector>

#include "common.cuh"

struct lf_tree {
    int n_seg = 0;
    int64_t cap = 0;
    int64_t n = 0;
    std::vector<double> env_min, env_max;       // [node][n_seg]
    std::vector<int32_t> left, right, split_seg;
    std::vector<double> split_thr;
    std::vector<int64_t> size;
    std::vector<int8_t> oversized;
    std::vector<std::vector<int64_t>> members;  // leaf members (ascending ids)
    std::vector<int8_t> is_leaf;
};

namespace {

void paa_rows(const float* v, int64_t n, int m, int l, double* out, int threads) {
    std::vector<int> st(l), w(l);
    const int base = m / l, rem = m % l;
    for (int i = 0, s = 0; i < l; ++i) {
        w[i] = base + (i < rem ? 1 : 0);
        st[i] = s;
        s += w[i];
    }
    auto work = [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; ++r)
            for (int i = 0; i < l; ++i) out[r * l + i] = lf::segment_mean(v + r * m, st[i], w[i]);
    };
    threads = std::max(1, threads);
    if (threads == 1 || n < 4096) {
        work(0, n);
        return;
    }
    std::vector<std::thread> pool;
    int64_t step = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        int64_t a = t * step, b = std::min(n, a + step);
        if (a < b) pool.emplace_back(work, a, b);
    }
    for (auto& th : pool) th.join();
}

int new_node(lf_tree& t) {
    const double inf = std::numeric_limits<double>::infinity();
    for (int i = 0; i < t.n_seg; ++i) {
        t.env_min.push_back(inf);
        t.env_max.push_back(-inf);
    }
    t.left.push_back(-1);
    t.right.push_back(-1);
    t.split_seg.push_back(-1);
    t.split_thr.push_back(std::numeric_limits<double>::quiet_NaN());
    t.size.push_back(0);
    t.oversized.push_back(0);
    t.members.emplace_back();
    t.is_leaf.push_back(1);
    return (int)t.left.size() - 1;
}

inline void widen(lf_tree& t, int node, const double* s) {
    double* mn = &t.env_min[(size_t)node * t.n_seg];
    double* mx = &t.env_max[(size_t)node * t.n_seg];
    for (int i = 0; i < t.n_seg; ++i) {
        mn[i] = std::min(mn[i], s[i]);   // np.minimum / np.maximum (no NaNs here)
        mx[i] = std::max(mx[i], s[i]);
    }
}

// tree.py:125-161
void try_split(lf_tree& t, int node, const double* summs) {
    const int l = t.n_seg;
    int seg = 0;
    double best = -std::numeric_limits<double>::infinity();
    for (int i = 0; i < l; ++i) {
        double wdt = t.env_max[(size_t)node * l + i] - t.env_min[(size_t)node * l + i];
        if (wdt > best) { best = wdt; seg = i; }              // first maximum
    }
    if (!(best > 0.0)) { t.oversized[node] = 1; return; }
    const std::vector<int64_t> ids = t.members[node];
    const size_t cnt = ids.size();
    std::vector<double> col(cnt);
    for (size_t i = 0; i < cnt; ++i) col[i] = summs[ids[i] * l + seg];
    std::vector<double> tmp(col);
    double thr;
    const size_t h = cnt / 2;
    std::nth_element(tmp.begin(), tmp.begin() + h, tmp.end());
    double hi = tmp[h];
    if (cnt % 2 == 1) {
        thr = hi;
    } else {
        double lo = *std::max_element(tmp.begin(), tmp.begin() + h);
        thr = (lo + hi) / 2.0;                                 // np.mean of the two middle values
    }
    auto count_left = [&](double th) {
        size_t c = 0;
        for (double v : col) c += (v <= th) ? 1 : 0;
        return c;
    };
    size_t nl = count_left(thr);
    if (nl == cnt || nl == 0) {
        double cmin = *std::min_element(col.begin(), col.end());
        double cmax = *std::max_element(col.begin(), col.end());
        thr = (cmin + cmax) / 2.0;
        nl = count_left(thr);
        if (nl == cnt || nl == 0) { t.oversized[node] = 1; return; }
    }
    const int a = new_node(t);
    const int b = new_node(t);
    for (size_t i = 0; i < cnt; ++i) {
        const int child = col[i] <= thr ? a : b;
        t.members[child].push_back(ids[i]);
        t.size[child] += 1;
        widen(t, child, summs + ids[i] * l);                    // NodeEnvelope.from_rows
    }
    t.members[node].clear();
    t.members[node].shrink_to_fit();
    t.is_leaf[node] = 0;
    t.split_seg[node] = seg;
    t.split_thr[node] = thr;
    t.left[node] = a;
    t.right[node] = b;
}

}  // namespace

extern "C" {

int lf_paa_host(const float* h_values, int64_t n, int32_t m, int32_t n_seg, double* h_out,
                int32_t n_threads) {
    LF_REQUIRE(n_seg >= 1 && n_seg <= m, "num_segments must be in [1, length]");
    paa_rows(h_values, n, m, n_seg, h_out, n_threads);
    return LF_OK;
}

static lf_tree* build_from(const double* summs, int64_t n, int32_t n_seg, int64_t max_leaf_size) {
    auto* t = new lf_tree();
    t->n_seg = n_seg;
    t->cap = max_leaf_size;
    t->n = n;
    new_node(*t);
    for (int64_t sid = 0; sid < n; ++sid) {
        const double* s = summs + sid * n_seg;
        int node = 0;
        while (!t->is_leaf[node]) {
            t->size[node] += 1;
            widen(*t, node, s);
            node = s[t->split_seg[node]] <= t->split_thr[node] ? t->left[node] : t->right[node];
        }
        t->members[node].push_back(sid);
        t->size[node] += 1;
        widen(*t, node, s);
        if (t->size[node] > t->cap) try_split(*t, node, summs);
    }
    return t;
}

lf_tree* lf_tree_build(const float* h_values, int64_t n, int32_t m, int32_t n_seg,
                       int64_t max_leaf_size, int32_t n_threads) {
    if (n < 1 || m < 2 || n_seg < 1 || n_seg > m || n_seg > LF_MAX_SEG || max_leaf_size < 2) {
        lf::fail(LF_EINVAL, "bad tree build arguments");
        return nullptr;
    }
    std::vector<double> summs((size_t)n * n_seg);
    paa_rows(h_values, n, m, n_seg, summs.data(), n_threads);
    return build_from(summs.data(), n, n_seg, max_leaf_size);
}

lf_tree* lf_tree_build_from_summaries(const double* h_summs, int64_t n, int32_t n_seg,
                                      int64_t max_leaf_size) {
    if (n < 1 || n_seg < 1 || n_seg > LF_MAX_SEG || max_leaf_size < 2) {
        lf::fail(LF_EINVAL, "bad tree build arguments");
        return nullptr;
    }
    return build_from(h_summs, n, n_seg, max_leaf_size);
}

int lf_tree_info(const lf_tree* t, int32_t* n_nodes, int32_t* n_leaves) {
    LF_REQUIRE(t != nullptr, "NULL tree");
    *n_nodes = (int32_t)t->left.size();
    int32_t c = 0;
    for (int8_t v : t->is_leaf) c += v;
    *n_leaves = c;
    return LF_OK;
}

int lf_tree_export(const lf_tree* t, double* env_min, double* env_max, int32_t* left,
                   int32_t* right, int32_t* split_seg, double* split_thr, int64_t* size,
                   int8_t* oversized, int64_t* member_ptr, int64_t* members) {
    LF_REQUIRE(t != nullptr, "NULL tree");
    const size_t nn = t->left.size();
    std::memcpy(env_min, t->env_min.data(), sizeof(double) * t->env_min.size());
    std::memcpy(env_max, t->env_max.data(), sizeof(double) * t->env_max.size());
    std::memcpy(left, t->left.data(), sizeof(int32_t) * nn);
    std::memcpy(right, t->right.data(), sizeof(int32_t) * nn);
    std::memcpy(split_seg, t->split_seg.data(), sizeof(int32_t) * nn);
    std::memcpy(split_thr, t->split_thr.data(), sizeof(double) * nn);
    std::memcpy(size, t->size.data(), sizeof(int64_t) * nn);
    std::memcpy(oversized, t->oversized.data(), sizeof(int8_t) * nn);
    int64_t off = 0;
    for (size_t i = 0; i < nn; ++i) {
        member_ptr[i] = off;
        if (t->is_leaf[i]) {
            std::memcpy(members + off, t->members[i].data(), sizeof(int64_t) * t->members[i].size());
            off += (int64_t)t->members[i].size();
        }
    }
    member_ptr[nn] = off;
    return LF_OK;
}

void lf_tree_free(lf_tree* t) { delete t; }

}  // extern "C"
