// Host control plane: static allocation (a1) and the self-adaptive controller (a10).
//
// Paper: static allocation §3.1, D_i = D·w_i/Σw, total batch minibatch·Σw;
// Algorithm 1, Eq. 10, integer rounding, stop rule.
// Readings: #1 unit of w, #3 Hamilton rounding with ties to the lowest rank, #6 first
// epoch, #7 stop rule, #9 exact-integer shard sizes, #10 epoch remainder, #34 floor clamping,
// #35 fixed fp64 operation order (compiled with -ffp-contract=off); #49 the affine step-cost model
// (PR_ALLOC_MODEL_AFFINE, an opt-in extension of Eq. 8-10 for steps with a fixed per-step cost).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <new>
#include <utility>
#include <vector>

#include "common.h"

struct pr_alloc {
    int64_t N = 0;
    int32_t P = 0;
    int64_t C = 0, g = 1, floor = 1;
    int64_t epoch = 0;
    int32_t frozen = 0;
    pr_alloc_policy policy{2, 0, 1, 1.0, PR_ALLOC_MODEL_PROPORTIONAL, 8};
    std::vector<int64_t> w;                  // current allocation, units
    std::vector<std::vector<int64_t>> hist;  // allocation history (initial vector first)
    std::vector<double> t_prev;              // EMA state (empty until the first successful update)
    std::vector<std::vector<double>> t_hist; // t used by update k (hist[k] was in effect): hist.size() − 1 rows
};

namespace {

// Indices of the `left` largest keys; ties -> lowest index.  key compare is exact (integers or
// exactly-computed doubles).
template <typename K>
std::vector<char> pick_largest(const std::vector<K>& key, int64_t left) {
    const int64_t n = (int64_t)key.size();
    std::vector<int64_t> order(n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return key[a] > key[b]; });
    std::vector<char> pick(n, 0);
    for (int64_t i = 0; i < left && i < n; ++i) pick[order[i]] = 1;
    return pick;
}

// Largest remainder over exact rationals num_i/den summing to total (shard sizes).
int hamilton_exact(const std::vector<int64_t>& num, int64_t den, int64_t total, std::vector<int64_t>& out) {
    const size_t n = num.size();
    std::vector<int64_t> base(n), rem(n);
    int64_t sb = 0;
    for (size_t i = 0; i < n; ++i) {
        base[i] = num[i] / den;
        rem[i] = num[i] % den;
        sb += base[i];
    }
    const int64_t left = total - sb;
    if (left < 0 || left > (int64_t)n) return PR_ERR_INTERNAL;
    auto pick = pick_largest(rem, left);
    out.assign(n, 0);
    for (size_t i = 0; i < n; ++i) out[i] = base[i] + (pick[i] ? 1 : 0);
    return PR_OK;
}

int hamilton_plain(const std::vector<double>& q, int64_t total, std::vector<int64_t>& out) {
    const size_t n = q.size();
    std::vector<int64_t> base(n);
    std::vector<double> frac(n);
    int64_t sb = 0;
    for (size_t i = 0; i < n; ++i) {
        const double f = std::floor(q[i]);
        base[i] = (int64_t)f;
        frac[i] = q[i] - f;  // exact for q >= 0
        sb += base[i];
    }
    const int64_t left = total - sb;
    if (left < 0 || left > (int64_t)n) return PR_ERR_INTERNAL;
    auto pick = pick_largest(frac, left);
    out.assign(n, 0);
    for (size_t i = 0; i < n; ++i) out[i] = base[i] + (pick[i] ? 1 : 0);
    return PR_OK;
}

// Largest remainder with a floor: clamp violators, re-apportion the rest with q_i·T'/S (S = Σ of the
// active original quotas left to right; product first, then division).
int hamilton(const std::vector<double>& q, int64_t total, int64_t floor, std::vector<int64_t>& out) {
    const int64_t n = (int64_t)q.size();
    if (total < n * floor) return PR_ERR_INFEASIBLE_FLOOR;
    std::vector<char> fixed(n, 0);
    for (;;) {
        std::vector<int64_t> active;
        for (int64_t i = 0; i < n; ++i)
            if (!fixed[i]) active.push_back(i);
        if (active.empty()) return PR_ERR_INTERNAL;
        const int64_t t_rem = total - floor * (n - (int64_t)active.size());
        std::vector<double> qa;
        if ((int64_t)active.size() == n) {
            qa = q;
        } else {
            double s = 0.0;
            for (int64_t i : active) s = s + q[i];
            for (int64_t i : active) qa.push_back((q[i] * (double)t_rem) / s);
        }
        std::vector<int64_t> a;
        int rc = hamilton_plain(qa, t_rem, a);
        if (rc) return rc;
        bool viol = false;
        for (size_t j = 0; j < active.size(); ++j)
            if (a[j] < floor) { fixed[active[j]] = 1; viol = true; }
        if (!viol) {
            out.assign(n, floor);
            for (size_t j = 0; j < active.size(); ++j) out[active[j]] = a[j];
            return PR_OK;
        }
    }
}

void shard_sizes(const pr_alloc* a, int64_t* len, int64_t* off) {
    std::vector<int64_t> num(a->P), out;
    for (int32_t i = 0; i < a->P; ++i) num[i] = a->N * a->w[i];  // N·w_i <= 2^62 checked at init
    hamilton_exact(num, a->C, a->N, out);
    int64_t acc = 0;
    for (int32_t i = 0; i < a->P; ++i) { len[i] = out[i]; off[i] = acc; acc += out[i]; }
}

bool is_stable(const pr_alloc* a) {
    const int64_t W = a->policy.window;
    if ((int64_t)a->hist.size() < W) return false;
    const size_t s0 = a->hist.size() - (size_t)W;
    for (size_t i = s0; i < a->hist.size(); ++i)
        for (size_t j = i + 1; j < a->hist.size(); ++j)
            for (int32_t r = 0; r < a->P; ++r) {
                int64_t d = a->hist[i][r] - a->hist[j][r];
                if (d < 0) d = -d;
                if (d > a->policy.tol) return false;
            }
    return true;
}

// ---- affine step-cost model (DESIGN.md §3 #49) ------------------------------------------------------
// Rank i's epoch time as a function of its units: t_i(w) = a_i + b_i·w, fitted by least squares over its
// last `fit_window` observations (w in effect, t measured), fixed fp64 order.  Returns false when the
// observations hold fewer than two distinct w (no slope can be estimated).  A fit with b <= 0 or a < 0 (noise)
// falls back to the proportional model of Eq. 8 through the latest observation: a = 0, b = t/w.
bool affine_fit(const std::vector<const std::vector<int64_t>*>& ow, const std::vector<const std::vector<double>*>& ot,
                int32_t i, double& a_out, double& b_out) {
    const size_t n = ow.size();
    bool distinct = false;
    for (size_t k = 1; k < n; ++k)
        if ((*ow[k])[i] != (*ow[0])[i]) distinct = true;
    if (!distinct) return false;
    double sw = 0.0, st = 0.0;
    for (size_t k = 0; k < n; ++k) { sw = sw + (double)(*ow[k])[i]; st = st + (*ot[k])[i]; }
    const double mw = sw / (double)n, mt = st / (double)n;
    double sxx = 0.0, sxy = 0.0;
    for (size_t k = 0; k < n; ++k) {
        const double d = (double)(*ow[k])[i] - mw;
        sxx = sxx + d * d;
        sxy = sxy + d * ((*ot[k])[i] - mt);
    }
    const double b = sxy / sxx;
    const double a = mt - b * mw;
    if (b > 0.0 && a >= 0.0 && std::isfinite(a) && std::isfinite(b)) {
        a_out = a;
        b_out = b;
    } else {
        a_out = 0.0;
        b_out = (*ot[n - 1])[i] / (double)(*ow[n - 1])[i];
    }
    return true;
}

// min over integer w (Σw = C, w_i >= floor) of max_i (a_i + b_i·w_i), b_i > 0: start every rank at the
// floor and hand out the remaining units one at a time to the rank whose cost after taking it is the
// smallest (ties -> lowest rank).  With increasing costs the k-th unit handed out is the k-th smallest
// marginal cost, so the final maximum is the minimum possible (greedy is exact for min-max).
// A binary heap keyed on (cost after the next unit, rank) gives the same choice as a scan for the smallest
// cost with ties to the lowest rank, in O(C log P) (C may be 2^20).
void minmax_greedy(const std::vector<double>& a, const std::vector<double>& b, int64_t C, int64_t floor,
                   std::vector<int64_t>& w) {
    const size_t P = a.size();
    w.assign(P, floor);
    using Key = std::pair<double, size_t>;
    std::vector<Key> heap;
    heap.reserve(P);
    for (size_t i = 0; i < P; ++i) heap.push_back({a[i] + b[i] * (double)(w[i] + 1), i});
    auto after = [](const Key& x, const Key& y) { return x.first > y.first || (x.first == y.first && x.second > y.second); };
    std::make_heap(heap.begin(), heap.end(), after);                   // top = smallest (cost, rank)
    for (int64_t left = C - (int64_t)P * floor; left > 0; --left) {
        std::pop_heap(heap.begin(), heap.end(), after);
        const size_t i = heap.back().second;
        w[i] += 1;
        heap.back() = {a[i] + b[i] * (double)(w[i] + 1), i};
        std::push_heap(heap.begin(), heap.end(), after);
    }
}

}  // namespace

extern "C" int pr_alloc_init(pr_alloc** out, int64_t N, int32_t P, const double* ratios, int64_t C, int64_t g,
                             int64_t floor) {
    if (!out || !ratios || P < 1 || P > PR_MAX_RANKS || N < 1 || g < 1 || floor < 0 || C < 0) return PR_ERR_INVALID;
    if (N > ((int64_t)1 << 40)) return PR_ERR_INVALID;
    for (int32_t i = 0; i < P; ++i)
        if (!std::isfinite(ratios[i]) || !(ratios[i] > 0.0)) return PR_ERR_INVALID;
    if (C == 0) {
        int64_t s = 0;
        for (int32_t i = 0; i < P; ++i) {
            if (ratios[i] != std::floor(ratios[i]) || ratios[i] > 1e15) return PR_ERR_INVALID;
            s += (int64_t)ratios[i];
        }
        C = s;
    }
    if (C > ((int64_t)1 << 20)) return PR_ERR_INVALID;
    if (C < (int64_t)P * floor) return PR_ERR_INFEASIBLE_FLOOR;
    if (g > ((int64_t)1 << 30) || N < g * C) return PR_ERR_DATASET_TOO_SMALL;
    double s = 0.0;
    for (int32_t i = 0; i < P; ++i) s = s + ratios[i];
    std::vector<double> q(P);
    for (int32_t i = 0; i < P; ++i) q[i] = ((double)C * ratios[i]) / s;
    std::vector<int64_t> w;
    int rc = hamilton(q, C, floor, w);
    if (rc) return rc;
    pr_alloc* a = new (std::nothrow) pr_alloc();
    if (!a) return PR_ERR_INTERNAL;
    a->N = N; a->P = P; a->C = C; a->g = g; a->floor = floor;
    a->w = w;
    a->hist.push_back(w);
    *out = a;
    return PR_OK;
}

namespace {
bool policy_ok(const pr_alloc_policy& p, int64_t floor) {
    return p.window >= 2 && p.tol >= 0 && p.ema_alpha > 0.0 && p.ema_alpha <= 1.0 &&
           (p.model == PR_ALLOC_MODEL_PROPORTIONAL || (p.model == PR_ALLOC_MODEL_AFFINE && floor >= 1)) &&
           p.fit_window >= 2 && p.fit_window <= 64 && (p.never_freeze == 0 || p.never_freeze == 1);
}
}  // namespace

extern "C" int pr_alloc_set_policy(pr_alloc* a, const pr_alloc_policy* p) {
    if (!a || !p || !policy_ok(*p, a->floor)) return PR_ERR_INVALID;
    a->policy = *p;
    return PR_OK;
}

extern "C" int pr_alloc_update(pr_alloc* a, const double* t_s, int32_t* changed) {
    if (!a || !t_s) return PR_ERR_INVALID;
    if (a->frozen) {
        if (changed) *changed = 0;
        return PR_OK;
    }
    const int32_t P = a->P;
    std::vector<double> t(t_s, t_s + P);
    for (int32_t i = 0; i < P; ++i)
        if (!std::isfinite(t[i]) || !(t[i] > 0.0)) return PR_ERR_ZERO_TIMING;
    if (a->policy.ema_alpha != 1.0 && !a->t_prev.empty()) {
        const double al = a->policy.ema_alpha;
        for (int32_t i = 0; i < P; ++i) t[i] = al * t[i] + (1.0 - al) * a->t_prev[i];
    }
    std::vector<int64_t> w2;
    bool done = false;
    if (a->policy.model == PR_ALLOC_MODEL_AFFINE) {
        // observations (w in effect, t measured): the last fit_window of the history plus this epoch's
        std::vector<const std::vector<int64_t>*> ow;
        std::vector<const std::vector<double>*> ot;
        const size_t nh = a->t_hist.size();
        const size_t keep = (size_t)a->policy.fit_window - 1;
        for (size_t k = nh > keep ? nh - keep : 0; k < nh; ++k) { ow.push_back(&a->hist[k]); ot.push_back(&a->t_hist[k]); }
        ow.push_back(&a->w);
        ot.push_back(&t);
        std::vector<double> ca(P), cb(P);
        bool any = false;
        for (int32_t i = 0; i < P; ++i) {
            if (affine_fit(ow, ot, i, ca[i], cb[i])) {
                any = true;
            } else {
                ca[i] = 0.0;                                   // one w seen: Eq. 8's proportional model
                cb[i] = t[i] / (double)a->w[i];
            }
        }
        if (any) {                                             // else: no slope anywhere -> Eq. 10 below
            minmax_greedy(ca, cb, a->C, a->floor, w2);
            done = true;
        }
    }
    if (!done) {
        // Eq. 10: v_i = w_i/t_i; S_v left to right; q_i = (C·v_i)/S_v.
        std::vector<double> v(P), q(P);
        for (int32_t i = 0; i < P; ++i) v[i] = (double)a->w[i] / t[i];
        double sv = 0.0;
        for (int32_t i = 0; i < P; ++i) sv = sv + v[i];
        for (int32_t i = 0; i < P; ++i) q[i] = ((double)a->C * v[i]) / sv;
        int rc = hamilton(q, a->C, a->floor, w2);
        if (rc) return rc;
    }
    const int32_t ch = (w2 != a->w) ? 1 : 0;
    a->t_prev = t;
    a->t_hist.push_back(t);
    a->w = w2;
    a->hist.push_back(w2);
    a->epoch += 1;
    if (!a->policy.never_freeze && is_stable(a)) a->frozen = 1;
    if (changed) *changed = ch;
    return PR_OK;
}

extern "C" int pr_alloc_query(const pr_alloc* a, pr_alloc_view* v) {
    if (!a || !v) return PR_ERR_INVALID;
    pr_alloc_view o;
    std::memset(&o, 0, sizeof(o));
    o.N = a->N; o.P = a->P; o.frozen = a->frozen; o.C = a->C; o.g = a->g; o.floor = a->floor;
    o.B = a->g * a->C;
    o.S = a->N / o.B;
    o.epoch = a->epoch;
    o.hist_len = (int64_t)a->hist.size();
    for (int32_t i = 0; i < a->P; ++i) { o.w[i] = a->w[i]; o.n[i] = a->g * a->w[i]; }
    shard_sizes(a, o.len, o.off);
    *v = o;
    return PR_OK;
}

extern "C" int pr_alloc_history(const pr_alloc* a, int64_t k, int64_t* w_out) {
    if (!a || !w_out || k < 0 || k >= (int64_t)a->hist.size()) return PR_ERR_INVALID;
    for (int32_t i = 0; i < a->P; ++i) w_out[i] = a->hist[(size_t)k][i];
    return PR_OK;
}

// ---- checkpoint: little-endian POD ---------------------------------------------------------------
namespace {
constexpr uint64_t kMagic = 0x31434f4c4c415250ull;  // "PRALLOC1"
struct SaveHeader {
    uint64_t magic;
    uint32_t version, P;
    int64_t N, C, g, floor, epoch;
    int32_t frozen, has_tprev;
    pr_alloc_policy policy;
    int64_t hist_len;
};
}  // namespace

extern "C" int pr_alloc_save(const pr_alloc* a, void* buf, size_t cap, size_t* size) {
    if (!a || !size) return PR_ERR_INVALID;
    const size_t need = sizeof(SaveHeader) + sizeof(int64_t) * a->P * (1 + a->hist.size()) +
                        sizeof(double) * a->P * a->hist.size();   // t_prev + t_hist (hist_len − 1 rows)
    if (!buf) { *size = need; return PR_OK; }
    if (cap < need) return PR_ERR_CAPACITY;
    SaveHeader h;
    std::memset(&h, 0, sizeof(h));
    h.magic = kMagic; h.version = PR_VERSION; h.P = (uint32_t)a->P;
    h.N = a->N; h.C = a->C; h.g = a->g; h.floor = a->floor; h.epoch = a->epoch;
    h.frozen = a->frozen; h.has_tprev = a->t_prev.empty() ? 0 : 1; h.policy = a->policy;
    h.hist_len = (int64_t)a->hist.size();
    char* p = (char*)buf;
    std::memcpy(p, &h, sizeof(h)); p += sizeof(h);
    std::memcpy(p, a->w.data(), sizeof(int64_t) * a->P); p += sizeof(int64_t) * a->P;
    for (auto& v : a->hist) { std::memcpy(p, v.data(), sizeof(int64_t) * a->P); p += sizeof(int64_t) * a->P; }
    std::vector<double> tp(a->P, 0.0);
    if (!a->t_prev.empty()) tp = a->t_prev;
    std::memcpy(p, tp.data(), sizeof(double) * a->P); p += sizeof(double) * a->P;
    for (auto& v : a->t_hist) { std::memcpy(p, v.data(), sizeof(double) * a->P); p += sizeof(double) * a->P; }
    *size = need;
    return PR_OK;
}

// Validates everything pr_alloc_init / pr_alloc_set_policy would have refused, so a corrupt or hostile
// buffer cannot reach a division by zero (C or g = 0), an N·w overflow, or an allocation failure that
// would throw across the C ABI.
extern "C" int pr_alloc_load(pr_alloc** out, const void* buf, size_t size) {
    if (!out || !buf || size < sizeof(SaveHeader)) return PR_ERR_INVALID;
    SaveHeader h;
    std::memcpy(&h, buf, sizeof(h));
    if (h.magic != kMagic || h.version != PR_VERSION || h.P < 1 || h.P > PR_MAX_RANKS || h.hist_len < 1)
        return PR_ERR_INVALID;
    // same bounds as pr_alloc_init
    if (h.N < 1 || h.N > ((int64_t)1 << 40) || h.C < 1 || h.C > ((int64_t)1 << 20) || h.g < 1 ||
        h.g > ((int64_t)1 << 30) || h.floor < 0 || h.C < (int64_t)h.P * h.floor || h.N < h.g * h.C || h.epoch < 0 ||
        (h.frozen != 0 && h.frozen != 1) || h.has_tprev != (h.hist_len > 1 ? 1 : 0))
        return PR_ERR_INVALID;
    // same bounds as pr_alloc_set_policy
    if (!policy_ok(h.policy, h.floor)) return PR_ERR_INVALID;
    // size check without overflow: (1 + hist_len)·P int64 (w, history) + hist_len·P doubles (t_prev, t_hist)
    const size_t row = sizeof(int64_t) * h.P;
    const size_t drow = sizeof(double) * h.P;
    const size_t fixed = sizeof(SaveHeader) + row;
    if (size < fixed || (uint64_t)h.hist_len > (size - fixed) / (row + drow) ||
        size != fixed + (row + drow) * (size_t)h.hist_len)
        return PR_ERR_INVALID;
    const char* p = (const char*)buf + sizeof(h);
    // every allocation vector (current and history) must be one pr_alloc could have produced: Σw = C, w >= floor
    auto valid_w = [&](const char* q) {
        int64_t sum = 0;
        for (uint32_t i = 0; i < h.P; ++i) {
            int64_t w;
            std::memcpy(&w, q + sizeof(int64_t) * i, sizeof(w));
            if (w < h.floor || w > h.C) return false;
            sum += w;
        }
        return sum == h.C;
    };
    for (int64_t k = 0; k <= h.hist_len; ++k)
        if (!valid_w(p + row * (size_t)k)) return PR_ERR_INVALID;
    std::vector<double> tp(h.P);
    std::memcpy(tp.data(), p + row * (size_t)(1 + h.hist_len), sizeof(double) * h.P);
    if (h.has_tprev)
        for (double t : tp)
            if (!std::isfinite(t) || !(t > 0.0)) return PR_ERR_INVALID;
    const char* th = p + row * (size_t)(1 + h.hist_len) + drow;      // t_hist rows
    for (int64_t k = 0; k + 1 < h.hist_len; ++k)
        for (uint32_t i = 0; i < h.P; ++i) {
            double t;
            std::memcpy(&t, th + drow * (size_t)k + sizeof(double) * i, sizeof(t));
            if (!std::isfinite(t) || !(t > 0.0)) return PR_ERR_INVALID;
        }
    pr_alloc* a = new (std::nothrow) pr_alloc();
    if (!a) return PR_ERR_INTERNAL;
    try {
        a->N = h.N; a->P = (int32_t)h.P; a->C = h.C; a->g = h.g; a->floor = h.floor; a->epoch = h.epoch;
        a->frozen = h.frozen; a->policy = h.policy;
        a->w.resize(h.P);
        std::memcpy(a->w.data(), p, row); p += row;
        a->hist.resize((size_t)h.hist_len, std::vector<int64_t>(h.P));
        for (auto& v : a->hist) { std::memcpy(v.data(), p, row); p += row; }
        if (h.has_tprev) a->t_prev = tp;
        a->t_hist.resize((size_t)(h.hist_len - 1), std::vector<double>(h.P));
        for (auto& v : a->t_hist) { std::memcpy(v.data(), th, drow); th += drow; }
    } catch (...) {   // std::bad_alloc must not cross the C ABI
        delete a;
        return PR_ERR_INTERNAL;
    }
    *out = a;
    return PR_OK;
}

extern "C" void pr_alloc_destroy(pr_alloc* a) { delete a; }

// Used by the sharder (shard.cu) to read the shard of one rank without exposing the struct.
int pr_internal_shard_range(const pr_alloc* a, int32_t rank, int64_t* N, int64_t* off, int64_t* len) {
    if (!a || rank < 0 || rank >= a->P) return PR_ERR_INVALID;
    std::vector<int64_t> l(a->P), o(a->P);
    shard_sizes(a, l.data(), o.data());
    *N = a->N; *off = o[rank]; *len = l[rank];
    return PR_OK;
}

int pr_internal_step_layout(const pr_alloc* a, int32_t rank, int64_t* N, int64_t* B, int64_t* S, int64_t* o,
                            int64_t* n) {
    if (!a || rank < 0 || rank >= a->P) return PR_ERR_INVALID;
    int64_t units = 0;
    for (int32_t i = 0; i < rank; ++i) units += a->w[i];
    *N = a->N; *B = a->g * a->C; *S = a->N / (a->g * a->C);
    *o = a->g * units; *n = a->g * a->w[rank];
    return PR_OK;
}
