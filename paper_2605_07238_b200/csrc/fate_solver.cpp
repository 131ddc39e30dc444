// fate_solver.cpp -- native host frontier solve.
//
// Restates wfsched.planner.solve_frontier and its front half
// (/root/reference/pkg/src/wfsched/planner.py:101-234) in C++ on the packed
// cost matrix, with the reference's exact semantics:
//
//   _stage_options (planner.py:101-138): per stage, every slot->device chain
//     enumerated depth first (a chain is recorded before its extensions,
//     extensions in ascending device order -- the reference's
//     sorted((device_id, psi)) with device index = rank of the id), value
//     accumulated left to right; kept iff nonempty and value - prefix >= 0.0
//     for every proper prefix, the prefix summed like CPython 3.12's builtin
//     sum() (Neumaier, first term 0 + x; _prefix_values, planner.py:141-147).
//     Depth-first preorder over ascending devices IS the lexicographic order
//     of the triples, so the reference's kept.sort(key=triples) is the
//     enumeration order.
//   solve_frontier (planner.py:150-214): optimistic suffix bound, memoised
//     search over (stage index, used-device mask), skip first then options in
//     order, replace on a strictly larger total or an equal total with a
//     lexicographically smaller selection tuple; node counting identical; the
//     deadline is checked on memo misses; budget <= 0 times out at the first
//     miss exactly like the reference's zero budget.
//   _greedy_fallback (planner.py:217-234).
//
// Selections are never materialised during the search: a memo entry stores
// its choice, and tie-break comparisons walk the two choice chains lazily.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <atomic>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "fate.h"
#include "fate_internal.h"

namespace {

struct PySumH {  // CPython 3.12 builtin sum() over floats
    double s = 0.0, c = 0.0;
    int n = 0;
    void add(double x) {
        if (n == 0) {
            s = 0.0 + x;
        } else {
            const double t = s + x;
            if (std::fabs(s) >= std::fabs(x)) c += (s - t) + x;
            else c += (x - t) + s;
            s = t;
        }
        ++n;
    }
    double result() const {
        if (n == 0) return 0.0;
        return (c != 0.0 && std::isfinite(c)) ? s + c : s;
    }
};

struct Option {
    double value;
    uint64_t mask;
    int32_t t0, nt;  // triples [t0, t0+nt) in Stage::trip
};

struct Stage {
    std::vector<Option> opts;
    std::vector<int32_t> trip;  // (slot, device) pairs flattened
    double best = 0.0;          // max option value (default 0.0)
};

struct Memo {
    double val;
    int32_t choice;  // -1 = skip this stage
};

struct Solver {
    const fate_frontier* p;
    std::vector<Stage> st;
    std::vector<double> suffix;
    std::vector<std::unordered_map<uint64_t, Memo>> memo;
    int64_t nodes = 0;
    bool timed = false;
    std::chrono::steady_clock::time_point deadline;
    bool immediate = false;

    struct Timeout {};

    // selection chain cursor: triples of (i, mask) onwards
    struct Cursor {
        const Solver* S;
        int i;
        uint64_t mask;
        int opt = -1, k = 0;  // current option and triple within it
        bool valid = false;
        void settle() {
            // advance to the next stage that contributes a triple
            while (true) {
                if (opt >= 0 && k < S->st[i].opts[opt].nt) {
                    valid = true;
                    return;
                }
                if (opt >= 0) {  // finished this option: continue at i+1
                    mask |= S->st[i].opts[opt].mask;
                    ++i;
                    opt = -1;
                }
                if (i >= (int)S->st.size() || S->suffix[i] <= 0.0) {
                    valid = false;
                    return;
                }
                auto it = S->memo[i].find(mask);
                if (it == S->memo[i].end()) {  // cannot happen after a full solve
                    valid = false;
                    return;
                }
                if (it->second.choice < 0) {
                    ++i;
                    continue;
                }
                opt = it->second.choice;
                k = 0;
            }
        }
        // (stage, slot, device) of the current triple
        void get(int* a, int* b, int* c) const {
            const Option& o = S->st[i].opts[opt];
            *a = i;
            *b = S->st[i].trip[2 * (o.t0 + k)];
            *c = S->st[i].trip[2 * (o.t0 + k) + 1];
        }
        void next() {
            ++k;
            settle();
        }
    };

    // (option o of stage i) + selection(i+1, mask | o.mask)  vs  selection
    // given as choice ch at (i, mask): is the first lexicographically smaller?
    bool less_opt_vs(int i, uint64_t mask, int oa, int ob_or_skip) const {
        Cursor A{this, i, mask, oa, 0, false};
        A.settle();
        Cursor B{this, i, mask, ob_or_skip, 0, false};
        if (ob_or_skip < 0) {
            B.i = i + 1;
            B.opt = -1;
        }
        B.settle();
        while (A.valid && B.valid) {
            int a1, a2, a3, b1, b2, b3;
            A.get(&a1, &a2, &a3);
            B.get(&b1, &b2, &b3);
            if (a1 != b1) return a1 < b1;
            if (a2 != b2) return a2 < b2;
            if (a3 != b3) return a3 < b3;
            A.next();
            B.next();
        }
        return !A.valid && B.valid;  // a proper prefix is smaller
    }

    double best(int i, uint64_t mask) {
        ++nodes;
        const int n = (int)st.size();
        if (i == n) return 0.0;
        if (suffix[i] <= 0.0) return 0.0;
        auto hit = memo[i].find(mask);
        if (hit != memo[i].end()) return hit->second.val;
        if (immediate || (timed && std::chrono::steady_clock::now() > deadline)) throw Timeout{};
        double bval = best(i + 1, mask);
        int bch = -1;
        const Stage& S = st[i];
        for (int o = 0; o < (int)S.opts.size(); ++o) {
            const Option& op = S.opts[o];
            if (op.mask & mask) continue;
            const double sub = best(i + 1, mask | op.mask);
            const double tot = op.value + sub;
            if (tot > bval || (tot == bval && less_opt_vs(i, mask, o, bch))) {
                bval = tot;
                bch = o;
            }
        }
        memo[i][mask] = Memo{bval, bch};
        return bval;
    }
};

int build_options(const fate_frontier* p, Solver& S, int64_t max_options) {
    const int n = p->n_stages;
    S.st.assign(n, Stage());
    int64_t total = 0;
    std::vector<double> psis;
    std::vector<int32_t> path;  // (slot, device) pairs of the current chain
    for (int i = 0; i < n; ++i) {
        Stage& G = S.st[i];
        const int s0 = p->slot_ptr[i], s1 = p->slot_ptr[i + 1];
        const int nslots = s1 - s0;
        // iterative depth-first preorder; frame = (slot depth, next candidate)
        struct Frame {
            int slot, next;
            double value;
            uint64_t mask;
        };
        std::vector<Frame> stack;
        stack.push_back({0, 0, 0.0, 0ull});
        path.clear();
        psis.clear();
        // the root (empty chain) is recorded and dropped by the filter
        while (!stack.empty()) {
            Frame& f = stack.back();
            if (f.slot >= nslots) {  // no slot to extend with
                stack.pop_back();
                if (!path.empty()) {
                    path.resize(path.size() - 2);
                    psis.pop_back();
                }
                continue;
            }
            const int c0 = p->cand_ptr[s0 + f.slot], c1 = p->cand_ptr[s0 + f.slot + 1];
            int c = c0 + f.next;
            while (c < c1 && ((f.mask >> p->cand_dev[c]) & 1ull)) ++c;
            if (c >= c1) {
                stack.pop_back();
                if (!path.empty()) {
                    path.resize(path.size() - 2);
                    psis.pop_back();
                }
                continue;
            }
            f.next = c - c0 + 1;
            const int dev = p->cand_dev[c];
            const double value = f.value + p->cand_psi[c];
            const uint64_t mask = f.mask | (1ull << dev);
            const int slot = f.slot;
            path.push_back(slot);
            path.push_back(dev);
            psis.push_back(p->cand_psi[c]);
            // record this chain (preorder) if it passes the suffix filter
            bool keep = value - 0.0 >= 0.0;  // sum([]) == 0
            PySumH pref;
            for (size_t k = 0; keep && k + 1 < psis.size(); ++k) {
                pref.add(psis[k]);
                keep = value - pref.result() >= 0.0;
            }
            if (keep) {
                Option o;
                o.value = value;
                o.mask = mask;
                o.t0 = (int32_t)(G.trip.size() / 2);
                o.nt = (int32_t)(path.size() / 2);
                G.trip.insert(G.trip.end(), path.begin(), path.end());
                G.opts.push_back(o);
                if (++total > max_options) return FATE_ETOOBIG;
            }
            stack.push_back({slot + 1, 0, value, mask});
        }
        double b = 0.0;
        bool first = true;
        for (const Option& o : G.opts) {
            if (first || o.value > b) b = o.value;
            first = false;
        }
        G.best = first ? 0.0 : b;
    }
    return 0;
}

void greedy(const Solver& S, double* objective, std::vector<int32_t>* sel) {
    const int n = (int)S.st.size();
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    // key (-best, stage): stable sort on -best, ties by stage index
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return -S.st[a].best < -S.st[b].best; });
    uint64_t used = 0;
    double total = 0.0;
    for (int i : order) {
        const Stage& G = S.st[i];
        int pick = -1;
        for (int o = 0; o < (int)G.opts.size(); ++o) {
            const Option& op = G.opts[o];
            if (!(op.value > 0) || (op.mask & used)) continue;
            // min by (-value, triples): options are in triples order
            if (pick < 0 || -op.value < -G.opts[pick].value) pick = o;
        }
        if (pick < 0) continue;
        const Option& op = G.opts[pick];
        used |= op.mask;
        total += op.value;
        for (int k = 0; k < op.nt; ++k) {
            sel->push_back(i);
            sel->push_back(G.trip[2 * (op.t0 + k)]);
            sel->push_back(G.trip[2 * (op.t0 + k) + 1]);
        }
    }
    *objective = total;
}

}  // namespace

extern "C" {

int fate_solve_frontier(const fate_frontier* p, double budget_s, int64_t max_options,
                        fate_selection* out) {
    if (!p || !out || !out->stage || !out->slot || !out->device)
        return fate_internal_fail(FATE_EINVAL, "fate_solve_frontier: NULL argument");
    if (p->n_stages < 0 || p->n_devices < 1 || p->n_devices > FATE_MAX_DEVICES)
        return fate_internal_fail(FATE_EINVAL, "fate_solve_frontier: bad sizes");
    const int64_t n_cand = p->n_stages ? p->cand_ptr[p->slot_ptr[p->n_stages]] : 0;
    if (n_cand == 0)
        return fate_internal_fail(FATE_EINVAL, "solve_frontier requires a nonempty problem");
    for (int i = 0; i < p->n_stages; ++i)
        for (int k = p->slot_ptr[i]; k < p->slot_ptr[i + 1]; ++k)
            for (int c = p->cand_ptr[k]; c < p->cand_ptr[k + 1]; ++c) {
                if (p->cand_dev[c] < 0 || p->cand_dev[c] >= p->n_devices ||
                    (c > p->cand_ptr[k] && p->cand_dev[c] <= p->cand_dev[c - 1]))
                    return fate_internal_fail(
                        FATE_EINVAL, "fate_solve_frontier: slot devices must ascend, in range");
            }
    const auto t0 = std::chrono::steady_clock::now();
    Solver S;
    S.p = p;
    int rc = build_options(p, S, max_options > 0 ? max_options : (int64_t)1 << 26);
    if (rc) return fate_internal_fail(rc, "fate_solve_frontier: option count over max_options");
    const int n = p->n_stages;
    S.suffix.assign(n + 1, 0.0);
    for (int i = n - 1; i >= 0; --i) S.suffix[i] = S.suffix[i + 1] + std::max(0.0, S.st[i].best);
    S.memo.assign(n, {});
    S.immediate = !(budget_s > 0.0);
    S.timed = true;
    S.deadline = t0 + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                          std::chrono::duration<double>(budget_s > 0.0 ? budget_s : 0.0));
    std::vector<int32_t> sel;
    double objective = 0.0;
    int optimal = 1;
    try {
        objective = S.best(0, 0);
        // materialise the chosen chain
        Solver::Cursor c{&S, 0, 0ull, -1, 0, false};
        c.settle();
        while (c.valid) {
            int a, b, d;
            c.get(&a, &b, &d);
            sel.push_back(a);
            sel.push_back(b);
            sel.push_back(d);
            c.next();
        }
    } catch (Solver::Timeout&) {
        optimal = 0;
        sel.clear();
        greedy(S, &objective, &sel);
    }
    // FrontierSolution.selected = tuple(sorted(selection))
    const int m = (int)sel.size() / 3;
    std::vector<int> idx(m);
    for (int k = 0; k < m; ++k) idx[k] = k;
    std::sort(idx.begin(), idx.end(), [&](int a, int b) {
        for (int f = 0; f < 3; ++f)
            if (sel[3 * a + f] != sel[3 * b + f]) return sel[3 * a + f] < sel[3 * b + f];
        return false;
    });
    if (m > out->capacity)
        return fate_internal_fail(FATE_ETOOBIG, "fate_solve_frontier: selection over capacity");
    for (int k = 0; k < m; ++k) {
        out->stage[k] = sel[3 * idx[k]];
        out->slot[k] = sel[3 * idx[k] + 1];
        out->device[k] = sel[3 * idx[k] + 2];
    }
    out->n = m;
    out->optimal = optimal;
    out->objective = objective;
    out->nodes = S.nodes;
    out->n_options = 0;
    for (const Stage& G : S.st) out->n_options += (int64_t)G.opts.size();
    out->wall_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return 0;
}

// Many independent problems straight from a scored batch (one problem =
// one (instance, scenario) frontier, its work items consecutive and in
// stage order): each problem's CSR rows are rebuilt from the dense Psi rows
// (eligible devices ascending) and solved exactly like fate_solve_frontier,
// problems distributed over host threads.
int fate_solve_batch(const fate_solve_batch_args* a, fate_solve_batch_out* o) {
    if (!a || !o || !a->item_ptr || !a->item_bound || !a->item_elig || !a->psi_off || !a->psi ||
        !o->n_sel || !o->sel || !o->objective || !o->optimal)
        return fate_internal_fail(FATE_EINVAL, "fate_solve_batch: NULL argument");
    const int D = a->n_devices;
    if (a->n_problems < 0 || D < 1 || D > FATE_MAX_DEVICES)
        return fate_internal_fail(FATE_EINVAL, "fate_solve_batch: bad sizes");
    int nt = a->n_threads > 0 ? a->n_threads : (int)std::thread::hardware_concurrency();
    nt = std::max(1, std::min(nt, std::max(1, a->n_problems)));
    std::atomic<int> next{0};
    std::atomic<int> status{0};
    std::string first_error;
    std::atomic<bool> have_error{false};
    auto work = [&]() {
        std::vector<int32_t> slot_ptr, cand_ptr, cand_dev, st, sl, dv;
        std::vector<double> cand_psi;
        st.resize(D);
        sl.resize(D);
        dv.resize(D);
        for (;;) {
            const int p = next.fetch_add(1);
            if (p >= a->n_problems || status.load() != 0) return;
            slot_ptr.assign(1, 0);
            cand_ptr.assign(1, 0);
            cand_dev.clear();
            cand_psi.clear();
            const int i0 = a->item_ptr[p], i1 = a->item_ptr[p + 1];
            for (int i = i0; i < i1; ++i) {
                const uint64_t m = a->item_elig[i];
                for (int k = 0; k < a->item_bound[i]; ++k) {
                    const double* row = a->psi + a->psi_off[i] + (int64_t)k * D;
                    for (int d = 0; d < D; ++d)
                        if ((m >> d) & 1ull) {
                            cand_dev.push_back(d);
                            cand_psi.push_back(row[d]);
                        }
                    cand_ptr.push_back((int32_t)cand_dev.size());
                }
                slot_ptr.push_back((int32_t)cand_ptr.size() - 1);
            }
            fate_frontier fr{i1 - i0, D, slot_ptr.data(), cand_ptr.data(), cand_dev.data(),
                             cand_psi.data()};
            fate_selection out{D, 0, st.data(), sl.data(), dv.data(), 0.0, 0, 0, 0, 0, 0.0};
            const int rc = fate_solve_frontier(&fr, a->budget_s, a->max_options, &out);
            if (rc) {
                bool expect = false;
                if (have_error.compare_exchange_strong(expect, true))
                    first_error = fate_last_error();
                status.store(rc);
                return;
            }
            o->n_sel[p] = out.n;
            for (int k = 0; k < out.n; ++k) {
                int32_t* t = o->sel + ((int64_t)p * D + k) * 3;
                t[0] = i0 + out.stage[k];  // work item of the selected stage
                t[1] = out.slot[k];
                t[2] = out.device[k];
            }
            o->objective[p] = out.objective;
            o->optimal[p] = out.optimal;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    o->wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    o->threads = nt;
    if (status.load() != 0) return fate_internal_fail(status.load(), first_error);
    return 0;
}

}  // extern "C"
