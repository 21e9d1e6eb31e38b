// context.cpp -- device context per host thread, shared packing helpers.
#include "context.hpp"

#include <map>

namespace quant {
namespace {
thread_local int t_device = 0;
thread_local int t_budget = 0;

struct Contexts {
    std::map<int, cqg_ctx *> by_device;
    ~Contexts() {
        for (auto &kv : by_device) cqg_destroy(kv.second);
    }
};
thread_local Contexts t_contexts;
} // namespace

void set_device(int device) { t_device = device; }

void set_sm_budget(int sms) {
    if (sms < 0) throw std::invalid_argument("set_sm_budget: negative SM count");
    t_budget = sms;
    auto it = t_contexts.by_device.find(t_device);
    if (it != t_contexts.by_device.end()) detail::check(cqg_set_sm_budget(it->second, sms));
}

namespace detail {

int current_device() { return t_device; }

cqg_ctx *ctx() {
    auto it = t_contexts.by_device.find(t_device);
    if (it != t_contexts.by_device.end()) return it->second;
    cqg_ctx *c = cqg_create(t_device);
    if (!c) throw std::runtime_error(std::string("libcqg: ") + cqg_last_error());
    t_contexts.by_device[t_device] = c;
    if (t_budget > 0) check(cqg_set_sm_budget(c, t_budget));
    return c;
}

bool on_grid(std::span<const ColorPoint> pts) {
    for (const ColorPoint &p : pts)
        for (double v : {p.r, p.g, p.b})
            if (!(v >= 0.0 && v <= 255.0) || v != static_cast<double>(static_cast<int>(v))) return false;
    return true;
}

std::vector<std::uint32_t> pack_all(std::span<const ColorPoint> pts) {
    std::vector<std::uint32_t> out(pts.size());
    for (std::size_t i = 0; i < pts.size(); ++i) out[i] = pack(pts[i]);
    return out;
}

cqg_term to_term(const ClusterOptions &o) {
    const Termination &t = o.term;
    if (t.fixed_iterations && *t.fixed_iterations <= 0) throw std::invalid_argument("clustering: fixed_iterations < 1");
    cqg_term ct{};
    ct.epsilon = t.epsilon;
    ct.max_iterations = t.max_iterations;
    ct.fixed_iterations = t.fixed_iterations ? *t.fixed_iterations : 0;
    ct.record_history = o.record_history ? 1 : 0;
    return ct;
}

ClusterState make_state(const std::vector<double> &cen, std::size_t k, const std::vector<std::uint32_t> &labels,
                        std::size_t n, const std::vector<double> &sse, const cqg_lloyd_stats &st,
                        const std::vector<std::uint32_t> &hl, const std::vector<double> &hc) {
    ClusterState s;
    s.centers = unflatten(cen.data(), k);
    s.memberships.assign(labels.begin(), labels.begin() + static_cast<std::ptrdiff_t>(n));
    s.sse_trace.assign(sse.begin(), sse.begin() + st.iterations);
    s.iterations = st.iterations;
    s.ndc_total = st.ndc_total;
    s.repair_count = st.repair_count;
    if (!hl.empty())
        for (int it = 0; it < st.iterations; ++it) {
            IterationSnapshot snap;
            snap.centers = unflatten(hc.data() + static_cast<std::size_t>(it) * 3 * k, k);
            snap.memberships.assign(hl.begin() + static_cast<std::ptrdiff_t>(it * n),
                                    hl.begin() + static_cast<std::ptrdiff_t>((it + 1) * n));
            s.history.push_back(std::move(snap));
        }
    return s;
}

ClusterState lloyd_counts(const std::vector<std::uint32_t> &packed, const std::vector<std::uint32_t> &counts,
                          std::uint64_t P, std::span<const ColorPoint> init, const ClusterOptions &options) {
    const cqg_term term = to_term(options);
    const std::size_t n = packed.size(), k = init.size();
    const int limit = term.fixed_iterations > 0 ? term.fixed_iterations : std::max(term.max_iterations, 1);
    std::vector<double> in = flatten(init), cen(3 * std::max<std::size_t>(k, 1));
    std::vector<std::uint32_t> labels(std::max<std::size_t>(n, 1)), hl;
    std::vector<double> sse(limit), hc;
    if (options.record_history) {
        hl.resize(static_cast<std::size_t>(limit) * n);
        hc.resize(static_cast<std::size_t>(limit) * 3 * k);
    }
    cqg_lloyd_stats st{};
    check(cqg_lloyd(ctx(), packed.data(), counts.data(), n, P, in.empty() ? nullptr : in.data(), static_cast<int>(k),
                    &term, cen.data(), labels.data(), sse.data(), &st, hl.empty() ? nullptr : hl.data(),
                    hc.empty() ? nullptr : hc.data()));
    return make_state(cen, k, labels, n, sse, st, hl, hc);
}

} // namespace detail
} // namespace quant
