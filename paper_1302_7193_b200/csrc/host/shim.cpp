// Glue of the host C++ shim (namespace anisocg) to the C ABI: status ->
// exception mapping (the reference's error contract, operator.hpp:21-24,
// field.hpp:95-98), device-context construction, and scratch-field pools.
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "acg.h"
#include "anisocg/field.hpp"
#include "anisocg/operator.hpp"

namespace anisocg {
namespace detail {

void check(acg_status st) {
    if (st == ACG_OK) return;
    const std::string msg = acg_last_error();
    switch (st) {
        case ACG_ERR_INVALID_ARGUMENT:
            throw std::invalid_argument(msg);
        case ACG_ERR_BREAKDOWN:
            throw NumericalBreakdown(msg);
        default:
            throw std::runtime_error("acg: " + msg);
    }
}

namespace {
std::mutex g_mu;
std::map<const acg_context*, std::vector<acg_field*>> g_pool;

void drop_pool(const acg_context* c) {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_pool.find(c);
    if (it == g_pool.end()) return;
    for (acg_field* f : it->second) acg_field_destroy(f);
    g_pool.erase(it);
}
}  // namespace

Scratch::Scratch(const acg_context* c) : ctx(const_cast<acg_context*>(c)), f(nullptr) {
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto& v = g_pool[c];
        if (!v.empty()) {
            f = v.back();
            v.pop_back();
        }
    }
    if (!f) check(acg_field_create(&f, c));
}

Scratch::~Scratch() {
    std::lock_guard<std::mutex> lk(g_mu);
    g_pool[ctx].push_back(f);
}

std::shared_ptr<acg_context> make_device_context(acg_dtype dtype, const VerticalProfile& p,
                                                 const PanelGeometry& g,
                                                 const acg_placement* placement) {
    if (static_cast<int>(p.a_prime.size()) != p.n_z || static_cast<int>(p.d.size()) != p.n_z ||
        static_cast<int>(g.cell_area.size()) != g.m * g.m)
        throw std::invalid_argument("OperatorContext: inconsistent profile or geometry");
    acg_operator_desc d{};
    d.m = g.m;
    d.n_z = p.n_z;
    d.a_prime = p.a_prime.data();
    d.b_prime = p.b_prime.data();
    d.c_prime = p.c_prime.data();
    d.d = p.d.data();
    d.cell_area = g.cell_area.data();
    d.alpha_east = g.alpha_east.data();
    d.alpha_north = g.alpha_north.data();
    d.alpha_diag = g.alpha_diag.data();
    acg_context* c = nullptr;
    check(acg_context_create(&c, dtype, &d, placement));
    return std::shared_ptr<acg_context>(c, [](acg_context* x) {
        drop_pool(x);
        acg_context_destroy(x);
    });
}

namespace {
std::mutex g_shape_mu;
std::map<std::tuple<int, int, int>, acg_context*>& shape_cache() {
    static auto* cache = new std::map<std::tuple<int, int, int>, acg_context*>();
    return *cache;
}
}  // namespace

void release_scratch(const acg_context* c) {
    drop_pool(c);
    check(acg_context_release_scratch(c));
}

// Shape-only contexts for the context-free level-1 API (axpy/scal/dot/nrm2/
// fill_random take fields, not an operator). The contexts themselves (profile
// and column tables) live for the process; their field-sized scratch is freed
// by release_device_scratch().
acg_context* shape_context(acg_dtype dtype, int m, int n_z) {
    std::lock_guard<std::mutex> lk(g_shape_mu);
    auto* cache = &shape_cache();
    const auto key = std::make_tuple(static_cast<int>(dtype), m, n_z);
    auto it = cache->find(key);
    if (it != cache->end()) return it->second;
    std::vector<double> zn(n_z, 0.0), one(n_z, 1.0), cols(static_cast<size_t>(m) * m, 1.0);
    std::vector<double> edges(static_cast<size_t>(m > 1 ? m - 1 : 1) * m, 0.0);
    std::vector<double> zc(static_cast<size_t>(m) * m, 0.0);
    acg_operator_desc d{};
    d.m = m;
    d.n_z = n_z;
    d.a_prime = zn.data();
    d.b_prime = zn.data();
    d.c_prime = zn.data();
    d.d = one.data();
    d.cell_area = cols.data();
    d.alpha_east = edges.data();
    d.alpha_north = edges.data();
    d.alpha_diag = zc.data();
    acg_context* c = nullptr;
    check(acg_context_create(&c, dtype, &d, nullptr));
    (*cache)[key] = c;
    return c;
}

}  // namespace detail

void release_device_scratch() {
    std::vector<const acg_context*> pooled;
    {
        std::lock_guard<std::mutex> lk(detail::g_mu);
        for (auto& kv : detail::g_pool) pooled.push_back(kv.first);
    }
    for (const acg_context* c : pooled) detail::drop_pool(c);
    std::vector<acg_context*> ctxs;
    {
        std::lock_guard<std::mutex> lk(detail::g_shape_mu);
        for (auto& kv : detail::shape_cache()) ctxs.push_back(kv.second);
    }
    for (acg_context* c : ctxs) detail::release_scratch(c);
}

}  // namespace anisocg
