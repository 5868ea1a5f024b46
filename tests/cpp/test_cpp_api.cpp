// The reference's own datastore / pipeline unit-test cases (test_datastore.cpp, test_pipeline.cpp),
// restated against the C++ mirror include/double_b200.hpp.  Built by __graft_entry__.build() into
// build/test_cpp_api; run by tests/test_gpu_cpp_api.py on a B200.  Exit code = failures.
#include <cstdio>
#include <random>
#include <vector>

#include "double_b200.hpp"

using namespace specpar_b200;

static int g_fail = 0;
#define CHECK(x)                                                          \
    do {                                                                  \
        if (!(x)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);      \
            ++g_fail;                                                     \
        }                                                                 \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

int main() {
    {  // test_datastore.cpp:62-70
        HierarchicalDatastore store(3, 10);
        store.prior.insert(TokenSeq{1, 2, 3, 4, 5, 6}, 0);
        const LookupResult r = store.lookup(TokenSeq{9, 2, 3}, 10);
        CHECK(r.source == LookupSource::Prior);
        CHECK(r.matched_order == 2);
        CHECK((r.candidates == TokenSeq{4, 5, 6}));
    }
    {  // :80-89 higher order beats layer priority
        HierarchicalDatastore store(3, 10);
        store.prior.insert(TokenSeq{2, 3, 9}, 0);
        store.dynamic.insert(TokenSeq{1, 2, 3, 7}, 1);
        const LookupResult r = store.lookup(TokenSeq{1, 2, 3}, 10);
        CHECK(r.source == LookupSource::Dynamic && r.matched_order == 3 && (r.candidates == TokenSeq{7}));
    }
    {  // :111-118 recency
        HierarchicalDatastore store(2, 10);
        store.dynamic.insert(TokenSeq{1, 2, 5}, 0);
        store.dynamic.insert(TokenSeq{1, 2, 6}, 3);
        store.dynamic.insert(TokenSeq{1, 2, 4}, 1);
        CHECK((store.lookup(TokenSeq{1, 2}, 10).candidates == TokenSeq{6}));
    }
    {  // :120-145 PLD fallback and miss; :147-159 stats
        HierarchicalDatastore store(3, 10);
        const LookupResult r = store.lookup(TokenSeq{1, 2, 9, 1, 2, 8, 1, 2}, 10);
        CHECK(r.source == LookupSource::ContextFallback && (r.candidates == TokenSeq{8, 1, 2}));
        CHECK(store.lookup(TokenSeq{1, 2, 3}, 10).source == LookupSource::Miss);
        CHECK(throws<std::invalid_argument>([&] { store.lookup(TokenSeq{}, 10); }));
        CHECK(store.stats().lookups == 2 && store.stats().fallback_hits == 1 && store.stats().misses == 1);
    }
    {  // :33-44 insert/occurrence_count, empty insert throws invalid_argument
        HierarchicalDatastore store(3, 10);
        store.prior.insert(TokenSeq{1, 2, 3, 4}, 0);
        store.prior.insert(TokenSeq{5, 6}, 1);
        CHECK(store.prior.occurrence_count() == 4 + 3 + 2 + 2 + 1);
        CHECK(throws<std::invalid_argument>([&] { store.prior.insert(TokenSeq{}, 2); }));
    }
    {  // test_pipeline.cpp:57-72 lossless (table models): DOUBLE == target-only greedy AR
        const int V = 16, order = 2;
        std::mt19937_64 g(5);
        std::uniform_real_distribution<double> U(0.01, 1.0);
        std::vector<int32_t> windows;
        std::vector<double> probs;
        for (int a = 0; a < V; ++a)
            for (int b = 0; b < V; ++b) {
                windows.push_back(a);
                windows.push_back(b);
                double s = 0;
                std::vector<double> row(V);
                for (auto& x : row) s += (x = U(g));
                for (auto& x : row) probs.push_back(x / s);
            }
        std::vector<double> fb(V, 1.0 / V);
        Model target = Model::table(order, V, windows, probs, fb);
        std::vector<int32_t> w1;
        std::vector<double> p1;
        for (int a = 0; a < V; ++a) {
            w1.push_back(a);
            double s = 0;
            std::vector<double> row(V);
            for (auto& x : row) s += (x = U(g));
            for (auto& x : row) p1.push_back(x / s);
        }
        Model draft = Model::table(1, V, w1, p1, fb);
        HierarchicalDatastore store(3, 10);
        build_prior(store, {{1, 2, 3, 4, 5, 1, 2, 3}, {4, 5, 6, 7, 1, 2}}, 10);
        const TokenSeq prompt{1, 2, 3, 4};
        const RunResult r = run(draft, target, store, prompt, 64, PipelineOptions{});
        const RunResult ar = run_vanilla_ar(target, prompt, 64);
        CHECK(r.output == ar.output);
        // batched DOUBLE / AR: every sequence equals its own single run
        HierarchicalDatastore s1(3, 10), s2(3, 10), s3(3, 10);
        for (HierarchicalDatastore* st : {&s1, &s2, &s3}) build_prior(*st, {{1, 2, 3, 4, 5, 1, 2, 3}, {4, 5, 6, 7, 1, 2}}, 10);
        const std::vector<TokenSeq> ps{prompt, TokenSeq{7, 7, 1}, TokenSeq{3}};
        const std::vector<RunResult> rb = run_batch(draft, target, {&s1, &s2, &s3}, ps, 48, PipelineOptions{});
        const std::vector<TokenSeq> ab = run_vanilla_ar_batch(target, ps, 48);
        for (size_t b = 0; b < ps.size(); ++b) {
            HierarchicalDatastore sb(3, 10);
            build_prior(sb, {{1, 2, 3, 4, 5, 1, 2, 3}, {4, 5, 6, 7, 1, 2}}, 10);
            CHECK(rb[b].output == run(draft, target, sb, ps[b], 48, PipelineOptions{}).output);
            CHECK(ab[b] == run_vanilla_ar(target, ps[b], 48).output);
        }
        // sampled run (SamplerConfig) is reproducible; forward_batch rows are distributions
        PipelineOptions so;
        so.sampler = SamplerConfig{1.0, 42};
        HierarchicalDatastore t1(3, 10), t2(3, 10);
        CHECK(run(draft, target, t1, prompt, 32, so).output == run(draft, target, t2, prompt, 32, so).output);
        const auto rows = forward_batch(target, prompt, TokenSeq{2, 3});
        CHECK(rows.size() == 3 && rows[0].size() == static_cast<size_t>(V));
        CHECK(throws<std::invalid_argument>([&] { run(draft, target, store, TokenSeq{}, 8, PipelineOptions{}); }));
        PipelineOptions bad;
        bad.gamma = 0;
        CHECK(throws<std::invalid_argument>([&] { run(draft, target, store, prompt, 8, bad); }));
    }
    {  // verifier: test_verification.cpp:187-245 through the C++ mirror
        const SamplerConfig greedy{0.0, 0}, stoch{1.0, 0};
        Rng rng(1);
        const TokenSeq draft{3, 4};
        GuidanceChain longer;
        longer.tokens = {3, 4, 7, 8};
        VerifyOutcome o = guided_output(draft, {}, longer, std::nullopt, greedy, rng);
        CHECK(o.kind == VerifyKind::Extension && (o.committed == TokenSeq{3, 4, 7, 8}));
        GuidanceChain g;
        g.tokens = {3};
        g.probs = {{0.9, 0.1}, {0.1, 0.9}};
        o = guided_output(draft, {}, g, 1, greedy, rng);
        CHECK(o.kind == VerifyKind::Correction && (o.committed == TokenSeq{3, 1}));
        CHECK(throws<std::invalid_argument>([&] { guided_output(draft, {}, GuidanceChain{}, 1, greedy, rng); }));
        Rng rng8(8);
        const std::vector<ProbVector> qp = {{0.9, 0.1}, {0.2, 0.5, 0.3}};
        GuidanceChain s;
        s.tokens = {0, 2, 4};
        s.probs = {{0.9, 0.1}, {0.6, 0.1, 0.3}};
        o = guided_output(TokenSeq{0, 1}, qp, s, 1, stoch, rng8);
        CHECK(o.kind == VerifyKind::ResidualCorrection && o.accepted_len == 1 && (o.committed == TokenSeq{0, 0}));
        CHECK(accept_prob({0.5, 0.5}, {0.25, 0.75}, 0) == 1.0);
        CHECK(throws<std::invalid_argument>([&] { accept_prob({0.5, 0.5}, {0.0, 1.0}, 0); }));
        CHECK(throws<std::runtime_error>([&] { residual_sample({0.5, 0.5}, {0.5, 0.5}, rng); }));
    }
    std::printf("test_cpp_api: %d failure(s)\n", g_fail);
    return g_fail;
}
