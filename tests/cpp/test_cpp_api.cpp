// The reference's own datastore / pipeline unit-test cases (test_datastore.cpp, test_pipeline.cpp),
// restated against the C++ mirror include/double_b200.hpp.  Built by __graft_entry__.build() into
// build/test_cpp_api; run by tests/test_gpu_cpp_api.py on a B200.  Exit code = failures.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
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

// order-1 table over vocab 5: t -> t+1 (4 wraps to 1), BOS row -> 1 (test_speculation.cpp:11-27)
static Model repeat_model() {
    const int V = 5;
    std::vector<int32_t> w;
    std::vector<double> p;
    const int next[5] = {1, 2, 3, 4, 1};
    for (int a = 0; a < V; ++a) {
        w.push_back(a);
        for (int t = 0; t < V; ++t) p.push_back(t == next[a] ? 1.0 : 0.0);
    }
    return Model::table(1, V, w, p, std::vector<double>(V, 0.2));
}

// a draft/target table pair that mostly agree (the reference's make_lab at rho = 0.9 plays this role):
// next ~ (3b + 1) mod V with the given mass, the rest spread by a seeded generator
static Model peaked_model(int order, int V, double mass, unsigned seed) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> U(0.01, 1.0);
    std::vector<int32_t> w;
    std::vector<double> p;
    const int rows = order == 1 ? V : V * V;
    for (int r = 0; r < rows; ++r) {
        const int b = r % V;
        if (order == 2) w.push_back(r / V);
        w.push_back(b);
        std::vector<double> row(V);
        double s = 0;
        for (auto& x : row) s += (x = U(g));
        for (auto& x : row) x = x / s * (1.0 - mass);
        row[(3 * b + 1) % V] += mass;
        p.insert(p.end(), row.begin(), row.end());
    }
    return Model::table(order, V, w, p, std::vector<double>(V, 1.0 / V));
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
    {  // the device n-gram index (dbl_store_build_index): lookups identical to the scan, before and after
       // more inserts (the appended tail is scanned), over a randomized store
        std::mt19937_64 g(17);
        HierarchicalDatastore scan(3, 10), idx(3, 10);
        std::vector<TokenSeq> seqs;
        for (int i = 0; i < 60; ++i) {
            TokenSeq q;
            for (int k = 0; k < 8 + static_cast<int>(g() % 40); ++k) q.push_back(static_cast<TokenId>(g() % 24));
            seqs.push_back(q);
        }
        for (int i = 0; i < 40; ++i) {
            scan.prior.insert(seqs[i], i);
            idx.prior.insert(seqs[i], i);
        }
        idx.build_index(DBL_LAYER_PRIOR);
        CHECK(idx.index_entries(DBL_LAYER_PRIOR) > 0 && scan.index_entries(DBL_LAYER_PRIOR) == 0);
        for (int i = 40; i < 60; ++i) {  // an appended tail, and dynamic / rejected layers
            const int layer = i % 3;
            (layer == 0 ? scan.prior : layer == 1 ? scan.dynamic : scan.rejected).insert(seqs[i], i);
            (layer == 0 ? idx.prior : layer == 1 ? idx.dynamic : idx.rejected).insert(seqs[i], i);
        }
        int same = 0;
        for (int k = 0; k < 200; ++k) {
            TokenSeq ctx;
            for (int j = 0; j < 1 + static_cast<int>(g() % 6); ++j) ctx.push_back(static_cast<TokenId>(g() % 24));
            const int d = 1 + static_cast<int>(g() % 10);
            const LookupResult a = scan.lookup(ctx, d), b = idx.lookup(ctx, d);
            same += a.candidates == b.candidates && a.source == b.source && a.matched_order == b.matched_order;
        }
        CHECK(same == 200);
        CHECK(idx.profile_lookup(TokenSeq{1, 2, 3}, 10, 20) > 0.0);
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
    {  // model.hpp helpers: test_model.cpp:140-172
        const ProbVector p = {0.1, 0.2, 0.3, 0.4};
        CHECK(tempered(p, 1.0) == p);
        const ProbVector sharp = tempered(p, 0.25);
        double denom = 0.0;
        for (double v : p) denom += std::pow(v, 4.0);
        CHECK(std::fabs(sharp[2] - std::pow(0.3, 4.0) / denom) < 1e-12);
        CHECK(sharp[3] > p[3] && sharp[0] < p[0]);
        CHECK(argmax_token({0.2, 0.4, 0.4}) == 1);
        CHECK(argmax_token({0.5, 0.5}) == 0);
        ProbVector big(151936, 1e-6);
        big[77777] = big[99999] = 0.5;  // a tie across CTA warps: the lowest id
        CHECK(argmax_token(big) == 77777);
        CHECK(throws<std::runtime_error>([&] { argmax_token({0.0, 0.0}); }));
        Rng a(7), b(7);
        CHECK(sample({0.1, 0.7, 0.2}, SamplerConfig{0.0, 0}, a) == 1);
        CHECK(a.uniform() == b.uniform());  // T = 0 consumes no randomness
        Rng c(7), d(7);
        d.uniform();
        sample({0.1, 0.7, 0.2}, SamplerConfig{1.0, 0}, c);
        CHECK(c.uniform() == d.uniform());  // T > 0 consumes exactly one uniform
    }
    {  // accept_with_model greedy: test_speculation.cpp:39-78
        const SamplerConfig cfg{0.0, 0};
        Rng rng(1);
        const std::vector<ProbVector> dists = {{0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}, {1.0, 0.0, 0.0}};
        RetrievalResult r = accept_with_model(dists, TokenSeq{1, 2}, cfg, rng);
        CHECK(r.matched_len == 2 && (r.emitted == TokenSeq{1, 2, 0}) && r.probs.size() == 3);
        r = accept_with_model(dists, TokenSeq{1, 0}, cfg, rng);
        CHECK(r.matched_len == 1 && (r.emitted == TokenSeq{1, 2}) && r.probs.size() == 2 && r.probs[1] == dists[1]);
        r = accept_with_model(std::vector<ProbVector>{dists[0]}, TokenSeq{}, cfg, rng);
        CHECK(r.matched_len == 0 && (r.emitted == TokenSeq{1}));
        CHECK(throws<std::invalid_argument>([&] { accept_with_model(dists, TokenSeq{1, 2, 0}, cfg, rng); }));
        r = accept_with_model(dists, TokenSeq{7, 2}, cfg, rng);
        CHECK(r.matched_len == 0 && (r.emitted == TokenSeq{1}));
    }
    {  // accept_with_model stochastic: emitted law and acceptance rate (test_speculation.cpp:80-110)
        const SamplerConfig cfg{1.0, 0};
        const ProbVector dist = {0.5, 0.3, 0.2};
        const std::vector<ProbVector> dists = {dist, {0.2, 0.2, 0.6}};
        for (TokenId cand : {0, 1, 2}) {
            ProbVector emp(3, 0.0);
            const int trials = 3000;
            Rng rng(42 + static_cast<std::uint64_t>(cand));
            for (int t = 0; t < trials; ++t)
                emp[static_cast<size_t>(accept_with_model(dists, TokenSeq{cand}, cfg, rng).emitted[0])] += 1.0 / trials;
            double tv = 0.0;
            for (int i = 0; i < 3; ++i) tv += std::fabs(emp[i] - dist[i]) / 2.0;
            CHECK(tv < 0.04);
        }
        Rng rng(11);
        const int trials = 3000;
        int matched = 0;
        for (int t = 0; t < trials; ++t)
            matched += accept_with_model(std::vector<ProbVector>{{0.7, 0.3}, {0.5, 0.5}}, TokenSeq{0}, cfg, rng).matched_len;
        CHECK(std::fabs(static_cast<double>(matched) / trials - 0.7) < 0.04);
    }
    {  // retrieval_forward / iterative_draft / measure_amt: test_speculation.cpp:112-200
        const Model m = repeat_model();
        const SamplerConfig cfg{0.0, 0};
        {
            HierarchicalDatastore store(3, 10);
            store.prior.insert(TokenSeq{1, 2, 3, 4}, 0);
            Rng rng(1);
            SimClock clock;
            const RetrievalResult r = retrieval_forward(m, store, TokenSeq{1, 2}, 10, cfg, rng, &clock);
            CHECK(r.source == LookupSource::Prior && r.matched_len == 2 && (r.emitted == TokenSeq{3, 4, 1}));
            CHECK(clock.now == m.forward_cost);  // one batched forward
        }
        {
            HierarchicalDatastore store(3, 10);
            Rng rng(1);
            const RetrievalResult r = retrieval_forward(m, store, TokenSeq{3}, 10, cfg, rng);
            CHECK(r.source == LookupSource::Miss && r.matched_len == 0 && (r.emitted == TokenSeq{4}) && r.probs.size() == 1);
        }
        {
            HierarchicalDatastore store(3, 10);
            store.prior.insert(TokenSeq{1, 2, 3, 4}, 0);
            Rng rng(1);
            const RetrievalResult r = retrieval_forward(m, store, TokenSeq{1, 2}, 10, cfg, rng, nullptr, false);
            CHECK(r.matched_len == 0 && (r.emitted == TokenSeq{3}) && store.stats().lookups == 0);
        }
        {
            HierarchicalDatastore store(3, 10);
            store.prior.insert(TokenSeq{1, 2, 3, 4, 1, 2, 3, 4}, 0);
            SimClock clock;
            Rng rng(5);
            const DraftChain chain = iterative_draft(m, store, TokenSeq{1}, 3, 4, cfg, rng, &clock);
            CHECK(chain.segments.size() == 3 && chain.total_len == static_cast<int>(chain.tokens.size()));
            CHECK(chain.probs.size() == chain.tokens.size() && clock.now == 3.0 * m.forward_cost);
            Rng rng2(5);
            TokenSeq grown{1}, flat;
            for (int j = 0; j < 3 && chain.segments.size() == 3; ++j) {
                const RetrievalResult seg = retrieval_forward(m, store, grown, 4, cfg, rng2);
                grown.insert(grown.end(), seg.emitted.begin(), seg.emitted.end());
                flat.insert(flat.end(), seg.emitted.begin(), seg.emitted.end());
                CHECK(seg.emitted == chain.segments[static_cast<size_t>(j)].emitted);
            }
            CHECK(chain.tokens == flat);
            Rng rng3(1);
            CHECK(throws<std::invalid_argument>([&] { iterative_draft(m, store, TokenSeq{1}, 0, 4, cfg, rng3); }));
        }
        std::vector<RetrievalResult> traces(3);
        traces[0].matched_len = 2;
        traces[1].matched_len = 0;
        traces[2].matched_len = 7;
        CHECK(measure_amt(traces) == 3.0);
        CHECK(throws<std::invalid_argument>([&] { measure_amt(std::vector<RetrievalResult>{}); }));
    }
    {  // the decoder state machine: test_pipeline.cpp:117-226
        const int V = 16;
        const Model draft = peaked_model(1, V, 0.8, 11), target = peaked_model(2, V, 0.9, 12);
        const std::vector<TokenSeq> corpus{{1, 4, 13, 8, 9, 12, 5, 0}, {2, 7, 6, 3, 10, 15, 14, 11}};
        PipelineOptions opts;
        opts.gamma = 4;
        const TokenSeq prompt{1, 4, 13, 8, 9, 12, 5, 0};
        {  // cold start enters pre-verify with prev_tokens = gamma (:117-136)
            HierarchicalDatastore store(3, 10);
            store.prior = build_prior(corpus, 3, 10);
            PipelineState state;
            state.committed = prompt;
            state.prev_tokens = 4;
            state.last_committed_len = static_cast<long>(prompt.size());
            CHECK(state.mode == Mode::PreVerify);
            const RoundTrace tr = run_round(state, draft, target, store, opts);
            CHECK(tr.round == 0 && tr.mode == "pre_verify" && tr.pending == 0 && tr.committed_count >= 1);
            if (state.mode == Mode::PostVerify) CHECK(state.prev_tokens == static_cast<int>(state.speculative.size()));
            else CHECK(state.speculative.empty() && state.prev_tokens == 4);
        }
        {  // run_round rejects inconsistent state (:138-149)
            HierarchicalDatastore store(3, 10);
            PipelineState state;
            state.committed = prompt;
            state.mode = Mode::PostVerify;
            state.speculative = {1, 2};
            state.spec_probs.resize(2, ProbVector(V, 1.0 / V));
            state.prev_tokens = 3;  // wrong on purpose
            CHECK(throws<std::logic_error>([&] { run_round(state, draft, target, store, opts); }));
            state.prev_tokens = 2;
            state.spec_probs.resize(1);
            CHECK(throws<std::logic_error>([&] { run_round(state, draft, target, store, opts); }));
        }
        {  // rollback truncates, clears speculation, and is idempotent (:151-168)
            PipelineState state;
            state.committed = {1, 2, 3, 4, 5};
            state.speculative = {6, 7};
            state.spec_probs.resize(2);
            state.mode = Mode::PostVerify;
            state.last_committed_len = 3;
            rollback(state, 4);
            CHECK((state.committed == TokenSeq{1, 2, 3, 4}) && state.speculative.empty() && state.mode == Mode::PreVerify);
            rollback(state, 4);
            CHECK((state.committed == TokenSeq{1, 2, 3, 4}));
            CHECK(throws<std::invalid_argument>([&] { rollback(state, 99); }));
            CHECK(throws<std::logic_error>([&] { rollback(state, 2); }));
        }
        {  // rollback to the committed boundary equals never having speculated (:170-197)
            HierarchicalDatastore base(3, 10);
            base.prior = build_prior(corpus, 3, 10);
            PipelineState a;
            a.committed = prompt;
            a.prev_tokens = opts.gamma;
            a.last_committed_len = static_cast<long>(prompt.size());
            HierarchicalDatastore store_a = base;
            run_round(a, draft, target, store_a, opts);
            const TokenSeq committed_after = a.committed;
            rollback(a, static_cast<long>(a.committed.size()));
            a.prev_tokens = opts.gamma;
            PipelineState b;
            b.committed = committed_after;
            b.prev_tokens = opts.gamma;
            b.round = a.round;
            b.last_committed_len = static_cast<long>(committed_after.size());
            HierarchicalDatastore store_b = store_a;
            HierarchicalDatastore store_a2 = store_a;
            run_round(a, draft, target, store_a2, opts);
            run_round(b, draft, target, store_b, opts);
            CHECK(a.committed == b.committed);
            CHECK(a.speculative == b.speculative);
            CHECK(store_a2.dynamic.occurrence_count() == store_b.dynamic.occurrence_count());
        }
        {  // run_round driven to the budget == run() (traces, JSONL and output), greedy and sampled
            for (double T : {0.0, 1.0}) {
                PipelineOptions o = opts;
                o.sampler = SamplerConfig{T, 3};
                HierarchicalDatastore s1(3, 10), s2(3, 10);
                s1.prior = build_prior(corpus, 3, 10);
                s2.prior = build_prior(corpus, 3, 10);
                const RunResult r = run(draft, target, s1, prompt, 40, o);
                PipelineState st;
                st.committed = prompt;
                st.prev_tokens = o.gamma;
                st.last_committed_len = static_cast<long>(prompt.size());
                s2.record_accepted(prompt);
                std::vector<RoundTrace> traces;
                while (st.committed.size() - prompt.size() < 40) {
                    traces.push_back(run_round(st, draft, target, s2, o));
                    bool eos = false;
                    for (size_t i = prompt.size(); i < st.committed.size(); ++i) eos = eos || st.committed[i] == V - 1;
                    if (eos) break;
                }
                CHECK(traces_to_jsonl(traces) == r.jsonl);
                CHECK(traces_to_jsonl(r.traces) == r.jsonl);
                CHECK(r.traces.size() == traces.size());
                const RunMetrics m = compute_metrics(traces, o.latency);
                CHECK(m.tokens == r.metrics.tokens && m.m == r.metrics.m && m.clock == r.metrics.clock);
                CHECK(std::fabs(st.clock.now - r.metrics.clock) < 1e-9);
            }
        }
        {  // compute_metrics segment accounting (:199-226) and write_traces
            std::vector<RoundTrace> traces(2);
            traces[0].committed_count = 7;
            traces[0].clock_delta = 1.0;
            traces[1].pending_reject = traces[1].rejected = true;
            traces[1].accepted_pending = 0;
            traces[1].committed_count = 1;
            traces[1].clock_delta = 1.0;
            const RunMetrics m = compute_metrics(traces, LatencyConfig{});
            CHECK(m.m == 4.0 && m.tokens == 8);
            std::vector<RoundTrace> ten(10);
            for (auto& t : ten) {
                t.committed_count = 5;
                t.clock_delta = 1.0;
            }
            CHECK(compute_metrics(ten, LatencyConfig{}).m == 50.0);
            CHECK(throws<std::invalid_argument>([&] { compute_metrics({}, LatencyConfig{}); }));
            write_traces(traces, "build/test_cpp_api_traces.jsonl");
            std::ifstream f("build/test_cpp_api_traces.jsonl");
            std::stringstream ss;
            ss << f.rdbuf();
            CHECK(ss.str() == traces_to_jsonl(traces));
            CHECK(throws<std::runtime_error>([&] { write_traces(traces, "/nonexistent-dir/x.jsonl"); }));
        }
    }
    std::printf("test_cpp_api: %d failure(s)\n", g_fail);
    return g_fail;
}
