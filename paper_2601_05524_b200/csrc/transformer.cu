// Random-init bf16 decoder-only transformer (Qwen3 / Llama shapes) behind the forward_batch contract.
//
// One forward processes the lane positions [start, L+c) padded to tp (multiple of 16) token columns:
//   embed -> L x [RMSNorm -> QKV GEMM -> qk-norm/RoPE/KV append -> split-KV attention -> O GEMM (+resid)
//                 -> RMSNorm -> gate|up GEMM (SiLU*up epilogue) -> down GEMM (+resid)]
//         -> RMSNorm -> LM head GEMM (fused per-tile argmax) -> argmax combine
// All GEMMs are the tcgen05 swap-AB stream-K kernel (gemm.cu); the weights are streamed from HBM
// exactly once per forward, which is the roofline of the verify step.
// Tensor parallel (tp_size > 1): column-parallel QKV / gate|up, row-parallel O / down with a
// deterministic all-gather + rank-ordered sum, vocab-parallel LM head with a (max, lowest global id)
// combine — see tp.cu.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "gemm.cuh"
#include "tf_kernels.cuh"
#include "tp.cuh"
#include "transformer.cuh"

namespace dbl {

namespace {
constexpr int kMaxTp = 256;  // token columns per forward (UMMA N limit)
enum TensorId : uint64_t { kEmbed = 1, kLmHead = 2 };
inline uint64_t layer_id(int l, int which) { return 1000 + static_cast<uint64_t>(l) * 16 + which; }
enum { kQ = 0, kK = 1, kV = 2, kO = 3, kGate = 4, kUp = 5, kDown = 6 };
}  // namespace

struct LayerW {
    DevBuf<__nv_bfloat16> attn_norm, mlp_norm, q_norm, k_norm, qkv, o, gateup, down;
    CUtensorMap t_qkv, t_o, t_gu, t_down;
};

struct Transformer::Impl {
    dbl_transformer_config c;
    int rank = 0, world = 1;
    int nh, nkv, hd, h, q_dim, kv_dim, qkv_rows, ffn_l, vocab_l;
    std::vector<LayerW> layers;
    DevBuf<__nv_bfloat16> embed, final_norm, lm_head_own;
    const __nv_bfloat16* lm_head = nullptr;
    CUtensorMap t_lm;
    std::unique_ptr<TpComm> comm;
    GemmProfiler* prof = nullptr;
};

void Transformer::set_profiler(GemmProfiler* p) { impl_->prof = p; }

struct TfCache final : LaneCache {
    int capacity, pages, max_chunks;
    DevBuf<__nv_bfloat16> kbuf, vbuf;  // [layers][pages][nkv][kPage][hd]
    DevBuf<int32_t> page_table;
    DevBuf<float> resid, part_o, part_ml, tp_partial;
    DevBuf<__nv_bfloat16> xn, qkv, qbuf, attn, act;
    CUtensorMap t_xn, t_attn, t_act;
    GemmWorkspace ws;
    size_t layer_stride = 0;
    // one CUDA graph per token-column bucket: the whole forward (~370 kernels with programmatic
    // dependent-launch edges) replays with a single launch; every argument is fixed per cache
    std::map<int, cudaGraphExec_t> graphs;
    std::map<int, long long> graph_nodes;
    ~TfCache() override {
        for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    }
};

namespace {
bool graphs_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("DBL_GRAPHS");
        return !(e && e[0] == '0');
    }();
    return on;
}
}  // namespace

Transformer::Transformer(const dbl_transformer_config& cfg, int device, void* nccl_comm)
    : cfg_(cfg), device_(device) {
    const auto& c = cfg;
    if (c.n_layers < 1 || c.hidden < 64 || c.ffn < 64 || c.n_heads < 1 || c.n_kv_heads < 1 || c.vocab < 2)
        throw_invalid("transformer: bad shape");
    if (c.head_dim != 64 && c.head_dim != 128) throw_invalid("transformer: head_dim must be 64 or 128");
    if (c.n_heads % c.n_kv_heads) throw_invalid("transformer: n_heads must be a multiple of n_kv_heads");
    if (c.hidden % 128) throw_invalid("transformer: hidden must be a multiple of 128");
    const int world = c.tp_size < 1 ? 1 : c.tp_size;
    if (c.n_kv_heads % world || c.n_heads % world || c.ffn % (64 * world) || c.vocab % world)
        throw_invalid("transformer: shapes do not shard evenly over tp_size");
    if (c.max_seq < 16) throw_invalid("transformer: max_seq too small");
    require_device(device);
    DeviceGuard g(device);
    impl_ = new Impl;
    Impl& m = *impl_;
    m.c = c;
    m.world = world;
    m.rank = c.tp_rank;
    if (m.rank < 0 || m.rank >= world) throw_invalid("transformer: tp_rank out of range");
    m.nh = c.n_heads / world;
    m.nkv = c.n_kv_heads / world;
    m.hd = c.head_dim;
    m.h = c.hidden;
    m.q_dim = m.nh * m.hd;
    m.kv_dim = m.nkv * m.hd;
    m.qkv_rows = m.q_dim + 2 * m.kv_dim;
    m.ffn_l = c.ffn / world;
    m.vocab_l = c.vocab / world;
    if (m.q_dim % 64) throw_invalid("transformer: per-rank q dim must be a multiple of 64");
    if (world > 1) {
        if (!nccl_comm) throw_invalid("transformer: tp_size > 1 needs an NCCL communicator");
        m.comm = std::make_unique<TpComm>(nccl_comm, m.rank, world, device);
    }
    cudaStream_t s = 0;
    const uint64_t seed = c.seed;
    const float sd = c.init_std;
    const int h = m.h;
    m.layers.resize(c.n_layers);
    for (int l = 0; l < c.n_layers; ++l) {
        LayerW& w = m.layers[l];
        w.attn_norm.alloc(h);
        w.mlp_norm.alloc(h);
        launch_fill(w.attn_norm.p, h, 1.0f, s);
        launch_fill(w.mlp_norm.p, h, 1.0f, s);
        if (c.qk_norm) {
            w.q_norm.alloc(m.hd);
            w.k_norm.alloc(m.hd);
            launch_fill(w.q_norm.p, m.hd, 1.0f, s);
            launch_fill(w.k_norm.p, m.hd, 1.0f, s);
        }
        w.qkv.alloc(static_cast<size_t>(m.qkv_rows) * h);
        launch_init_normal(w.qkv.p, m.q_dim, h, h, seed, layer_id(l, kQ), static_cast<int64_t>(m.rank) * m.q_dim, 0, h, sd, s);
        launch_init_normal(w.qkv.p + static_cast<size_t>(m.q_dim) * h, m.kv_dim, h, h, seed, layer_id(l, kK),
                           static_cast<int64_t>(m.rank) * m.kv_dim, 0, h, sd, s);
        launch_init_normal(w.qkv.p + static_cast<size_t>(m.q_dim + m.kv_dim) * h, m.kv_dim, h, h, seed,
                           layer_id(l, kV), static_cast<int64_t>(m.rank) * m.kv_dim, 0, h, sd, s);
        w.o.alloc(static_cast<size_t>(h) * m.q_dim);
        launch_init_normal(w.o.p, h, m.q_dim, m.q_dim, seed, layer_id(l, kO), 0,
                           static_cast<int64_t>(m.rank) * m.q_dim, static_cast<int64_t>(c.n_heads) * m.hd, sd, s);
        w.gateup.alloc(static_cast<size_t>(2) * m.ffn_l * h);
        launch_init_gateup(w.gateup.p, m.ffn_l, h, seed, layer_id(l, kGate), layer_id(l, kUp),
                           static_cast<int64_t>(m.rank) * m.ffn_l, sd, s);
        w.down.alloc(static_cast<size_t>(h) * m.ffn_l);
        launch_init_normal(w.down.p, h, m.ffn_l, m.ffn_l, seed, layer_id(l, kDown), 0,
                           static_cast<int64_t>(m.rank) * m.ffn_l, c.ffn, sd, s);
        w.t_qkv = make_tmap_bf16_2d(w.qkv.p, m.qkv_rows, h, 128);
        w.t_o = make_tmap_bf16_2d(w.o.p, h, m.q_dim, 128);
        w.t_gu = make_tmap_bf16_2d(w.gateup.p, 2 * m.ffn_l, h, 128);
        w.t_down = make_tmap_bf16_2d(w.down.p, h, m.ffn_l, 128);
    }
    m.final_norm.alloc(h);
    launch_fill(m.final_norm.p, h, 1.0f, s);
    m.embed.alloc(static_cast<size_t>(c.vocab) * h);
    launch_init_normal(m.embed.p, c.vocab, h, h, seed, kEmbed, 0, 0, h, sd, s);
    if (c.tied_embeddings) {
        m.lm_head = m.embed.p + static_cast<size_t>(m.rank) * m.vocab_l * h;
    } else {
        m.lm_head_own.alloc(static_cast<size_t>(m.vocab_l) * h);
        launch_init_normal(m.lm_head_own.p, m.vocab_l, h, h, seed, kLmHead, static_cast<int64_t>(m.rank) * m.vocab_l, 0,
                           h, sd, s);
        m.lm_head = m.lm_head_own.p;
    }
    m.t_lm = make_tmap_bf16_2d(m.lm_head, m.vocab_l, h, 128);
    CUDA_CHECK(cudaDeviceSynchronize());
}

Transformer::~Transformer() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    delete impl_;
}

int64_t Transformer::weight_bytes() const {
    const Impl& m = *impl_;
    const int64_t per_layer = (static_cast<int64_t>(m.qkv_rows) * m.h + static_cast<int64_t>(m.h) * m.q_dim +
                               2LL * m.ffn_l * m.h + static_cast<int64_t>(m.h) * m.ffn_l) * 2 +
                              2LL * m.h * 2 + (cfg_.qk_norm ? 4LL * m.hd : 0);
    return per_layer * cfg_.n_layers + static_cast<int64_t>(m.vocab_l) * m.h * 2 + m.h * 2;
}

int Transformer::max_forward_tokens() const { return kMaxTp; }

std::unique_ptr<LaneCache> Transformer::make_cache(int capacity) {
    const Impl& m = *impl_;
    DeviceGuard g(device_);
    auto cp = std::make_unique<TfCache>();
    TfCache& c = *cp;
    c.capacity = capacity;
    c.pages = (capacity + kPage - 1) / kPage;
    c.max_chunks = (c.pages * kPage + kAttnChunk - 1) / kAttnChunk;
    c.layer_stride = static_cast<size_t>(c.pages) * m.nkv * kPage * m.hd;
    c.kbuf.alloc(c.layer_stride * cfg_.n_layers);
    c.vbuf.alloc(c.layer_stride * cfg_.n_layers);
    std::vector<int32_t> pt(c.pages);
    for (int i = 0; i < c.pages; ++i) pt[i] = i;  // one sequence per lane: identity page map
    c.page_table.alloc(c.pages);
    CUDA_CHECK(cudaMemcpy(c.page_table.p, pt.data(), c.pages * 4, cudaMemcpyHostToDevice));
    c.resid.alloc(static_cast<size_t>(kMaxTp) * m.h);
    c.xn.alloc(static_cast<size_t>(kMaxTp) * m.h);
    c.qkv.alloc(static_cast<size_t>(kMaxTp) * m.qkv_rows);
    c.qbuf.alloc(static_cast<size_t>(kMaxTp) * m.q_dim);
    c.attn.alloc(static_cast<size_t>(kMaxTp) * m.q_dim);
    c.act.alloc(static_cast<size_t>(kMaxTp) * m.ffn_l);
    c.xn.zero();
    c.attn.zero();
    c.act.zero();
    c.part_o.alloc(static_cast<size_t>(kMaxTp) * m.nh * c.max_chunks * m.hd);
    c.part_ml.alloc(static_cast<size_t>(kMaxTp) * m.nh * c.max_chunks * 2);
    if (m.world > 1) c.tp_partial.alloc(static_cast<size_t>(kMaxTp) * m.h);
    c.t_xn = make_tmap_bf16_2d(c.xn.p, kMaxTp, m.h, 16);
    c.t_attn = make_tmap_bf16_2d(c.attn.p, kMaxTp, m.q_dim, 16);
    c.t_act = make_tmap_bf16_2d(c.act.p, kMaxTp, m.ffn_l, 16);
    const int max_tiles = std::max({(m.qkv_rows + 127) / 128, (2 * m.ffn_l + 127) / 128, (m.vocab_l + 127) / 128,
                                    (m.h + 127) / 128});
    c.ws.ensure(num_sms(device_), kMaxTp, max_tiles);
    CUDA_CHECK(cudaDeviceSynchronize());
    return cp;
}

namespace {
void run_forward(Transformer::Impl& m, Lane& lane, int max_tokens, float* logits, int ld_logits, cudaStream_t s);
}

void Transformer::forward(Lane& lane, int max_tokens, cudaStream_t s) {
    if (!graphs_enabled() || impl_->prof || impl_->world > 1) {
        run_forward(*impl_, lane, max_tokens, nullptr, 0, s);
        return;
    }
    TfCache& c = *static_cast<TfCache*>(lane.cache.get());
    const int tp = (std::max(max_tokens, 1) + 15) / 16 * 16;
    auto it = c.graphs.find(tp);
    if (it == c.graphs.end()) {
        gemm_prepare();  // kernel attributes must be set outside capture
        cudaGraph_t g = nullptr;
        const long long l0 = launch_counter();
        CUDA_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
            run_forward(*impl_, lane, tp, nullptr, 0, s);
        } catch (...) {
            cudaStreamEndCapture(s, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        CUDA_CHECK(cudaStreamEndCapture(s, &g));
        c.graph_nodes[tp] = launch_counter() - l0;
        launch_counter() = l0;  // counted when replayed
        cudaGraphExec_t exec = nullptr;
        CUDA_CHECK(cudaGraphInstantiate(&exec, g, 0));
        CUDA_CHECK(cudaGraphDestroy(g));
        it = c.graphs.emplace(tp, exec).first;
    }
    CUDA_CHECK(cudaGraphLaunch(it->second, s));
    launch_counter() += c.graph_nodes[tp];
}

void Transformer::logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) {
    // logits rows are written for every processed position; the caller's row0 == start here
    run_forward(*impl_, lane, max_tokens, out_dev, cfg_.vocab, s);
}

namespace {
void run_forward(Transformer::Impl& m, Lane& lane, int max_tokens, float* logits, int ld_logits, cudaStream_t s) {
    if (max_tokens < 1) max_tokens = 1;
    if (max_tokens > kMaxTp) throw_runtime("forward exceeds 256 token columns (decoder must chunk)");
    const int tp = (max_tokens + 15) / 16 * 16;
    TfCache& c = *static_cast<TfCache*>(lane.cache.get());
    const auto& cfg = m.c;
    const int h = m.h;
    // every GEMM goes through G (optional per-launch event timing for the bench roofline)
    const GemmNext* nx = nullptr;  // the GEMM after the one being launched (L2 warm-up target)
    auto G = [&](Epi e, const CUtensorMap& W, const CUtensorMap& X, int n_out, int K, int n_valid, void* out, int ld,
                 float* lgp, int ldl, const LaneState* ln) {
        if (m.prof) m.prof->next(s);
        gemm_launch(e, W, X, n_out, K, tp, n_valid, out, ld, lgp, ldl, c.ws, s, ln, nx);
        if (m.prof) {
            m.prof->next(s);
            m.prof->bytes.push_back(2.0 * n_out * K + 2.0 * tp * K);
        }
    };
    launch_forward_begin(lane.state, s);
    launch_embed(m.embed.p, h, lane.buf.p, lane.state, tp, c.resid.p, s);
    for (int l = 0; l < cfg.n_layers; ++l) {
        LayerW& w = m.layers[l];
        KVView kv{c.kbuf.p + c.layer_stride * l, c.vbuf.p + c.layer_stride * l, c.page_table.p, m.nkv, m.hd};
        const GemmNext n_o{&w.t_o, h, m.q_dim}, n_gu{&w.t_gu, 2 * m.ffn_l, h}, n_down{&w.t_down, h, m.ffn_l};
        const GemmNext n_after = l + 1 < cfg.n_layers ? GemmNext{&m.layers[l + 1].t_qkv, m.qkv_rows, h}
                                                      : GemmNext{&m.t_lm, m.vocab_l, h};
        launch_rmsnorm(c.resid.p, w.attn_norm.p, h, cfg.rms_eps, tp, c.xn.p, s);
        nx = &n_o;
        G(Epi::StoreBF16, w.t_qkv, c.t_xn, m.qkv_rows, h, m.qkv_rows, c.qkv.p, m.qkv_rows, nullptr, 0, nullptr);
        launch_qkv_post(c.qkv.p, m.nh, m.nkv, m.hd, cfg.qk_norm ? w.q_norm.p : nullptr,
                        cfg.qk_norm ? w.k_norm.p : nullptr, cfg.rms_eps, cfg.rope_theta, lane.state, kv, c.qbuf.p, tp, s);
        launch_attention(c.qbuf.p, m.nh, m.nkv, m.hd, kv, lane.state, tp, c.max_chunks, c.part_o.p, c.part_ml.p,
                         c.attn.p, s);
        nx = &n_gu;
        if (m.world == 1) {
            G(Epi::ResidAdd, w.t_o, c.t_attn, h, m.q_dim, h, c.resid.p, h, nullptr, 0, nullptr);
        } else {
            G(Epi::StoreF32, w.t_o, c.t_attn, h, m.q_dim, h, c.tp_partial.p, h, nullptr, 0, nullptr);
            m.comm->allreduce_add(c.tp_partial.p, tp, h, c.resid.p, s);
        }
        launch_rmsnorm(c.resid.p, w.mlp_norm.p, h, cfg.rms_eps, tp, c.xn.p, s);
        nx = &n_down;
        G(Epi::SiluMul, w.t_gu, c.t_xn, 2 * m.ffn_l, h, 2 * m.ffn_l, c.act.p, m.ffn_l, nullptr, 0, nullptr);
        nx = &n_after;
        if (m.world == 1) {
            G(Epi::ResidAdd, w.t_down, c.t_act, h, m.ffn_l, h, c.resid.p, h, nullptr, 0, nullptr);
        } else {
            G(Epi::StoreF32, w.t_down, c.t_act, h, m.ffn_l, h, c.tp_partial.p, h, nullptr, 0, nullptr);
            m.comm->allreduce_add(c.tp_partial.p, tp, h, c.resid.p, s);
        }
    }
    launch_rmsnorm(c.resid.p, m.final_norm.p, h, cfg.rms_eps, tp, c.xn.p, s);
    const int lm_tiles = (m.vocab_l + 127) / 128;
    float* lg = logits ? logits + static_cast<size_t>(m.rank) * m.vocab_l : nullptr;
    nx = nullptr;
    G(Epi::Argmax, m.t_lm, c.t_xn, m.vocab_l, h, m.vocab_l, nullptr, 0, lg, ld_logits, lane.state);
    if (m.world == 1) {
        argmax_finish(c.ws, lm_tiles, tp, lane.state, lane.argmax.p, s);
    } else {
        m.comm->argmax_combine(c.ws, lm_tiles, tp, m.rank * m.vocab_l, lane.state, lane.argmax.p, s);
        if (logits) m.comm->gather_logits(logits, tp, m.vocab_l, ld_logits, s);
    }
    launch_forward_end(lane.state, s);
}
}  // namespace

void Transformer::get_weight(const std::string& name, int layer, uint16_t* out, int64_t numel) {
    Impl& m = *impl_;
    if (m.world != 1) throw_invalid("get_weight: only for unsharded models");
    if (!out) throw_invalid("null out");
    DeviceGuard g(device_);
    const int h = m.h;
    auto fetch = [&](const __nv_bfloat16* src, int64_t n, std::vector<uint16_t>& dst) {
        dst.resize(n);
        CUDA_CHECK(cudaMemcpy(dst.data(), src, n * 2, cudaMemcpyDeviceToHost));
    };
    std::vector<uint16_t> v;
    auto need_layer = [&]() -> LayerW& {
        if (layer < 0 || layer >= cfg_.n_layers) throw_invalid("get_weight: layer out of range");
        return m.layers[layer];
    };
    if (name == "embed") fetch(m.embed.p, static_cast<int64_t>(cfg_.vocab) * h, v);
    else if (name == "lm_head") fetch(m.lm_head, static_cast<int64_t>(m.vocab_l) * h, v);
    else if (name == "final_norm") fetch(m.final_norm.p, h, v);
    else if (name == "attn_norm") fetch(need_layer().attn_norm.p, h, v);
    else if (name == "mlp_norm") fetch(need_layer().mlp_norm.p, h, v);
    else if (name == "q_norm" && cfg_.qk_norm) fetch(need_layer().q_norm.p, m.hd, v);
    else if (name == "k_norm" && cfg_.qk_norm) fetch(need_layer().k_norm.p, m.hd, v);
    else if (name == "q_proj") fetch(need_layer().qkv.p, static_cast<int64_t>(m.q_dim) * h, v);
    else if (name == "k_proj") fetch(need_layer().qkv.p + static_cast<size_t>(m.q_dim) * h, static_cast<int64_t>(m.kv_dim) * h, v);
    else if (name == "v_proj")
        fetch(need_layer().qkv.p + static_cast<size_t>(m.q_dim + m.kv_dim) * h, static_cast<int64_t>(m.kv_dim) * h, v);
    else if (name == "o_proj") fetch(need_layer().o.p, static_cast<int64_t>(h) * m.q_dim, v);
    else if (name == "down_proj") fetch(need_layer().down.p, static_cast<int64_t>(h) * m.ffn_l, v);
    else if (name == "gate_proj" || name == "up_proj") {
        std::vector<uint16_t> gu;
        fetch(need_layer().gateup.p, static_cast<int64_t>(2) * m.ffn_l * h, gu);
        const int half = name == "up_proj";
        v.resize(static_cast<size_t>(m.ffn_l) * h);
        for (int64_t p = 0; p < 2LL * m.ffn_l; ++p) {
            if (((p % 32) / 16) != half) continue;
            const int64_t f = (p / 128) * 64 + ((p % 128) / 32) * 16 + p % 16;
            std::memcpy(v.data() + f * h, gu.data() + p * h, h * 2);
        }
    } else {
        throw_invalid("get_weight: unknown tensor " + name);
    }
    if (static_cast<int64_t>(v.size()) != numel)
        throw_invalid("get_weight: numel mismatch (tensor has " + std::to_string(v.size()) + ")");
    std::memcpy(out, v.data(), v.size() * 2);
}

}  // namespace dbl
