// Random-init bf16 decoder-only transformer (Qwen3 / Llama shapes) behind the forward_batch contract.
//
// One forward processes the lane positions [start, L+c) padded to tp (multiple of 16) token columns:
//   embed -> L x [RMSNorm -> QKV GEMM -> qk-norm/RoPE/KV append -> split-KV attention -> O GEMM (+resid)
//                 -> RMSNorm -> gate|up GEMM (SiLU*up epilogue) -> down GEMM (+resid)]
//         -> RMSNorm -> LM head GEMM (fused per-tile argmax) -> argmax combine
// and runs as ONE persistent kernel (fwd.cu, design in fwd.cuh): every weight byte is streamed from
// HBM exactly once per forward by TMA into tcgen05 tiles, with the activations of each phase gated by
// device-side completion counters — the verify step's roofline is the weight stream.
// Tensor parallel (tp_size > 1) is declared (column-parallel QKV / gate|up, row-parallel O / down,
// vocab-parallel LM head, shard-exact init) but its exchange is not implemented yet (tp.cu).
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fwd.cuh"
#include "gemm.cuh"
#include "tf_kernels.cuh"
#include "sampling.cuh"
#include "transformer.cuh"

namespace dbl {

namespace {
constexpr int kMaxTp = 256;  // token columns per forward (UMMA N limit)
enum TensorId : uint64_t { kEmbed = 1, kLmHead = 2 };
inline uint64_t layer_id(int l, int which) { return 1000 + static_cast<uint64_t>(l) * 16 + which; }
enum { kQ = 0, kK = 1, kV = 2, kO = 3, kGate = 4, kUp = 5, kDown = 6 };
}  // namespace

struct LayerW {
    DevBuf<__nv_bfloat16> attn_norm, mlp_norm, q_norm, k_norm;
    __nv_bfloat16 *qkv = nullptr, *o = nullptr, *gateup = nullptr, *down = nullptr;  // views into Impl::w_*
};

struct Transformer::Impl {
    dbl_transformer_config c;
    int rank = 0, world = 1;
    int nh, nkv, hd, h, q_dim, kv_dim, qkv_rows, ffn_l, vocab_l;
    std::vector<LayerW> layers;
    DevBuf<__nv_bfloat16> embed, final_norm, lm_head_own;
    const __nv_bfloat16* lm_head = nullptr;
    // every layer's projection of one kind is stored contiguously ([layers * rows, cols]) so a whole
    // forward streams through five tensor maps (kernel parameters, not global-memory descriptors)
    DevBuf<__nv_bfloat16> w_qkv, w_o, w_gu, w_down;
    CUtensorMap t_qkv, t_o, t_gu, t_down, t_lm;
    GemmProfiler* prof = nullptr;
    int smem_budget = kFwdSmemBudget;  // per forward CTA (fwd.cuh: the target / draft roles)
    int grid_div = 1;                  // draft beside a target: a forward on 1/grid_div of the SMs,
    bool coop = true;                  // launched plainly so it runs beside the target's grid
    // one process per shard (IPC): this rank's exchange buffers (model-level, exported once), every
    // rank's addresses (peers' opened from their IPC handles) and the model-level exchange-tag counter
    DevBuf<float> ipc_xch;
    DevBuf<unsigned long long> ipc_xflag, ipc_aflag, ipc_epoch;
    DevBuf<float2> ipc_axch;
    TpPeers ipc_peers{};
    bool ipc_linked = false;
    std::vector<void*> ipc_opened;
};

void Transformer::set_profiler(GemmProfiler* p) { impl_->prof = p; }

struct TfCache final : LaneCache {
    int capacity, pages, max_chunks;
    DevBuf<__nv_bfloat16> kbuf, vbuf;  // [layers][pages][nkv][kPage][hd]
    DevBuf<int32_t> page_table;
    DevBuf<float> resid, ssq, part_o, part_ml;
    DevBuf<__nv_bfloat16> xb, qbuf, attn, act;
    DevBuf<int> err;
    DevBuf<float2> rope;                    // [capacity][hd/2] (cos, sin)
    DevBuf<FwdPhase> phases;
    CUtensorMap xmaps[3][5];  // xb, attn, act x boxes of 4, 8, 16, 32, 64 token rows
    DevBuf<unsigned long long> done, epoch, slot_flag;
    DevBuf<int> row_base;  // batched forwards: per-lane forward-row base (FwdBatch::row_base)
    // tensor parallel: this rank's exchange buffers (written by every rank) and all ranks' addresses
    DevBuf<float> xch;
    DevBuf<unsigned long long> xflag, aflag;
    DevBuf<float2> axch;
    TpPeers peers{};
    int n_ph = 0;
    int grid = 0;  // CTAs per forward (the phase table's split is built for this grid)
    int grid_div = 1;
    GemmWorkspace ws;
    size_t layer_stride = 0;
};

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
    (void)nccl_comm;  // the tensor-parallel exchange runs inside fwd_kernel over peer memory (tp.cu)
    if (world > kMaxTpRanks) throw_invalid("transformer: tp_size > 8");
    cudaStream_t s = 0;
    const uint64_t seed = c.seed;
    const float sd_embed = c.init_std;  // embedding / LM head
    const float sd_scaled = c.init_std * (c.layer_std_scale > 0.f ? c.layer_std_scale : 1.f);
    const int h = m.h;
    m.layers.resize(c.n_layers);
    // weights live in HBM as tiled images (launch_tile_weights: every 128 x 64 tile one contiguous
    // 16 KiB block, so a CTA's stream-K range is one sequential read); each is generated row-major
    // into `scratch` first
    const size_t n_qkv = static_cast<size_t>(tiled_rows(m.qkv_rows)) * h, n_o = static_cast<size_t>(tiled_rows(h)) * m.q_dim;
    const size_t n_gu = static_cast<size_t>(tiled_rows(2LL * m.ffn_l)) * h, n_down = static_cast<size_t>(tiled_rows(h)) * m.ffn_l;
    m.w_qkv.alloc(n_qkv * c.n_layers);
    m.w_o.alloc(n_o * c.n_layers);
    m.w_gu.alloc(n_gu * c.n_layers);
    m.w_down.alloc(n_down * c.n_layers);
    DevBuf<__nv_bfloat16> scratch;
    scratch.alloc(std::max({n_qkv, n_o, n_gu, n_down, static_cast<size_t>(tiled_rows(m.vocab_l) * h)}));
    for (int l = 0; l < c.n_layers; ++l) {
        LayerW& w = m.layers[l];
        const float sd = l >= c.scale_from_layer ? sd_scaled : sd_embed;  // decoder layer l
        // RMSNorm weights are 1 in this random-init family; the stream forward folds them (fwd.cuh)
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
        w.qkv = m.w_qkv.p + n_qkv * l;
        launch_init_qkv(scratch.p, m.q_dim, m.kv_dim, m.hd, h, seed, layer_id(l, kQ), layer_id(l, kK), layer_id(l, kV),
                        static_cast<int64_t>(m.rank) * m.q_dim, static_cast<int64_t>(m.rank) * m.kv_dim, sd, s);
        launch_tile_weights(w.qkv, scratch.p, m.qkv_rows, h, s);
        w.o = m.w_o.p + n_o * l;
        launch_init_normal(scratch.p, h, m.q_dim, m.q_dim, seed, layer_id(l, kO), 0,
                           static_cast<int64_t>(m.rank) * m.q_dim, static_cast<int64_t>(c.n_heads) * m.hd, sd, s);
        launch_tile_weights(w.o, scratch.p, h, m.q_dim, s);
        w.gateup = m.w_gu.p + n_gu * l;
        launch_init_gateup(scratch.p, m.ffn_l, h, seed, layer_id(l, kGate), layer_id(l, kUp),
                           static_cast<int64_t>(m.rank) * m.ffn_l, sd, s);
        launch_tile_weights(w.gateup, scratch.p, 2 * m.ffn_l, h, s);
        w.down = m.w_down.p + n_down * l;
        launch_init_normal(scratch.p, h, m.ffn_l, m.ffn_l, seed, layer_id(l, kDown), 0,
                           static_cast<int64_t>(m.rank) * m.ffn_l, c.ffn, sd, s);
        launch_tile_weights(w.down, scratch.p, h, m.ffn_l, s);
    }
    const uint64_t nl = static_cast<uint64_t>(c.n_layers);
    m.t_qkv = make_tmap_bf16_tiled(m.w_qkv.p, nl * n_qkv / (128 * 64));
    m.t_o = make_tmap_bf16_tiled(m.w_o.p, nl * n_o / (128 * 64));
    m.t_gu = make_tmap_bf16_tiled(m.w_gu.p, nl * n_gu / (128 * 64));
    m.t_down = make_tmap_bf16_tiled(m.w_down.p, nl * n_down / (128 * 64));
    m.final_norm.alloc(h);
    launch_fill(m.final_norm.p, h, 1.0f, s);
    m.embed.alloc(static_cast<size_t>(c.vocab) * h);
    launch_init_normal(m.embed.p, c.vocab, h, h, seed, kEmbed, 0, 0, h, sd_embed, s);
    // the LM head is streamed, so it is tiled too; a tied model keeps the row-major table for the
    // embedding gather and a tiled copy of its vocab shard for the head
    m.lm_head_own.alloc(tiled_rows(m.vocab_l) * h);
    if (c.tied_embeddings) {
        launch_tile_weights(m.lm_head_own.p, m.embed.p + static_cast<size_t>(m.rank) * m.vocab_l * h, m.vocab_l, h, s);
    } else {
        launch_init_normal(scratch.p, m.vocab_l, h, h, seed, kLmHead, static_cast<int64_t>(m.rank) * m.vocab_l, 0,
                           h, sd_embed, s);
        launch_tile_weights(m.lm_head_own.p, scratch.p, m.vocab_l, h, s);
    }
    m.lm_head = m.lm_head_own.p;
    m.t_lm = make_tmap_bf16_tiled(m.lm_head, tiled_rows(m.vocab_l) / 128 * (h / 64));
    CUDA_CHECK(cudaDeviceSynchronize());  // before `scratch` is freed
}

Transformer::~Transformer() {
    cudaSetDevice(device_);
    cudaDeviceSynchronize();
    pool_.clear();
    for (void* p : impl_->ipc_opened) cudaIpcCloseMemHandle(p);
    delete impl_;
}

int64_t Transformer::weight_bytes() const { return weight_bytes_of(*impl_); }

int64_t Transformer::weight_bytes_of(const Impl& m) {
    const int64_t per_layer = (static_cast<int64_t>(m.qkv_rows) * m.h + static_cast<int64_t>(m.h) * m.q_dim +
                               2LL * m.ffn_l * m.h + static_cast<int64_t>(m.h) * m.ffn_l) * 2 +
                              2LL * m.h * 2 + (m.c.qk_norm ? 4LL * m.hd : 0);
    return per_layer * m.c.n_layers + static_cast<int64_t>(m.vocab_l) * m.h * 2 + m.h * 2;
}

int64_t Transformer::kv_bytes_per_token() const {
    const Impl& m = *impl_;
    return static_cast<int64_t>(cfg_.n_layers) * 2 * m.nkv * m.hd * 2;
}

int Transformer::max_forward_tokens() const { return kMaxTp; }

void Transformer::recycle_cache(std::unique_ptr<LaneCache> c) {
    if (!c || impl_->world != 1) return;  // tensor-parallel shard caches are linked to their peers
    std::lock_guard<std::mutex> lk(pool_mu_);
    if (pool_.size() < 4) pool_.push_back(std::move(c));
}

std::unique_ptr<LaneCache> Transformer::make_cache(int capacity) {
    if (impl_->world == 1) {
        std::lock_guard<std::mutex> lk(pool_mu_);
        for (auto it = pool_.begin(); it != pool_.end(); ++it) {
            const TfCache* pc = static_cast<TfCache*>(it->get());
            // exact capacity (batched forwards need every lane's KV at the same stride) and the grid the
            // phase table was split for
            if (pc->capacity == capacity && pc->grid_div == impl_->grid_div) {
                std::unique_ptr<LaneCache> c = std::move(*it);
                pool_.erase(it);
                return c;
            }
        }
    }
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
    c.ssq.alloc(static_cast<size_t>(m.h / 128) * kMaxTp);
    c.xb.alloc(static_cast<size_t>(kMaxTp) * m.h);
    c.qbuf.alloc(static_cast<size_t>(kMaxTp) * m.q_dim);
    c.attn.alloc(static_cast<size_t>(kMaxTp) * m.q_dim);
    c.act.alloc(static_cast<size_t>(kMaxTp) * m.ffn_l);
    c.xb.zero();
    c.attn.zero();
    c.act.zero();
    c.part_o.alloc(static_cast<size_t>(kMaxTp) * m.nh * c.max_chunks * m.hd);
    c.part_ml.alloc(static_cast<size_t>(kMaxTp) * m.nh * c.max_chunks * 2);
    c.err.alloc(1);
    c.err.zero();
    {  // RoPE table (rotate-half): angle(pos, i) = pos * theta^(-2i/hd)
        const int half = m.hd / 2;
        std::vector<float2> tab(static_cast<size_t>(capacity) * half);
        for (int p = 0; p < capacity; ++p)
            for (int i = 0; i < half; ++i) {
                const double inv = std::pow(static_cast<double>(cfg_.rope_theta), -2.0 * i / m.hd);
                const double ang = static_cast<double>(p) * inv;
                tab[static_cast<size_t>(p) * half + i] = make_float2(static_cast<float>(std::cos(ang)),
                                                                     static_cast<float>(std::sin(ang)));
            }
        c.rope.alloc(tab.size());
        CUDA_CHECK(cudaMemcpy(c.rope.p, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
    }
    const int max_tiles = std::max({(m.qkv_rows + 127) / 128, (2 * m.ffn_l + 127) / 128, (m.vocab_l + 127) / 128,
                                    (m.h + 127) / 128});
    // CTAs of this model's forward: one per SM, or 1/k of the SMs when k tensor-parallel shards share
    // the GPU (every shard's grid must be resident at once)
    static const int env_div = [] {  // DBL_FWD_GRID_DIV=k: every forward on 1/k of the SMs (experiment)
        const char* e = std::getenv("DBL_FWD_GRID_DIV");
        return e ? std::max(1, std::atoi(e)) : 1;
    }();
    const int sms = std::max(1, num_sms(device_) / std::max(1, shards_per_device_) / env_div / impl_->grid_div);
    c.grid = sms;
    c.grid_div = impl_->grid_div;
    c.ws.ensure(sms, kMaxTp, max_tiles);
    // ---- the forward's phase list (fwd.cuh); tensor maps: W 0..4 = qkv, o, gate|up, down, lm head;
    // X 0..2 = xb, attn, act
    for (int b = 0; b < 5; ++b) {
        c.xmaps[0][b] = make_tmap_bf16_2d(c.xb.p, kMaxTp, m.h, 4 << b);
        c.xmaps[1][b] = make_tmap_bf16_2d(c.attn.p, kMaxTp, m.q_dim, 4 << b);
        c.xmaps[2][b] = make_tmap_bf16_2d(c.act.p, kMaxTp, m.ffn_l, 4 << b);
    }
    const int x_xb = 0, x_attn = 1, x_act = 2;
    std::vector<FwdPhase> ph;
    int offset = 0;
    auto add = [&](FwdPhase p) {
        p.dep = ph.empty() ? -1 : static_cast<int>(ph.size()) - 1;
        if (p.kind == kPhGemm) {
            p.n_tiles = (p.n_out + 127) / 128;
            p.kb = p.K / 64;
            const long long units = static_cast<long long>(p.n_tiles) * p.kb;
            if ((units + 1) * (sms + 1) >= (1LL << 31)) throw_invalid("stream forward: projection too large for 32-bit units");
            p.units = static_cast<int>(units);
            p.active = std::max(1, std::min(sms, p.units / kFwdMinUnits));
            p.offset = offset;
            offset = (offset + p.active) % sms;
            p.count = p.n_tiles;
        } else {
            p.active = sms;
            p.count = sms;
        }
        ph.push_back(p);
    };
    auto gemm = [&](int epi, int wmap, int xmap, int n_out, int K, int layer) {
        FwdPhase p{};
        p.kind = kPhGemm;
        p.epi = epi;
        p.wmap = wmap;
        p.w_row0 = layer >= 0 ? layer * static_cast<int>(tiled_rows(n_out)) : 0;  // tiled images: padded rows
        p.xmap = xmap;
        p.n_out = n_out;
        p.K = K;
        p.layer = layer;
        if (layer >= 0) {
            p.kc = c.kbuf.p + c.layer_stride * layer;
            p.vc = c.vbuf.p + c.layer_stride * layer;
            p.qn = cfg_.qk_norm ? m.layers[layer].q_norm.p : nullptr;
            p.kn = cfg_.qk_norm ? m.layers[layer].k_norm.p : nullptr;
        }
        add(p);
    };
    {
        FwdPhase e{};
        e.kind = kPhEmbed;
        e.layer = -1;
        add(e);
    }
    for (int l = 0; l < cfg_.n_layers; ++l) {
        gemm(kFeQkv, 0, x_xb, m.qkv_rows, m.h, l);
        FwdPhase at{};
        at.kind = kPhAttn;
        at.layer = l;
        at.kc = c.kbuf.p + c.layer_stride * l;
        at.vc = c.vbuf.p + c.layer_stride * l;
        add(at);
        FwdPhase cb{};
        cb.kind = kPhCombine;
        cb.layer = l;
        add(cb);
        gemm(kFeResid, 1, x_attn, m.h, m.q_dim, l);
        gemm(kFeSilu, 2, x_xb, 2 * m.ffn_l, m.h, l);
        gemm(kFeResid, 3, x_act, m.h, m.ffn_l, l);
    }
    gemm(kFeLogits, 4, x_xb, m.vocab_l, m.h, -1);
    {
        FwdPhase am{};
        am.kind = kPhArgmax;
        am.layer = -1;
        add(am);
    }
    c.n_ph = static_cast<int>(ph.size());
    c.phases.alloc(ph.size());
    CUDA_CHECK(cudaMemcpy(c.phases.p, ph.data(), ph.size() * sizeof(FwdPhase), cudaMemcpyHostToDevice));
    c.done.alloc(ph.size());
    c.done.zero();
    c.epoch.alloc(1);
    c.epoch.zero();
    if (ph.size() >= 4095) throw_invalid("stream forward: too many phases for the slot-flag tag");
    c.slot_flag.alloc(2 * static_cast<size_t>(sms) + 2);
    c.slot_flag.zero();
    if (m.world > 1 && m.ipc_linked) {
        c.peers = m.ipc_peers;  // one process per shard: the model-level buffers, linked once
    } else if (m.world > 1) {
        const size_t nth = static_cast<size_t>(m.h / 128);
        c.xch.alloc(kMaxTpRanks * nth * kMaxTp * 128);
        c.xflag.alloc(kMaxTpRanks * nth);
        c.xflag.zero();
        c.axch.alloc(static_cast<size_t>(kMaxTpRanks) * kMaxTp);
        c.aflag.alloc(kMaxTpRanks);
        c.aflag.zero();
    }
    CUDA_CHECK(cudaDeviceSynchronize());
    return cp;
}

namespace {
void run_forward(Transformer::Impl& m, int device, LaneState* state, const int32_t* buf, int32_t* argmax,
                 LaneCache* cache, int max_tokens, float* logits, int ld_logits, cudaStream_t s,
                 const std::vector<Lane*>* batch = nullptr) {
    if (max_tokens < 1) max_tokens = 1;
    if (max_tokens > kMaxTp) throw_runtime("forward exceeds 256 token columns (decoder must chunk)");
    int tp = (max_tokens + 15) / 16 * 16;
    TfCache& c = *static_cast<TfCache*>(cache);
    if (m.world > 1 && !c.peers.xch[m.world - 1]) throw_logic("tensor-parallel lane cache not linked to its peers");
    FwdArgs a{};
    a.ph = c.phases.p;
    a.n_ph = c.n_ph;
    a.wmaps[0] = m.t_qkv;
    a.wmaps[1] = m.t_o;
    a.wmaps[2] = m.t_gu;
    a.wmaps[3] = m.t_down;
    a.wmaps[4] = m.t_lm;
    for (int i = 0; i < 3; ++i)
        for (int b = 0; b < 5; ++b) a.xmaps[i][b] = c.xmaps[i][b];
    a.dbg = [] {
        const char* e = std::getenv("DBL_FWD_DBG");
        return e ? std::atoi(e) : 0;
    }();
    if (a.dbg >= 4 && a.dbg <= 8) tp = std::max(tp, 32);  // experiments: the 32-column machinery at <= 16 tokens (5: epilogues on the first 16 columns only)
    a.tp = tp;
    size_t smem = 0;
    a.stages = fwd_stages(tp, m.smem_budget, &smem);
    a.acc_cols = tp <= 32 ? 32 : tp <= 64 ? 64 : tp <= 128 ? 128 : 256;
    a.nacc = tp <= 128 ? 2 : 1;
    a.lane = state;
    a.buf = buf;
    a.argmax = argmax;
    a.embed = m.embed.p;
    a.h = m.h;
    a.nh = m.nh;
    a.nkv = m.nkv;
    a.hd = m.hd;
    a.q_dim = m.q_dim;
    a.kv_dim = m.kv_dim;
    a.ffn_l = m.ffn_l;
    a.vocab_l = m.vocab_l;
    a.max_chunks = c.max_chunks;
    a.eps = m.c.rms_eps;
    a.resid = c.resid.p;
    a.xb = c.xb.p;
    a.qbuf = c.qbuf.p;
    a.attn = c.attn.p;
    a.act = c.act.p;
    a.ssq = c.ssq.p;
    a.part_o = c.part_o.p;
    a.part_ml = c.part_ml.p;
    a.rope = c.rope.p;
    a.max_seq = c.capacity;
    a.page_table = c.page_table.p;
    a.ws = c.ws.partials.p;
    a.slot_flag = c.slot_flag.p;
    a.amax = c.ws.amax.p;
    a.logits = logits;
    a.ld_logits = ld_logits;
    a.done = c.done.p;
    a.epoch = c.epoch.p;
    a.err = c.err.p;
    a.wd_ns = [] {  // DBL_FWD_WATCHDOG_MS (tests shorten it); default 4 s
        const char* e = std::getenv("DBL_FWD_WATCHDOG_MS");
        const long long ms = e ? std::atoll(e) : 4000;
        return static_cast<unsigned long long>(ms > 0 ? ms : 4000) * 1000000ull;
    }();
    a.trace = fwd_trace_buffer(c.n_ph, c.grid);
    a.tp_world = m.world;
    a.tp_rank = m.rank;
    a.vocab_off = m.rank * m.vocab_l;
    a.peers = c.peers;
    a.tp_epoch = m.ipc_linked ? m.ipc_epoch.p : nullptr;
    if (batch) {  // several lanes in one forward; lane 0's cache holds the shared scratch and phase table
        if (batch->empty() || static_cast<int>(batch->size()) > kMaxBatch)
            throw_invalid("batched forward: 1.." + std::to_string(kMaxBatch) + " lanes");
        if (m.world > 1) throw_invalid("batched forward: tensor-parallel models are not supported");
        a.batch.n = static_cast<int>(batch->size());
        if (!c.row_base.p) c.row_base.alloc(kMaxBatch);
        a.batch.row_base = c.row_base.p;
        for (int b = 0; b < a.batch.n; ++b) {
            Lane& l = *(*batch)[b];
            TfCache& cb = *static_cast<TfCache*>(l.cache.get());
            if (cb.capacity != c.capacity) throw_invalid("batched forward: lanes must have equal capacity");
            a.batch.lane[b] = l.state;
            a.batch.buf[b] = l.buf.p;
            a.batch.argmax[b] = l.argmax.p;
            a.batch.page_table[b] = cb.page_table.p;
            a.batch.koff[b] = static_cast<long long>(reinterpret_cast<intptr_t>(cb.kbuf.p) -
                                                     reinterpret_cast<intptr_t>(c.kbuf.p)) / 2;
            a.batch.voff[b] = static_cast<long long>(reinterpret_cast<intptr_t>(cb.vbuf.p) -
                                                     reinterpret_cast<intptr_t>(c.vbuf.p)) / 2;
        }
    }
    // vocab-parallel logits: this rank's columns of the caller's [rows][vocab] buffer
    if (logits) a.logits = logits + static_cast<size_t>(m.rank) * m.vocab_l;
    if (m.prof) m.prof->next(s);
    fwd_launch(a, c.grid, smem, s, m.coop);
    if (m.prof) {
        m.prof->next(s);
        m.prof->bytes.push_back(static_cast<double>(Transformer::weight_bytes_of(m)));
    }
}
}  // namespace

void Transformer::set_smem_budget(int bytes) { impl_->smem_budget = bytes; }
void Transformer::set_draft_grid(int div) {
    impl_->grid_div = std::max(1, div);
    impl_->coop = impl_->grid_div == 1;
}

std::string Transformer::debug_state_hash(Lane& lane, int upto) {
    const Impl& m = *impl_;
    TfCache& c = *static_cast<TfCache*>(lane.cache.get());
    DeviceGuard g(device_);
    CUDA_CHECK(cudaDeviceSynchronize());
    auto fnv = [](const void* p, size_t n, unsigned long long h) {
        const unsigned char* b = static_cast<const unsigned char*>(p);
        for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
        return h;
    };
    std::string out;
    char buf[64];
    const int pages = (upto + kPage - 1) / kPage;
    std::vector<__nv_bfloat16> host(static_cast<size_t>(pages) * m.nkv * kPage * m.hd);
    for (int l = 0; l < cfg_.n_layers; ++l)
        for (int kv = 0; kv < 2; ++kv) {
            const __nv_bfloat16* src = (kv ? c.vbuf.p : c.kbuf.p) + c.layer_stride * l;
            CUDA_CHECK(cudaMemcpy(host.data(), src, host.size() * 2, cudaMemcpyDeviceToHost));
            unsigned long long h = 0xcbf29ce484222325ull;
            for (int pg = 0; pg < pages; ++pg)
                for (int hh = 0; hh < m.nkv; ++hh)
                    for (int ps = 0; ps < kPage; ++ps)
                        if (pg * kPage + ps < upto)
                            h = fnv(host.data() + ((static_cast<size_t>(pg) * m.nkv + hh) * kPage + ps) * m.hd, m.hd * 2, h);
            std::snprintf(buf, sizeof buf, "%s%d=%016llx ", kv ? "v" : "k", l, h);
            out += buf;
            if (l == 0 && kv == 0) {  // layer 0's K per page (one prefill piece per page at DBL_PREFILL_CHUNK=64)
                out += "[";
                for (int pg = 0; pg < pages; ++pg) {
                    unsigned long long hp = 0xcbf29ce484222325ull;
                    for (int hh = 0; hh < m.nkv; ++hh)
                        for (int ps = 0; ps < kPage; ++ps)
                            if (pg * kPage + ps < upto)
                                hp = fnv(host.data() + ((static_cast<size_t>(pg) * m.nkv + hh) * kPage + ps) * m.hd, m.hd * 2, hp);
                    std::snprintf(buf, sizeof buf, "%04llx ", hp & 0xffff);
                    out += buf;
                }
                out += "] ";
            }
        }
    return out;
}

void Transformer::forward(Lane& lane, int max_tokens, cudaStream_t s) {
    run_forward(*impl_, device_, lane.state, lane.buf.p, lane.argmax.p, lane.cache.get(), max_tokens, nullptr, 0, s);
}

void Transformer::forward_lanes(const std::vector<Lane*>& lanes, int max_tokens, cudaStream_t s) {
    if (lanes.empty()) return;
    Lane& l0 = *lanes[0];
    run_forward(*impl_, device_, l0.state, l0.buf.p, l0.argmax.p, l0.cache.get(), max_tokens, nullptr, 0, s, &lanes);
}

void Transformer::dists_lanes(const std::vector<Lane*>& lanes, int max_tokens, const std::vector<int>& max_rows,
                              const std::vector<double*>& outs, cudaStream_t s) {
    if (lanes.size() == 1) {
        dists(*lanes[0], max_tokens, max_rows[0], outs[0], s);
        return;
    }
    Lane& l0 = *lanes[0];
    const size_t need = static_cast<size_t>(std::max(max_tokens, 1)) * static_cast<size_t>(cfg_.vocab);
    if (l0.logit_scratch.n < need) l0.logit_scratch.alloc(need);
    run_forward(*impl_, device_, l0.state, l0.buf.p, l0.argmax.p, l0.cache.get(), max_tokens, l0.logit_scratch.p,
                cfg_.vocab, s, &lanes);
    const int* base = static_cast<TfCache*>(l0.cache.get())->row_base.p;
    for (size_t b = 0; b < lanes.size(); ++b)
        launch_softmax_rows(l0.logit_scratch.p, lanes[b]->state, cfg_.vocab, outs[b], max_rows[b], base + b, s);
}

void Transformer::logits(Lane& lane, int max_tokens, float* out_dev, cudaStream_t s) {
    // logits rows are written for every processed position; the caller's row0 == start here
    run_forward(*impl_, device_, lane.state, lane.buf.p, lane.argmax.p, lane.cache.get(), max_tokens, out_dev,
                cfg_.vocab, s);
}

void Transformer::forward_raw(LaneState* state, const int32_t* buf, int32_t* argmax, LaneCache* cache,
                              int max_tokens, float* logits_dev, cudaStream_t s) {
    DeviceGuard g(device_);
    run_forward(*impl_, device_, state, buf, argmax, cache, max_tokens, logits_dev, logits_dev ? cfg_.vocab : 0, s);
}

void Transformer::ensure_xbuf() {
    Impl& m = *impl_;
    if (m.world < 2) throw_invalid("tensor-parallel exchange: not a shard (tp_size < 2)");
    DeviceGuard g(device_);
    if (!m.ipc_xch.p) {
        const size_t nth = static_cast<size_t>(m.h / 128);
        m.ipc_xch.alloc(kMaxTpRanks * nth * kMaxTp * 128);
        m.ipc_xflag.alloc(kMaxTpRanks * nth);
        m.ipc_xflag.zero();
        m.ipc_axch.alloc(static_cast<size_t>(kMaxTpRanks) * kMaxTp);
        m.ipc_aflag.alloc(kMaxTpRanks);
        m.ipc_aflag.zero();
        m.ipc_epoch.alloc(1);
        m.ipc_epoch.zero();
        CUDA_CHECK(cudaDeviceSynchronize());
    }
}

void Transformer::link_models(const std::vector<Transformer*>& shards) {
    // in-process group: every shard addresses the others' model-level buffers directly (same device or
    // a peer device over NVLink) — the same exchange state the IPC path links across processes
    TpPeers p{};
    for (size_t r = 0; r < shards.size(); ++r) {
        shards[r]->ensure_xbuf();
        Impl& m = *shards[r]->impl_;
        if (m.rank != static_cast<int>(r) || m.world != static_cast<int>(shards.size()))
            throw_invalid("link_models: shards must be ranks 0..world-1 in order");
        p.xch[r] = m.ipc_xch.p;
        p.xflag[r] = m.ipc_xflag.p;
        p.axch[r] = m.ipc_axch.p;
        p.aflag[r] = m.ipc_aflag.p;
    }
    for (Transformer* t : shards) {
        t->impl_->ipc_peers = p;
        t->impl_->ipc_linked = true;
    }
}

void Transformer::ipc_export(void* out) {
    Impl& m = *impl_;
    ensure_xbuf();
    DeviceGuard g(device_);
    cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(out);
    CUDA_CHECK(cudaIpcGetMemHandle(&h[0], m.ipc_xch.p));
    CUDA_CHECK(cudaIpcGetMemHandle(&h[1], m.ipc_xflag.p));
    CUDA_CHECK(cudaIpcGetMemHandle(&h[2], m.ipc_axch.p));
    CUDA_CHECK(cudaIpcGetMemHandle(&h[3], m.ipc_aflag.p));
}

void Transformer::ipc_import(const void* all, int world) {
    Impl& m = *impl_;
    if (world != m.world) throw_invalid("ipc_import: handle count does not match tp_size");
    if (!m.ipc_xch.p) throw_logic("ipc_import: call ipc_export first");
    if (m.ipc_linked) throw_logic("ipc_import: already linked");
    DeviceGuard g(device_);
    const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(all);
    TpPeers p{};
    for (int r = 0; r < world; ++r) {
        if (r == m.rank) {
            p.xch[r] = m.ipc_xch.p;
            p.xflag[r] = m.ipc_xflag.p;
            p.axch[r] = m.ipc_axch.p;
            p.aflag[r] = m.ipc_aflag.p;
            continue;
        }
        void* ptr[4];
        for (int k = 0; k < 4; ++k) {
            CUDA_CHECK(cudaIpcOpenMemHandle(&ptr[k], h[4 * r + k], cudaIpcMemLazyEnablePeerAccess));
            m.ipc_opened.push_back(ptr[k]);
        }
        p.xch[r] = static_cast<float*>(ptr[0]);
        p.xflag[r] = static_cast<unsigned long long*>(ptr[1]);
        p.axch[r] = static_cast<float2*>(ptr[2]);
        p.aflag[r] = static_cast<unsigned long long*>(ptr[3]);
    }
    m.ipc_peers = p;
    m.ipc_linked = true;
}

void Transformer::link_tp(const std::vector<LaneCache*>& caches) {
    if (caches.size() > static_cast<size_t>(kMaxTpRanks) || caches.empty()) throw_invalid("link_tp: 1..8 caches");
    TpPeers p{};
    for (size_t r = 0; r < caches.size(); ++r) {
        TfCache& c = *static_cast<TfCache*>(caches[r]);
        if (!c.xch.p) throw_logic("link_tp: cache of a tp_size == 1 model");
        p.xch[r] = c.xch.p;
        p.xflag[r] = c.xflag.p;
        p.axch[r] = c.axch.p;
        p.aflag[r] = c.aflag.p;
    }
    for (LaneCache* lc : caches) static_cast<TfCache*>(lc)->peers = p;
}

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
    auto fetch_tiled = [&](const __nv_bfloat16* src, int rows, int K, std::vector<uint16_t>& dst) {  // row-major
        DevBuf<__nv_bfloat16> tmp;
        tmp.alloc(static_cast<size_t>(rows) * K);
        launch_untile_weights(tmp.p, src, rows, K, 0);
        CUDA_CHECK(cudaDeviceSynchronize());
        fetch(tmp.p, static_cast<int64_t>(rows) * K, dst);
    };
    std::vector<uint16_t> v;
    auto need_layer = [&]() -> LayerW& {
        if (layer < 0 || layer >= cfg_.n_layers) throw_invalid("get_weight: layer out of range");
        return m.layers[layer];
    };
    if (name == "embed") fetch(m.embed.p, static_cast<int64_t>(cfg_.vocab) * h, v);
    else if (name == "lm_head") fetch_tiled(m.lm_head, m.vocab_l, h, v);
    else if (name == "final_norm") fetch(m.final_norm.p, h, v);
    else if (name == "attn_norm") fetch(need_layer().attn_norm.p, h, v);
    else if (name == "mlp_norm") fetch(need_layer().mlp_norm.p, h, v);
    else if (name == "q_norm" && cfg_.qk_norm) fetch(need_layer().q_norm.p, m.hd, v);
    else if (name == "k_norm" && cfg_.qk_norm) fetch(need_layer().k_norm.p, m.hd, v);
    else if (name == "q_proj" || name == "k_proj" || name == "v_proj") {
        // stored with the rows of every head permuted (launch_init_qkv); returned in logical order
        const int region = name == "q_proj" ? 0 : name == "k_proj" ? 1 : 2;
        const int rows = region == 0 ? m.q_dim : m.kv_dim;
        const size_t off = region == 0 ? 0 : region == 1 ? m.q_dim : m.q_dim + m.kv_dim;
        std::vector<uint16_t> all;
        fetch_tiled(need_layer().qkv, m.qkv_rows, h, all);
        const uint16_t* phys = all.data() + off * h;
        v.resize(static_cast<size_t>(rows) * h);
        for (int p = 0; p < rows; ++p) {
            const int logical = (p / m.hd) * m.hd + qkv_perm_dim(p % m.hd, m.hd);
            std::memcpy(v.data() + static_cast<size_t>(logical) * h, phys + static_cast<size_t>(p) * h, h * 2);
        }
    }
    else if (name == "o_proj") fetch_tiled(need_layer().o, h, m.q_dim, v);
    else if (name == "down_proj") fetch_tiled(need_layer().down, h, m.ffn_l, v);
    else if (name == "gate_proj" || name == "up_proj") {
        std::vector<uint16_t> gu;
        fetch_tiled(need_layer().gateup, 2 * m.ffn_l, h, gu);
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
