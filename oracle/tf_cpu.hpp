// oracle/tf_cpu.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU port of the transformer models the CUDA path serves (the Qwen2-shaped target and the
// EAGLE-3-style drafter of paper_2510_26475_b200/csrc/model.h), as Model objects the restated
// engine (restate.hpp) can drive. The reference has no transformer (its engine is typed on
// TabularARModel, model.hpp:56-108), so this is what makes BASELINE cfg1 "CPU-runnable" and gives
// a CPU timing of the SAME workload as the GPU bench (bench.py cpu_baseline.same_workload_port).
//
// Same architecture and the same synthetic weights: the generator of model.cu init_normal_kernel
// (splitmix64(seed, tensor id, index) -> Box-Muller in double -> bf16), the same tensor ids, the
// gate/up rows interleaved pairwise. fp32 arithmetic with bf16 rounding where the CUDA path stores
// bf16 activations (normed inputs, q/k/v after RoPE, attention output, SwiGLU output, P of P.V),
// like tests/torch_ref.py. Every row is computed independently in a fixed order, so a row's
// logits do not depend on the batch or tree it is asked in (greedy SD == greedy decoding holds
// exactly on the CPU, as on the GPU).
//
// Parity: the forward is checked against the fp32 torch reference (tests/torch_ref.py) on the
// same weights (tests/test_tf_cpu.py) and, on the GPU, against the CUDA engine's rows.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "restate.hpp"

namespace orc {

struct TfShape {
    int V = 0, d = 0, L = 0, H = 0, KV = 0, hd = 128, dff = 0;
    float rope_theta = 1e6f, eps = 1e-6f, std = 0.02f, logit_scale = 1.0f;
    int qkv() const { return (H + 2 * KV) * hd; }
};

struct TfLayer {
    std::vector<uint16_t> qkv_w, qkv_b, o_w, gu_w, down_w;  // bf16 bit patterns, [rows][cols]
    std::vector<float> ln1, ln2;
};

// Weights of the target (L layers, tied LM head) and of its drafter (fc, norms, one layer with
// QKV input 2d, own LM head), generated exactly like model.cu's init_transformer / init_drafter.
struct TfWeights {
    TfShape s;
    std::vector<uint16_t> emb;  // [V][d]
    std::vector<TfLayer> layers;
    std::vector<float> final_norm;
    std::vector<float> rope;    // [max_pos][hd/2][2]
    int feat_layers[3] = {0, 0, 0};
    // drafter
    std::vector<uint16_t> fc_w, lm_w;
    std::vector<float> norm_emb, norm_hid, d_final;
    TfLayer dl;
    void init_target(const TfShape & s, uint64_t seed, int max_pos);
    void init_drafter(uint64_t seed);
};

// One sequence's cached forward state (KV per layer and the per-position outputs the models need).
struct TfSeqState {
    std::vector<int> tokens;              // positions covered
    std::vector<std::vector<float>> k, v;  // per layer [pos][KV*hd]
    std::vector<float> feats;             // target: [pos][3][d] EAGLE features (bf16-rounded)
    std::vector<float> hidden;            // drafter: [pos][d] output hidden state
    int root = 0;                         // drafter: positions >= root take their own previous hidden
};

class CpuTransformer : public Model {
public:
    explicit CpuTransformer(std::shared_ptr<const TfWeights> w, double temperature = 1.0);
    std::vector<double> logits(const std::vector<int> & ctx) const override;
    // target features [3][d] at position p of ctx (the drafter's input), computing what is missing
    std::vector<float> features(const std::vector<int> & ctx, int p) const;
    // fill positions [0, n) of ctx with synthetic K/V and features (timing samples: a long
    // context without its CPU prefill; the rows computed afterwards are real forwards over it)
    void synthetic_prefix(const std::vector<int> & ctx, int n, uint64_t seed) const;
    const TfWeights & weights() const { return *w_; }

private:
    std::shared_ptr<const TfWeights> w_;
    mutable std::mutex mu_;
    mutable std::vector<TfSeqState> cache_;  // small LRU of sequences (requests of a batch)
    TfSeqState & state_for(const std::vector<int> & ctx) const;
    void extend(TfSeqState & st, const std::vector<int> & ctx, bool want_logits, std::vector<float> * last) const;
};

class CpuEagleDrafter : public Model {
public:
    CpuEagleDrafter(std::shared_ptr<const TfWeights> w, std::shared_ptr<const CpuTransformer> target, int version = 0);
    std::vector<double> logits(const std::vector<int> & ctx) const override { return logits_at(ctx, 0); }
    std::vector<double> logits_at(const std::vector<int> & ctx, int depth) const override;
    void synthetic_prefix(const std::vector<int> & ctx, int n, uint64_t seed) const;

private:
    std::shared_ptr<const TfWeights> w_;
    std::shared_ptr<const CpuTransformer> tgt_;
    mutable std::mutex mu_;
    mutable std::vector<TfSeqState> cache_;
};

}  // namespace orc
