// gemm.h -- tcgen05 bf16 GEMM launcher (gemm_sm100.cu).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

namespace rs {

// kEpiSwiGLU: gate/up rows interleaved per 256-row block as [128 gate, 128 up];
// kEpiSwiGLU2: interleaved pairwise (row 2i gate_i, row 2i+1 up_i) -- the model layout.
// kEpiQKVRope: QKV projection + bias, then RoPE on Q and K and the K/V cache store (SM-pair
// kernel only; replaces the separate RoPE / KV-store kernel).
enum GemmEpiKind { kEpiBF16 = 0, kEpiF32 = 1, kEpiResidual = 2, kEpiSwiGLU = 3, kEpiSwiGLU2 = 4, kEpiQKVRope = 5 };

// Where kEpiQKVRope sends its outputs: q [T][H][hd] and the per-token K/V cache slot
// ((layer * B + seq) * KV + kv_head) * max_ctx + phys (RowDesc of each token).
struct QkvStore {
    const void *rows = nullptr;  // RowDesc[T]
    const float *rope = nullptr; // [max_ctx][hd/2][2] cos, sin
    void *q = nullptr, *k = nullptr, *v = nullptr;
    int H = 0, KV = 0, layer = 0, B = 0, max_ctx = 0;
};

struct GemmEpi {
    int kind = kEpiBF16;
    void *out = nullptr;         // bf16 [M, ldo] (BF16/SwiGLU) or fp32 [M, ldo] (F32/Residual)
    int ldo = 0;
    const void *bias = nullptr;  // bf16 [N] (kEpiBF16 only)
    float scale = 1.0f;          // kEpiF32 only
    const int *row_map = nullptr;  // kEpiF32 only: output row of A-row m (-1 = drop); null = identity
    // kEpiF32 only, BN = 256: per (output row, 256-column tile) softmax partials of
    // y = out / tau over the tile's columns except the last global column (EOS):
    // stats[(orow * ntiles + tile) * 2] = max y, [.. + 1] = sum exp(y - max)   (fp64)
    double *stats = nullptr;
    double tau = 1.0;
    QkvStore qkv;                // kEpiQKVRope only
};

struct GemmArgs {
    const void *A = nullptr;  // bf16 [M, lda], K-major
    const void *B = nullptr;  // bf16 [N, ldb], K-major (weights)
    int M = 0, N = 0, K = 0, lda = 0, ldb = 0;
    int block_n = 0;          // 0 = auto (256)
    // kEpiResidual only: K split into `splits` balanced ranges whose partials are added to the
    // output in split order (deterministic; keep it a function of (N, K) only so a row's
    // result stays independent of M).
    int splits = 1;
    bool force_1sm = false;   // keep the single-SM kernel (e.g. fused softmax statistics tests)
    GemmEpi epi;
};

// SwiGLU layout: B rows are interleaved per 256-row block as [128 gate rows, 128 up rows];
// output column j = silu(gate_j) * up_j, N_out = N / 2.
void gemm_bf16(const GemmArgs &g, cudaStream_t st);

// 2D bf16 TMA map over a row-major [rows, cols] matrix (leading dim `ld` elements), box of
// 64 columns x box_rows rows, 128B swizzle (gemm_sm100.cu).
CUtensorMap make_tma_map_bf16(const void *base, int rows, int cols, int ld, int box_rows);

// SM-pair GEMM (gemm_2sm.cu): same contract as gemm_bf16 (C[M, N] = A . B^T, A = M token rows,
// B = N weight rows), computed with the weights as the 256-row M operand of
// tcgen05.mma.cta_group::2. block_n = token tile (0 = auto). No fused softmax statistics and
// no block-interleaved SwiGLU (kEpiSwiGLU2 only).
bool gemm2_supported(const GemmArgs &g);
void gemm2_bf16(const GemmArgs &g, cudaStream_t st);

}  // namespace rs
