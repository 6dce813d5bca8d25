/* ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this code; the
 * product (paper_2208_14049_b200) never links it.
 *
 * CPU restatement of the ensemble member forward pass, the per-member softmax
 * and the combination fold.
 *
 *  - Member forward: the reference has NO member arithmetic (its predictors sleep
 *    and emit hashes, /root/reference/proj/src/runtime/backend.cpp:33-69), so the
 *    MLP below is the oracle's own definition of the member contract
 *    `Predictor::predict(SampleView, span<float>)`
 *    (/root/reference/proj/include/enserve/runtime/backend.hpp:25-34): output
 *    depends only on (member, sample row), never on batching
 *    (backend.hpp:43-45).  Parity for this part is pinned against this file only
 *    ("parity unpinned" w.r.t. the reference).
 *  - bf16 mode quantises X, every weight matrix and every post-ReLU hidden
 *    activation to bf16 (round-to-nearest-even) at the points the sm_100a kernel
 *    does; biases and accumulation stay fp32.
 *  - Synthetic weights: Glorot-uniform U(+-sqrt(6/(fan_in+fan_out))) and biases
 *    U(+-0.01), keyed by splitmix64 (the mixer of backend.cpp:12-17) on
 *    (seed, layer, element index) — SURVEY.md §8-D.
 *  - Fold: restates PredictionAccumulator::fold_segment
 *    (/root/reference/proj/src/runtime/combine.cpp:93-136) over whole arrays.
 */
#ifndef ENSERVE_ORACLE_CPU_MEMBER_H
#define ENSERVE_ORACLE_CPU_MEMBER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_LAYERS 8

uint64_t orc_splitmix64(uint64_t x);
float orc_round_bf16(float x);

/* Element idx of W_l stored [fan_out][fan_in] row-major. */
float orc_weight(uint64_t seed, int layer, uint64_t idx, int fan_in, int fan_out);
float orc_bias(uint64_t seed, int layer, uint64_t idx);
/* Synthetic feature value for flat element `idx` of X (U[0,1), 24-bit exact). */
float orc_feature(uint64_t seed, uint64_t idx);
void orc_fill_features(uint64_t seed, size_t rows, size_t width, float* x);

typedef struct orc_mlp orc_mlp;

/* widths[0] = input width, widths[n_layers] = classes C. */
orc_mlp* orc_mlp_create(int n_layers, const int* widths, uint64_t seed,
                        int quantize_bf16);
void orc_mlp_destroy(orc_mlp* m);
int orc_mlp_classes(const orc_mlp* m);
/* out[rows][C] logits for rows of x[rows][width]. */
void orc_mlp_forward(const orc_mlp* m, const float* x, size_t rows, float* out);
/* Copies the (quantised) weights of layer l as stored [fan_out][fan_in]. */
void orc_mlp_layer(const orc_mlp* m, int l, float* w, float* b);

/* CNN member: an S x S one-channel image (x row of S*S), conv P x P stride P
 * -> c1 (ReLU), conv 3 x 3 pad 1 -> c2 (ReLU), dense (S/P)^2*c2 -> hidden
 * (ReLU) -> C.  Weight matrices, in generation order (layer index):
 *   0: [c1][P*P],     K index a*P + b (pixel (P*i+a, P*j+b) of block (i, j));
 *   1: [c2][9*c1],    K index tap*c1 + channel, tap = 3*(dh+1) + (dw+1);
 *   2: [hidden][G*G*c2], K index (h*G + w)*c2 + channel (HWC flatten);
 *   3: [C][hidden].
 * The convolutions are dense layers over im2col rows (zero outside the
 * image); bf16 mode rounds X, every weight and every post-ReLU activation. */
typedef struct orc_cnn orc_cnn;
orc_cnn* orc_cnn_create(int S, int P, int c1, int c2, int hidden, int C, uint64_t seed,
                        int quantize_bf16);
void orc_cnn_destroy(orc_cnn* m);
int orc_cnn_classes(const orc_cnn* m);
void orc_cnn_forward(const orc_cnn* m, const float* x, size_t rows, float* out);
/* The last layer's inputs (post-ReLU hidden activations) [rows][hidden]. */
void orc_cnn_hidden(const orc_cnn* m, const float* x, size_t rows, float* out);
void orc_cnn_layer(const orc_cnn* m, int l, float* w, float* b);

/* p = softmax(z) per row, fp32, expf(z - max) / sum. */
void orc_softmax_rows(const float* z, size_t rows, int C, float* p);

/* Fold rule: 0 = averaging, 1 = majority vote, 2 = weighted averaging. */
void orc_fold(int rule, int M, size_t rows, int C, const float* const* blocks,
              const double* weights, float* y, int32_t* winners);
/* Lowest-index argmax per row (strict >), as combine.cpp:120-122. */
void orc_argmax_rows(const float* y, size_t rows, int C, int32_t* out);

#ifdef __cplusplus
}
#endif

#endif
