// pipefill/kfac/kfac.hpp — per-layer K-FAC calls of the PipeFisher path.
//
// Source-compatible with /root/reference/proj/include/pipefill/kfac/kfac.hpp
// for the hot-path subset: BatchTape, curvature_factors,
// precondition, KfacState, ngd_step, block_diag_split_factor and the flop
// helpers, SplitMix64.  curvature_factors / KfacState::update_factors run the
// tcgen05 SYRK (pf_curvature_syrk_grouped; tapes rounded to bf16, fp32
// accumulation), refresh_inverses the batched damped inverse, precondition /
// ngd_step the fused precondition-update (pf_precondition[_update]).
// forward_backward, empirical_fisher_block and train_toy are fixture/oracle
// code of the reference (out of scope) and are not declared.
// Implementation: paper_2211_14133_b200/csrc/host/kfac_host.cpp.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "pipefill/kfac/matrix.hpp"

namespace pipefill::kfac {

enum class Activation { Identity, Tanh };
enum class LossKind { MeanSquaredError, SoftmaxCrossEntropy };

/// Fully-connected network without biases (reference kfac.hpp:16-20).
struct TinyMlp {
    std::vector<Matrix> weights;
    std::vector<Activation> activations;
    LossKind loss = LossKind::MeanSquaredError;
};

/// Per-layer inputs a_l (d_in x batch) and output-gradients e_l (d_out x batch),
/// examples as columns; e carries the 1/|B| averaging (reference kfac.hpp:29-37).
struct BatchTape {
    std::vector<Matrix> layer_inputs;
    std::vector<Matrix> layer_errors;
    int batch_size = 0;
};

/// A_l = (1/batch) a a^T and B_l = (1/batch) e e^T (reference kfac.cpp:125-131).
std::pair<Matrix, Matrix> curvature_factors(const BatchTape& tape, int layer);

/// B_inv * G * A_inv (reference kfac.cpp:133-137); std::invalid_argument on
/// a shape mismatch.
Matrix precondition(const Matrix& grad, const Matrix& a_inv, const Matrix& b_inv);

/// Per-layer factors, damped inverses and staleness (reference kfac.hpp:60-73).
/// update_factors overwrites (no EMA) with ONE grouped SYRK launch over every
/// layer; refresh_inverses inverts every layer with ONE batched call.
struct KfacState {
    std::vector<Matrix> factor_a, factor_b;
    std::vector<Matrix> inv_a, inv_b;
    std::vector<int> staleness;
    std::vector<char> refreshed_this_step;
    double damping = 0.0;
    double learning_rate = 0.0;

    explicit KfacState(int layers = 0);
    bool has_inverses(int layer) const;
    void update_factors(const BatchTape& tape);
    void refresh_inverses();
};

struct NgdStepResult {
    bool used_plain_gradient = false;
};

/// theta_l <- theta_l - eta * B_inv G_l A_inv, the update fused into the
/// second GEMM's epilogue; layers without inverses take the plain gradient
/// and set the flag (reference kfac.cpp:186-201).
NgdStepResult ngd_step(TinyMlp& mlp, KfacState& state, const std::vector<Matrix>& gradients);

/// K principal diagonal blocks of size d/K (reference kfac.cpp:203-217).
std::vector<Matrix> block_diag_split_factor(const Matrix& m, int k);
double inversion_flops(int dim);
double block_diag_inversion_flops(int dim, int k);

/// Deterministic uniform stream for seeded fixtures (reference kfac.cpp:228-238).
struct SplitMix64 {
    std::uint64_t state;
    explicit SplitMix64(std::uint64_t seed) : state(seed) {}
    std::uint64_t next();
    double uniform();
    double symmetric();
};

}  // namespace pipefill::kfac
