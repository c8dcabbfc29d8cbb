// TEST INFRASTRUCTURE ONLY.  Declarations of the reference's toy-trainer API
// (proj/include/pipefill/kfac/kfac.hpp:25-45, :53-56, :101-128: the FP64 MLP
// fixture behind acceptance criteria 7-8), which this repo does not ship (out
// of scope).  They exist so /root/reference/proj/tests/acceptance.cpp
// compiles as one translation unit; acceptance_1_6.cpp never calls them, so
// nothing is defined and nothing links against them.
#pragma once

#include <cstdint>
#include <vector>

#include "pipefill/kfac/kfac.hpp"

namespace pipefill::kfac {

struct Batch {
    Matrix inputs;
    Matrix targets;
};

struct ForwardBackwardResult {
    double loss = 0.0;
    std::vector<Matrix> gradients;
    BatchTape tape;
};

ForwardBackwardResult forward_backward(const TinyMlp& mlp, const Batch& batch);
Matrix empirical_fisher_block(const BatchTape& tape, int layer);

enum class ToyOptimizer { Kfac, GradientDescent };

struct ToyConfig {
    std::vector<int> layer_dims{8, 1};
    Activation hidden_activation = Activation::Identity;
    LossKind loss = LossKind::MeanSquaredError;
    std::uint64_t data_seed = 42;
    int samples = 32;
    double condition_number = 1e3;
    int steps = 100;
    double learning_rate = 1e-3;
    double damping = 1e-3;
    int refresh_period = 1;
    ToyOptimizer optimizer = ToyOptimizer::Kfac;
};

struct ToyResult {
    std::vector<double> losses;
    std::vector<int> max_staleness;
    bool diverged = false;
    int divergence_step = -1;
};

ToyResult train_toy(const ToyConfig& config);
int steps_to_loss(const std::vector<double>& losses, double target);

}  // namespace pipefill::kfac
