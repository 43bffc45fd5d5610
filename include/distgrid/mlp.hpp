// distgrid/mlp.hpp — the MLP parameter containers of the reference API (mlp.hpp:10-62):
// DenseLayer / DenseLayerGrads / Mlp with the reference's Xavier initialisation order, so
// FieldParams built here holds exactly the reference's initial weights.  The networks are
// evaluated only as parts of a field (query_density / query_color / field_backward and the
// fused tcgen05 kernels of the training step), so Mlp has no free-standing forward/backward here.
#pragma once

#include <cmath>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <vector>

#include "distgrid/rng.hpp"

namespace distgrid {

enum class Activation : uint8_t { None = 0, ReLU = 1, Sigmoid = 2 };

struct DenseLayer {
  uint32_t in_width = 0;
  uint32_t out_width = 0;
  std::vector<double> weights;  // out x in, row-major
  std::vector<double> bias;
};

struct DenseLayerGrads {
  std::vector<double> weights;
  std::vector<double> bias;
};

struct MlpCache {  // kept for API shape: the device backward re-derives its activations
  std::vector<double> input;
  std::vector<std::vector<double>> pre_activations;
};

class Mlp {
 public:
  Mlp() = default;
  // weights U[-b, b], b = sqrt(6 / (in + out)), layer by layer; biases 0 (mlp.cpp:38-53)
  Mlp(std::span<const uint32_t> widths, Activation hidden_activation, Rng& rng) : act_(hidden_activation) {
    if (widths.size() < 2) throw std::invalid_argument("mlp: need at least input and output widths");
    for (size_t i = 0; i + 1 < widths.size(); ++i) {
      DenseLayer l;
      l.in_width = widths[i];
      l.out_width = widths[i + 1];
      l.weights.resize(size_t(l.in_width) * l.out_width);
      l.bias.assign(l.out_width, 0.0);
      const double b = std::sqrt(6.0 / double(l.in_width + l.out_width));
      for (double& w : l.weights) w = rng.uniform(-b, b);
      layers_.push_back(std::move(l));
    }
  }

  uint32_t input_width() const { return layers_.empty() ? 0 : layers_.front().in_width; }
  uint32_t output_width() const { return layers_.empty() ? 0 : layers_.back().out_width; }
  Activation hidden_activation() const { return act_; }
  std::vector<DenseLayer>& layers() { return layers_; }
  const std::vector<DenseLayer>& layers() const { return layers_; }

  std::vector<DenseLayerGrads> make_grads() const {
    std::vector<DenseLayerGrads> g;
    for (const DenseLayer& l : layers_) g.push_back({std::vector<double>(l.weights.size(), 0.0),
                                                     std::vector<double>(l.bias.size(), 0.0)});
    return g;
  }
  std::vector<std::span<double>> parameter_arrays() {
    std::vector<std::span<double>> a;
    for (DenseLayer& l : layers_) {
      a.emplace_back(l.weights);
      a.emplace_back(l.bias);
    }
    return a;
  }

 private:
  std::vector<DenseLayer> layers_;
  Activation act_ = Activation::ReLU;
};

}  // namespace distgrid
