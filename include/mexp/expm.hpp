// Drop-in for the reference's proj/include/mexp/expm.hpp (arXiv 1710.10989
// scaling and squaring with the reduced-product Taylor schemes), running on a
// B200: the 1-norm, the (m, s) selection, the scheme and the s squarings all
// happen on the device (C ABI: include/mexp_b200.h, mexp_expm), for all three
// families (TaylorNew, TaylorPS, PadeDiagonal). Same signatures, same
// ExpmReport, same exceptions: std::invalid_argument("non-finite matrix
// entry"), ("norm must be finite and nonnegative"); std::runtime_error
// ("singular denominator") from a Pade solve; a CUDA failure or a missing
// device throws std::runtime_error (there is no CPU fallback).
#pragma once

#include <cstdint>

#include "mexp/dense_matrix.hpp"
#include "mexp/theta_tables.hpp"

namespace mexp {

struct Selection {
    int degree = 0;
    int s = 0;
};

Selection select(double norm, const SelectionTable& table);

/// x^(2^s) by s successive squarings on the device, each counted as one product.
DenseMatrix squarings(CostContext& ctx, DenseMatrix x, int s);

struct ExpmReport {
    DenseMatrix result;
    Family family = Family::TaylorNew;
    int degree = 0;
    int s = 0;
    std::int64_t cost_thirds = 0;  // 3 * (products of the scheme + s)
    double norm_in = 0.0;

    double product_cost() const { return double(cost_thirds) / 3.0; }
};

ExpmReport expm(const DenseMatrix& a, Accuracy u, Family family);

}  // namespace mexp
