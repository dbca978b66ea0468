// Derivation of the per-step AdamW scalars, shared by the GPU and CPU optimizers so both
// consume bit-identical fp32 constants (oracle/adam_oracle.c restates the same recipe).
#pragma once

#include <cmath>
#include <cstdint>

#include "autohete.h"

namespace ah {

struct AdamConsts {
    float decay, beta1, one_minus_beta1, beta2, one_minus_beta2, step_size, inv_sqrt_bc2, eps;
};

inline AdamConsts derive_adam_scalars(const ah_adam_hparams& hp) {
    const double lr = hp.lr, b1 = hp.beta1, b2 = hp.beta2, wd = hp.weight_decay;
    const double t = hp.step < 1 ? 1.0 : static_cast<double>(hp.step);
    AdamConsts c;
    c.decay = static_cast<float>(1.0 - lr * wd);
    c.beta1 = hp.beta1;
    c.one_minus_beta1 = static_cast<float>(1.0 - b1);
    c.beta2 = hp.beta2;
    c.one_minus_beta2 = static_cast<float>(1.0 - b2);
    c.step_size = static_cast<float>(lr / (1.0 - std::pow(b1, t)));
    c.inv_sqrt_bc2 = static_cast<float>(1.0 / std::sqrt(1.0 - std::pow(b2, t)));
    c.eps = hp.eps;
    return c;
}

}  // namespace ah
