// hetsim::core drop-in version tag (reference: proj/core/include/hetsim/version.hpp:5).
#pragma once

namespace hetsim {

inline constexpr const char* kVersion = "0.1.0";

}  // namespace hetsim
