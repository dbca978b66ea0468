// Launch policy shared by the kernel launchers (kernels.h).
#include <cstdlib>
#include <cstring>

#include "kernels.h"

namespace ah {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("AH_PDL");
        return !(e && std::strcmp(e, "0") == 0);
    }();
    return on;
}

}  // namespace ah
