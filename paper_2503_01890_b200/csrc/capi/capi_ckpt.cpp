// extern "C" checkpoint entry points of the training executor.
#include <stdexcept>
#include <string>

#include "autohete.h"
#include "../runtime/executor.h"
#include "capi_util.h"

namespace {
template <class F>
int ck_guard(F&& f) {
    try {
        f();
        return AH_OK;
    } catch (const std::invalid_argument& e) {
        return ah::set_error(AH_ERR_INVALID, e.what());
    } catch (const std::exception& e) {
        return ah::set_error(AH_ERR_INTERNAL, e.what());
    }
}
}  // namespace

extern "C" int ah_trainer_save(void* tr, const char* path) {
    if (!tr || !path) return ah::set_error(AH_ERR_INVALID, "ah_trainer_save: null argument");
    return ck_guard([&] { static_cast<ah::Trainer*>(tr)->save(path); });
}

extern "C" int ah_trainer_load(void* tr, const char* path) {
    if (!tr || !path) return ah::set_error(AH_ERR_INVALID, "ah_trainer_load: null argument");
    return ck_guard([&] { static_cast<ah::Trainer*>(tr)->load(path); });
}
