#include "gpu_engine.hpp"

#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

namespace cascade::gpu_binding {

namespace {
struct EngineHolder {
    cg_engine* e = nullptr;
    ~EngineHolder() {
        if (e) cg_engine_destroy(e);
    }
};
}  // namespace

cg_engine* engine() {
    static EngineHolder holder;
    static std::once_flag once;
    static std::string error;
    std::call_once(once, [] {
        int dev = 0;
        if (const char* s = std::getenv("CASCADE_PLANNER_GPU")) dev = std::atoi(s);
        cg_status st = cg_engine_create(dev, &holder.e);
        if (st.code != CG_OK) error = st.message;
    });
    if (!holder.e) throw std::runtime_error("cascade GPU engine unavailable: " + error);
    return holder.e;
}

void raise(const cg_status& st) {
    if (st.code >= 0 && st.code <= static_cast<int>(Errc::no_feasible_point))
        throw CascadeError(static_cast<Errc>(st.code), st.message);
    throw std::runtime_error(st.message);
}

}  // namespace cascade::gpu_binding
