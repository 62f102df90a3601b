#include "gpu_engine.hpp"

#include <cstdlib>
#include <mutex>
#include <sstream>
#include <vector>
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
        // CASCADE_PLANNER_GPUS: "all" or a comma-separated device list -> one
        // engine over those GPUs (sharded sweeps, NCCL inside the library);
        // otherwise CASCADE_PLANNER_GPU (default 0) alone.
        cg_status st;
        const char* multi = std::getenv("CASCADE_PLANNER_GPUS");
        if (multi && *multi) {
            std::vector<int32_t> devs;
            if (std::string(multi) != "all") {  // "all": empty list = every visible device
                std::stringstream ss(multi);
                std::string item;
                while (std::getline(ss, item, ',')) devs.push_back(std::atoi(item.c_str()));
            }
            st = cg_engine_create_multi(devs.empty() ? nullptr : devs.data(), static_cast<int32_t>(devs.size()),
                                        &holder.e);
        } else {
            int dev = 0;
            if (const char* s = std::getenv("CASCADE_PLANNER_GPU")) dev = std::atoi(s);
            st = cg_engine_create(dev, &holder.e);
        }
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
