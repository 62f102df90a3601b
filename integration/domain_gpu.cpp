// Reference-side binding: cascade::read_trace_jsonl (proj/include/cascade/
// domain.hpp:162, proj/src/domain.cpp:361-387) on the B200 engine's trace
// ingest (cg_read_trace_jsonl).  Same records (bit-identical doubles), same
// CascadeError codes and messages; the reference's own body is compiled
// alongside under another name (oracle/Makefile `dropin`).
#include <string>
#include <vector>

#include "cascade/domain.hpp"
#include "gpu_engine.hpp"

namespace cascade {

std::vector<TraceRecord> read_trace_jsonl(const std::string& path) {
    cg_trace_buffer* buf = nullptr;
    const cg_status st = cg_read_trace_jsonl(gpu_binding::engine(), path.c_str(), &buf);
    if (st.code != CG_OK) gpu_binding::raise(st);
    const cg_trace& t = buf->host;
    std::vector<TraceRecord> trace(static_cast<size_t>(t.n));
    for (int64_t r = 0; r < t.n; ++r) {
        TraceRecord& rec = trace[static_cast<size_t>(r)];
        rec.arrival_s = t.arrival_s[r];
        rec.input_tokens = t.input_tokens[r];
        rec.per_stage.resize(static_cast<size_t>(t.stages));
        for (int i = 0; i < t.stages; ++i) {
            rec.per_stage[static_cast<size_t>(i)].output_tokens = t.output_tokens[int64_t(i) * t.n + r];
            rec.per_stage[static_cast<size_t>(i)].score = t.scores[int64_t(i) * t.n + r];
        }
    }
    cg_trace_buffer_free(buf);
    return trace;
}

}  // namespace cascade
