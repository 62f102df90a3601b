// Host half of the trace ingest: decoding of the (rare) lines the device
// parser does not take on, and the reference's error messages.
//
// read_trace_jsonl (proj/src/domain.cpp:361-387) parses each line with
// nlohmann::json::parse + from_json (domain.cpp:299-315); on failure it throws
// invalid_input "<path>:<lineno>: bad trace record: <e.what()>".  The device
// parser (k_ingest.cu) decides which lines are well-formed records; every
// line it cannot decode with certainty comes here, so parse/schema errors
// carry nlohmann's exact exception text.
#include <sstream>

#include "cg_ingest.h"
#include "json.hpp"

namespace cg {

using nlohmann::json;

namespace {
// Local mirror of StageRecord's from_json (domain.cpp:299-302) so that
// get_to(std::vector<...>) raises nlohmann's own exceptions.
struct StageRec {
    double output_tokens = 0, score = 0;
};
void from_json(const json& j, StageRec& v) {
    j.at("output_tokens").get_to(v.output_tokens);
    j.at("score").get_to(v.score);
}
}  // namespace

bool host_parse_trace_line(const char* p, size_t len, const std::string& path, long long lineno,
                           HostRecord& rec, std::string& msg) {
    try {
        const json j = json::parse(std::string(p, len));
        // from_json(TraceRecord) / from_json(StageRecord) order (domain.cpp:299-315)
        HostRecord r;
        j.at("arrival_s").get_to(r.arrival_s);
        j.at("input_tokens").get_to(r.input_tokens);
        std::vector<StageRec> ps;
        j.at("per_stage").get_to(ps);
        for (const StageRec& e : ps) {
            r.output_tokens.push_back(e.output_tokens);
            r.score.push_back(e.score);
        }
        rec = std::move(r);
        return true;
    } catch (const json::exception& e) {
        msg = path + ":" + std::to_string(lineno) + ": bad trace record: " + e.what();
        return false;
    }
}

std::string host_record_problems(const HostRecord& r, int expected_stages) {
    std::vector<std::string> problems;
    if (r.input_tokens < 0) problems.push_back("input_tokens negative");
    if (expected_stages >= 0 && r.score.size() != static_cast<size_t>(expected_stages))
        problems.push_back("per_stage length != C");
    for (size_t i = 0; i < r.score.size(); ++i) {
        if (r.output_tokens[i] < 0) problems.push_back("output_tokens negative");
        if (r.score[i] < 0.0 || r.score[i] > 100.0) problems.push_back("score outside [0,100]");
    }
    if (problems.empty()) return "";
    std::ostringstream m;  // throw_if_any (domain.cpp:40-46)
    m << "invalid TraceRecord:";
    for (const auto& q : problems) m << " " << q << ";";
    return m.str();
}

}  // namespace cg
