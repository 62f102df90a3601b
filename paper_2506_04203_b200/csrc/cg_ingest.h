// Trace ingest: cascade::read_trace_jsonl
// (proj/src/domain.cpp:361-387) on the GPU.  Internal interface between the
// device parser (k_ingest.cu), the host-side error formatter
// (ingest_host.cpp) and the C ABI (engine.cu).
#pragma once

#include <string>
#include <vector>

#include "cg_cuda.h"

namespace cg {

// One decoded trace record (TraceRecord, domain.hpp:96-101).
struct HostRecord {
    double arrival_s = 0, input_tokens = 0;
    std::vector<double> output_tokens, score;
};

// json::parse(line).get<TraceRecord>() exactly as read_trace_jsonl does it.
// Returns true and fills rec, or false with the reference's message
// "<path>:<lineno>: bad trace record: <what>" (domain.cpp:370-377).
bool host_parse_trace_line(const char* p, size_t len, const std::string& path, long long lineno,
                           HostRecord& rec, std::string& msg);
// require_valid(TraceRecord, expected) (domain.cpp:196-209): the reference's
// message, or "" when the record is valid.
std::string host_record_problems(const HostRecord& rec, int expected_stages);

struct IngestBuffers {
    DevBuf bytes, nl, bsum, lrec, status, recline, nst, hostlist, misc;
    DevBuf arrival, in, out, scores;
    HostBuf pinned;
};

struct IngestOut {
    long long n = 0;          // records
    int stages = 0;
    long long lines = 0;
    long long host_lines = 0; // lines the device parser left to the host decoder
    // device columns (IngestBuffers-owned)
    const double* d_arrival = nullptr;
    const double* d_in = nullptr;
    const double* d_out = nullptr;
    const double* d_scores = nullptr;
    double ms_h2d = 0, ms_device = 0, ms_total = 0;
    int launches = 0;
};

// Parses `len` bytes (host memory) of a JSONL trace.  Throws EngineError with
// the reference's Errc/message on invalid input.
void ingest_jsonl(IngestBuffers& B, cudaStream_t s, const char* bytes, long long len, const std::string& path,
                  IngestOut& out);

}  // namespace cg
