// Output serialisation on the GPU: the text of
// nlohmann::json(SweepResult).dump(indent) -- sweep.json (cli.cpp:171-172,
// outerplan.cpp:52-59) -- and of json(ParetoFront).dump(indent) (front.json,
// cli.cpp:167-168), byte-identical.
//
// Every evaluation / front point / skipped candidate is an independent text
// segment: one thread per segment measures it (pass 1), the host turns the
// lengths into offsets and writes the few bytes of glue between the arrays,
// one thread per segment writes it (pass 2).  Formatting (json_emit.cuh) is
// nlohmann's serializer: sorted keys, pretty layout, Grisu2 doubles.
#include <cuda_runtime.h>

#include <algorithm>
#include <string>
#include <vector>

#include "cascade_gpu.h"
#include "cg_cuda.h"
#include "cg_json.h"
#include "json_emit.cuh"

namespace cg {

namespace {

using json::Out;
using json::ResultView;

enum : int { SEG_EVAL = 0, SEG_FRONT = 1, SEG_SKIP = 2 };

struct SegArgs {
    ResultView r;
    int step;
    int what;                    // 0 sweep.json, 1 front.json
    long long E, F, S;
    const long long* front;      // [F] evaluation index
    const double* skip_thr;      // [S][C-1]
    const long long* offsets;    // [E+F+S] (pass 2)
    unsigned long long* lengths; // [E+F+S] (pass 1)
    char* text;
};

__device__ void emit_segment(Out& o, const SegArgs& a, long long s) {
    const int st = a.step;
    if (s < a.E) {  // sweep.json: evaluations[] element at 2 steps
        o.spaces(2 * st);
        json::emit_point(o, 2 * st, st, a.r, s);
        o.sep(s + 1 == a.E);
        return;
    }
    s -= a.E;
    if (s < a.F) {  // points[] element: front.points at 3 steps (sweep) / 2 steps (front.json)
        const int ind = (a.what == 0 ? 3 : 2) * st;
        o.spaces(ind);
        json::emit_point(o, ind, st, a.r, a.front[s]);
        o.sep(s + 1 == a.F);
        return;
    }
    s -= a.F;
    const int D = a.r.C - 1;
    o.spaces(2 * st);
    json::emit_thresholds(o, 2 * st, st, a.skip_thr + s * D, D);
    o.sep(s + 1 == a.S);
}

__global__ void k_seg_len(SegArgs a) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= a.E + a.F + a.S) return;
    Out o{nullptr, 0};
    emit_segment(o, a, s);
    a.lengths[s] = (unsigned long long)o.n;
}

__global__ void k_seg_write(SegArgs a) {
    const long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (s >= a.E + a.F + a.S) return;
    Out o{a.text + a.offsets[s], 0};
    emit_segment(o, a, s);
}

template <class T>
T* upload(DevBuf& b, const T* src, size_t count, cudaStream_t s) {
    T* d = b.as<T>(count ? count : 1);
    if (count) CG_CUDA(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
    return d;
}

}  // namespace

std::string result_json(JsonBuffers& B, cudaStream_t s, const cg_sweep_result& r, int step, int what, int flags,
                        int* launches) {
    const int C = r.stages, D = C - 1;
    const long long E = r.num_evaluations, F = r.front_size, S = what == 0 ? r.num_skipped : 0;
    const long long P = r.num_plans, R = r.num_replicas;
    // plans / replicas as SoA on the device
    std::vector<int> pg(P), pd(P), rt(R), rp(R);
    std::vector<long long> po(P);
    for (long long p = 0; p < P; ++p) {
        pg[p] = r.plans[p].gpus_used;
        pd[p] = r.plans[p].dp;
        po[p] = r.plans[p].replica_offset;
    }
    for (long long k = 0; k < R; ++k) {
        rt[k] = r.replicas[k].tp;
        rp[k] = r.replicas[k].pp;
    }
    // evaluation records referenced: the evaluations, and whatever the front
    // indexes (a flattened SweepResult may append its front points after them)
    long long NE = E;
    for (long long k = 0; k < F; ++k) NE = std::max(NE, (long long)r.front[k] + 1);
    SegArgs a{};
    a.r.C = C;
    a.r.compact_ints = (flags & CG_JSON_COMPACT_INT_ARRAYS) ? 1 : 0;
    a.r.thr = upload(B.thr, r.eval_thresholds, (size_t)NE * D, s);
    a.r.lat = upload(B.lat, r.eval_latency, (size_t)NE, s);
    a.r.qual = upload(B.qual, r.eval_quality, (size_t)NE, s);
    a.r.ratios = upload(B.ratios, r.eval_ratios, (size_t)NE * C, s);
    a.r.alloc = upload(B.alloc, r.eval_allocations, (size_t)NE * C, s);
    a.r.eplan = reinterpret_cast<const long long*>(upload(B.eplan, r.eval_plan, (size_t)NE * C, s));
    a.r.plan_gpus = upload(B.pg, pg.data(), (size_t)P, s);
    a.r.plan_dp = upload(B.pd, pd.data(), (size_t)P, s);
    a.r.plan_off = upload(B.po, po.data(), (size_t)P, s);
    a.r.rep_tp = upload(B.rt, rt.data(), (size_t)R, s);
    a.r.rep_pp = upload(B.rp, rp.data(), (size_t)R, s);
    a.step = step;
    a.what = what;
    a.E = what == 0 ? E : 0;
    a.F = F;
    a.S = S;
    a.front = reinterpret_cast<const long long*>(upload(B.front, r.front, (size_t)F, s));
    a.skip_thr = upload(B.skip, r.skipped_thresholds, (size_t)S * D, s);
    const long long nseg = a.E + a.F + a.S;
    std::vector<unsigned long long> len(nseg);
    if (nseg) {
        a.lengths = B.len.as<unsigned long long>((size_t)nseg);
        k_seg_len<<<(unsigned)((nseg + 127) / 128), 128, 0, s>>>(a);
        CG_LAUNCH_CHECK();
        ++*launches;
        CG_CUDA(cudaMemcpyAsync(len.data(), a.lengths, nseg * 8, cudaMemcpyDeviceToHost, s));
        CG_CUDA(cudaStreamSynchronize(s));
    }
    // layout: glue (host) + segments (device) in document order
    const int st = step;
    std::string out;
    std::vector<long long> off(nseg);
    auto spaces = [&](int k) { out.append((size_t)k, ' '); };
    auto put_segments = [&](long long first, long long count) {
        for (long long i = 0; i < count; ++i) {
            off[first + i] = (long long)out.size();
            out.append((size_t)len[first + i], '\0');
        }
    };
    auto host_dbl = [&](double x) {
        char t[64];
        Out h{t, 0};
        h.dbl(x);
        out.append(t, (size_t)h.n);
    };
    auto host_int = [&](long long v) {
        char t[32];
        Out h{t, 0};
        h.i64(v);
        out.append(t, (size_t)h.n);
    };
    if (what == 1) {
        // json(ParetoFront).dump(step): {"points": [...]}
        out += "{\n";
        spaces(st);
        out += "\"points\": ";
        if (F == 0) {
            out += "[]";
        } else {
            out += "[\n";
            put_segments(a.E, F);
            spaces(st);
            out += "]";
        }
        out += "\n}";
    } else {
        out += "{\n";
        spaces(st);
        out += "\"evaluations\": ";
        if (E == 0) out += "[]";
        else {
            out += "[\n";
            put_segments(0, E);
            spaces(st);
            out += "]";
        }
        out += ",\n";
        spaces(st);
        out += "\"front\": {\n";
        spaces(2 * st);
        out += "\"points\": ";
        if (F == 0) out += "[]";
        else {
            out += "[\n";
            put_segments(a.E, F);
            spaces(2 * st);
            out += "]";
        }
        out += "\n";
        spaces(st);
        out += "},\n";
        spaces(st);
        out += "\"skipped\": ";
        if (S == 0) out += "[]";
        else {
            out += "[\n";
            put_segments(a.E + a.F, S);
            spaces(st);
            out += "]";
        }
        out += ",\n";
        spaces(st);
        out += "\"utopia\": {\n";
        spaces(2 * st);
        out += "\"z1_star\": ";
        host_dbl(r.z1_star);
        out += ",\n";
        spaces(2 * st);
        out += "\"z2_star\": ";
        host_dbl(r.z2_star);
        out += "\n";
        spaces(st);
        out += "},\n";
        spaces(st);
        out += "\"weight_selection\": ";
        const int W = r.num_weights;
        if (W == 0) out += "[]";
        else if (a.r.compact_ints) {
            out += "[";
            for (int k = 0; k < W; ++k) {
                if (k) out += ",";
                host_int(r.weight_selection[k]);
            }
            out += "]";
        } else {
            out += "[\n";
            for (int k = 0; k < W; ++k) {
                spaces(2 * st);
                host_int(r.weight_selection[k]);
                out += k + 1 == W ? "\n" : ",\n";
            }
            spaces(st);
            out += "]";
        }
        out += ",\n";
        spaces(st);
        out += "\"weights\": ";
        if (W == 0) out += "[]";
        else {
            out += "[\n";
            for (int k = 0; k < W; ++k) {
                spaces(2 * st);
                out += "{\n";
                spaces(3 * st);
                out += "\"lambda1\": ";
                host_dbl(r.weights[2 * k]);
                out += ",\n";
                spaces(3 * st);
                out += "\"lambda2\": ";
                host_dbl(r.weights[2 * k + 1]);
                out += "\n";
                spaces(2 * st);
                out += k + 1 == W ? "}\n" : "},\n";
            }
            spaces(st);
            out += "]";
        }
        out += "\n}";
    }
    if (nseg) {
        char* text = B.text.as<char>(out.size());
        a.offsets = upload(B.off, off.data(), (size_t)nseg, s);
        a.text = text;
        k_seg_write<<<(unsigned)((nseg + 127) / 128), 128, 0, s>>>(a);
        CG_LAUNCH_CHECK();
        ++*launches;
        // each array's segments are contiguous in the document: copy them
        // straight into place between the host-written glue
        const long long groups[3][2] = {{0, a.E}, {a.E, a.F}, {a.E + a.F, a.S}};
        for (const auto& gr : groups) {
            if (gr[1] == 0) continue;
            const long long b0 = off[gr[0]];
            const long long b1 = off[gr[0] + gr[1] - 1] + (long long)len[gr[0] + gr[1] - 1];
            CG_CUDA(cudaMemcpyAsync(&out[(size_t)b0], text + b0, (size_t)(b1 - b0), cudaMemcpyDeviceToHost, s));
        }
        CG_CUDA(cudaStreamSynchronize(s));
    }
    return out;
}

}  // namespace cg
