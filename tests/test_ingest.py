"""GPU parity tests of the trace ingest:
cg_read_trace_jsonl vs the reference's cascade::read_trace_jsonl
(proj/src/domain.cpp:361-387), run live from oracle/_ref.

Bar: every decoded double bit-identical to the reference reader's; every
error with the same Errc code and the same message text."""
import json
import math
import os
import struct

import numpy as np
import pytest

from parity_util import small_trace
from paper_2506_04203_b200 import engine as eng
from paper_2506_04203_b200 import workloads as W

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def same_trace(a, b):
    for k in ("arrival_s", "input_tokens", "output_tokens", "scores"):
        x, y = np.asarray(a[k], dtype=np.float64), np.asarray(b[k], dtype=np.float64)
        assert x.shape == y.shape, (k, x.shape, y.shape)
        assert np.array_equal(bits(x), bits(y)), k


def ours_vs_ref(engine, path, cap=None):
    from oracle import refpy
    cap = cap or 1 + sum(1 for _ in open(path, "rb"))
    try:
        ref = refpy.read_trace_jsonl(str(path), cap)
        ref_err = None
    except refpy.RefError as e:
        ref, ref_err = None, e
    try:
        got = engine.read_trace_jsonl(str(path))
        got_err = None
    except eng.CascadeError as e:
        got, got_err = None, e
    if ref_err is not None:
        assert got_err is not None, f"reference raised {ref_err.code_name}: {ref_err.message}"
        assert got_err.code == ref_err.code
        assert got_err.message == ref_err.message
        return None
    assert got_err is None, got_err
    same_trace(got, ref)
    return got


@pytest.mark.parametrize("stages,count,hetero", [(2, 5000, False), (3, 20000, True), (4, 3001, False),
                                                 (1, 777, False)])
def test_roundtrip_reference_writer(engine, tmp_path, stages, count, hetero):
    from oracle import refpy
    sc = [(60, 20), (80, 12), (92, 5), (50, 22)][:stages]
    t, _ = small_trace(count, 2.0, sc, seed=stages, hetero=hetero)
    path = tmp_path / "trace.jsonl"
    refpy.write_trace_jsonl(t, str(path))
    got = ours_vs_ref(engine, path)
    same_trace(got, t)
    assert engine.last_ingest["host_lines"] == 0
    assert engine.last_ingest["records"] == count


def test_bursty_concatenated_trace(engine, tmp_path):
    from oracle import refpy
    parts = [eng.generate_trace(s, seed) for s, seed in W.trace_specs("C3", 20000)]
    t = eng.concat_traces(parts)
    path = tmp_path / "c3.jsonl"
    refpy.write_trace_jsonl(t, str(path))
    same_trace(ours_vs_ref(engine, path), t)


def rec_line(arr, inp, stages):
    return json.dumps({"arrival_s": arr, "input_tokens": inp,
                       "per_stage": [{"output_tokens": o, "score": s} for o, s in stages]},
                      separators=(",", ":"))


GOOD = rec_line(1.5, 512.0, [(256.0, 60.25), (128.0, 90.5)])

CASES = {
    "empty_file": "",
    "only_newlines": "\n\n\n",
    "no_trailing_newline": GOOD + "\n" + GOOD.replace("1.5", "2.5"),
    "blank_lines_between": "\n" + GOOD + "\n\n\n" + GOOD.replace("1.5", "3.0") + "\n\n",
    "crlf": GOOD + "\r\n" + GOOD + "\r\n",
    "bom_first_line": "\ufeff" + GOOD + "\n" + GOOD + "\n",
    "whitespace_reordered": ' { "per_stage" : [ { "score" : 60.25 , "output_tokens" : 256 } ,'
                            '{"score":90.5,"output_tokens":128.0}] ,\t"input_tokens":512, "arrival_s": 1.5e0 } \n'
                            + GOOD + "\n",
    "unknown_keys_nested": '{"x":{"a":[1,2,{"b":null}],"c":"s\\u00e9\\n"},"arrival_s":1,"input_tokens":2,'
                           '"per_stage":[{"output_tokens":3,"score":4,"extra":[true,false]}],"z":-0.5e-3}\n'
                           + rec_line(2, 3, [(4, 5)]) + "\n",
    "duplicate_keys_last_wins": '{"arrival_s":9,"arrival_s":1,"input_tokens":2,"per_stage":[{"output_tokens":3,'
                                '"score":4}],"per_stage":[{"output_tokens":5,"score":6}]}\n',
    "integers_and_signs": rec_line(0, 0, [(0, 0)]) + "\n" + '{"arrival_s":-0,"input_tokens":-0.0,'
                          '"per_stage":[{"output_tokens":18446744073709551615,"score":1E+1}]}\n',
    "twenty_digit_integer_overflow": '{"arrival_s":1,"input_tokens":123456789012345678901234,'
                                     '"per_stage":[{"output_tokens":1,"score":1}]}\n',
    "long_mantissa": '{"arrival_s":1.00000000000000000000000000001,"input_tokens":3.141592653589793238462643,'
                     '"per_stage":[{"output_tokens":1,"score":99.99999999999999999999}]}\n',
    "subnormal_and_tiny": '{"arrival_s":4.9e-324,"input_tokens":2.2250738585072011e-308,'
                          '"per_stage":[{"output_tokens":1e-400,"score":0.0}]}\n',
    "utf8_in_unknown_key": '{"\u00e9t\u00e9":"\u4e2d\u6587","arrival_s":1,"input_tokens":2,'
                           '"per_stage":[{"output_tokens":3,"score":4}]}\n',
    # --- errors
    "syntax_truncated": GOOD + "\n" + GOOD[:-3] + "\n",
    "syntax_trailing_comma": '{"arrival_s":1,"input_tokens":2,"per_stage":[],}\n',
    "syntax_leading_zero": '{"arrival_s":01,"input_tokens":2,"per_stage":[]}\n',
    "syntax_trailing_garbage": GOOD + " x\n",
    "syntax_bare_word": "hello\n",
    "syntax_unterminated_string": '{"arrival_s\n',
    "syntax_bad_escape": '{"a":"\\q","arrival_s":1,"input_tokens":2,"per_stage":[]}\n',
    "syntax_lone_surrogate": '{"a":"\\udc00","arrival_s":1,"input_tokens":2,"per_stage":[]}\n',
    "syntax_invalid_utf8": b'{"a":"\xff","arrival_s":1,"input_tokens":2,"per_stage":[]}\n',
    "number_overflow": '{"arrival_s":1e400,"input_tokens":2,"per_stage":[]}\n',
    "schema_missing_key": '{"arrival_s":1,"per_stage":[]}\n',
    "schema_wrong_type": '{"arrival_s":"1","input_tokens":2,"per_stage":[]}\n',
    "schema_per_stage_object": '{"arrival_s":1,"input_tokens":2,"per_stage":{}}\n',
    "schema_stage_missing_score": '{"arrival_s":1,"input_tokens":2,"per_stage":[{"output_tokens":1}]}\n',
    "schema_bool_number": '{"arrival_s":true,"input_tokens":2,"per_stage":[]}\n',
    "schema_empty_object": "{}\n",
    "schema_array_line": "[1,2]\n",
    "invalid_negative_input": GOOD + "\n" + rec_line(2, -1, [(1, 50), (1, 50)]) + "\n",
    "invalid_score_range": GOOD + "\n" + rec_line(2, 1, [(1, 100.5), (-2, -0.5)]) + "\n",
    "invalid_stage_count": GOOD + "\n" + rec_line(2, 1, [(1, 50)]) + "\n",
    "invalid_first_record": rec_line(1, -5, [(-1, 200)]) + "\n" + GOOD + "\n",
    "order_violation": GOOD.replace("1.5", "5") + "\n" + GOOD.replace("1.5", "7") + "\n" + GOOD + "\n",
    "order_and_invalid_same_line": GOOD.replace("1.5", "5") + "\n" + rec_line(1, -1, [(1, 1), (1, 1)]) + "\n",
    "error_after_host_line": '{"\u00e9":1,"arrival_s":1,"input_tokens":2,"per_stage":[{"output_tokens":3,"score":4}]}\n'
                             + rec_line(0.5, 1, [(1, 1)]) + "\n",
    "zero_stage_records": rec_line(1, 2, []) + "\n" + rec_line(2, 3, []) + "\n",
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_reader_cases_match_reference(engine, tmp_path, name):
    data = CASES[name]
    path = tmp_path / f"{name}.jsonl"
    path.write_bytes(data if isinstance(data, bytes) else data.encode())
    ours_vs_ref(engine, path, cap=64)


def test_missing_file(engine, tmp_path):
    ours_vs_ref(engine, tmp_path / "does_not_exist.jsonl", cap=4)


def test_unsorted_fixture_like_reference_artefact(engine, tmp_path):
    """Like proj/cascade_test_tmp/domain/trace.jsonl (test_domain.cpp:239-242):
    the reference writer's output with the first and last arrivals swapped."""
    from oracle import refpy
    t, _ = small_trace(50, 0.5, ((50, 30), (50, 30), (50, 30)), seed=9)
    t = {k: np.array(v, copy=True) for k, v in t.items()}
    t["arrival_s"][0], t["arrival_s"][-1] = t["arrival_s"][-1], t["arrival_s"][0]
    path = tmp_path / "trace.jsonl"
    refpy.write_trace_jsonl(t, str(path))
    ours_vs_ref(engine, path)


def test_number_conversion_exact(engine, tmp_path):
    """Decimal -> binary64 on the device: shortest repr, %.17g and random
    precisions over the whole exponent range equal strtod (Python float) and
    the reference reader, bit for bit."""
    rng = np.random.default_rng(2026)
    n = 60000
    mant = rng.random(n) + 0.5
    expo = rng.integers(-330, 300, n)
    vals = np.sort(np.abs(mant * np.power(10.0, expo.astype(np.float64))))
    vals = vals[np.isfinite(vals) & (vals > 0)]
    fmts = []
    for i, v in enumerate(vals):
        k = i % 4
        if k == 0:
            s = repr(float(v))
        elif k == 1:
            s = "%.17g" % v
        elif k == 2:
            s = "%.*e" % (int(rng.integers(0, 19)), v)
        else:
            s = "%.*f" % (int(rng.integers(0, 12)), v) if v < 1e15 else repr(float(v))
        fmts.append(s)
    dec = np.array([float(s) for s in fmts])
    order = np.argsort(dec, kind="stable")
    lines = [f'{{"arrival_s":{fmts[i]},"input_tokens":{fmts[i]},"per_stage":[{{"output_tokens":{fmts[i]},"score":1}}]}}'
             for i in order]
    path = tmp_path / "numbers.jsonl"
    path.write_text("\n".join(lines) + "\n")
    got = ours_vs_ref(engine, path)
    assert np.array_equal(bits(got["arrival_s"]), bits(dec[order]))
    assert engine.last_ingest["host_lines"] <= len(lines) // 1000 + 1


def test_ingest_feeds_sweep_on_device(engine, tmp_path):
    """The device columns of an ingest drive cg_sweep directly: same result as
    the reference sweep on the reference reader's trace."""
    from oracle import refpy
    from parity_util import diff_json
    t, _ = small_trace(3000, 1.0, ((60, 20), (92, 5)), seed=1)
    cfg, _ = W.planner_config("C1", t["scores"], grid=8)
    path = tmp_path / "trace.jsonl"
    refpy.write_trace_jsonl(t, str(path))
    tb = engine.ingest_to_device(str(path))
    got = engine.sweep(tb, cfg["models"], cfg["hardware"], cfg["cost_model"], 16, cfg["sweep"])
    ref = refpy.sweep(refpy.read_trace_jsonl(str(path), 3001), cfg, 16)["result"]
    assert not diff_json(got, ref)
