"""The #pragma compar pre-compiler, -m "not gpu".

Pins of the oracle (oracle/precompile.py) against SPEC.md's worked examples (S:36-100, S:158-170,
S:222-260) and invariants; then parity of the native tool (comparcc, C++) with the oracle: the same
normalized IR (directives, interfaces, lifecycle, call sites, diagnostics) and byte-identical
translated source, on the golden sample and on hypothesis-generated directive files."""
import json
import os
import re
import subprocess

import pytest

from oracle import precompile as pc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPARCC = os.path.join(ROOT, "paper_2311_03543_b200", "bin", "comparcc")
SAMPLE = os.path.join(ROOT, "tests", "golden", "compar_sample.cu")


def kinds(line):
    toks, bad = pc.tokenize(line)
    assert bad is None
    return [t[1] for t in toks]


# ---------------------------------------------------------------- oracle pins (SPEC examples)
def test_tokenize_spec_examples():
    """the method_declare example is 13 tokens, terminate one.  The parameter example is 17
    tokens (the keyword + 4 clauses x 4 tokens); S:52's "16 tokens" hand count is off by one
    (R31)."""
    assert kinds("#pragma compar method_declare interface(sort) target(CUDA) name(sort_cuda)") == [
        "method_declare", "interface", "(", "sort", ")", "target", "(", "CUDA", ")", "name", "(", "sort_cuda", ")"]
    assert kinds("#pragma compar terminate") == ["terminate"]
    t = kinds("#pragma compar parameter name(arr) type(float) size(N) access_mode(readwrite)")
    assert len(t) == 17 and t[0] == "parameter" and t[-1] == ")"


def test_lex_error_column():
    toks, bad = pc.tokenize("#pragma compar parameter name(a) type(float*) access_mode(read)")
    assert bad == ("*", 44)
    ir = pc.run("#pragma compar parameter name(a) type(float*) access_mode(read)\n")
    assert ir["diagnostics"] == [["error", "lex", 1, 44]]


def test_scan_spec_examples():
    """classification; empty input; a directive needs `#pragma compar` as its first words."""
    assert [d for _, _, d in pc.scan("int x;\n#pragma compar initialize\n")] == [False, True]
    assert pc.scan("") == []
    assert [d for _, _, d in pc.scan("  #pragma compar include\n#pragma omp parallel\n#pragma compare x\n")] == [
        True, False, False]


def test_parse_spec_examples():
    """clause lists, a 2-D size, missing required clauses (two errors, no directive)."""
    ir = pc.run("#pragma compar method_declare interface(sort) target(CUDA) name(sort_cuda)\n")
    assert ir["directives"][0]["clauses"] == [["interface", ["sort"]], ["target", ["CUDA"]], ["name", ["sort_cuda"]]]
    ir = pc.run("#pragma compar parameter name(A) type(float) size(N, M) access_mode(read)\n")
    assert ir["directives"][0]["clauses"][2] == ["size", ["N", "M"]]
    ir = pc.run("#pragma compar method_declare interface(sort)\n")
    assert ir["directives"] == [] and [d[1] for d in ir["diagnostics"]] == ["missing-clause", "missing-clause"]


@pytest.mark.parametrize("line,code", [
    ("#pragma compar method_declare interface(a) interface(b) target(CUDA) name(f)", "duplicate-clause"),
    ("#pragma compar parameter name(x) type(int) size(a,b,c,d,e) access_mode(read)", "clause-arity"),
    ("#pragma compar parameter name(x, y) type(int) access_mode(read)", "clause-arity"),
    ("#pragma compar method_declare interface(a) target(CUDA) name(f) speed(3)", "unknown-clause"),
    ("#pragma compar initialize now(1)", "clauses-not-allowed"),
    ("#pragma compar launch", "unknown-directive"),
    ("#pragma compar method_declare interface(a target(CUDA) name(f)", "syntax"),
    ("#pragma compar method_declare interface() target(CUDA) name(f)", "syntax"),
])
def test_parse_errors(line, code):
    ir = pc.run(line + "\n")
    assert ir["directives"] == [] and code in [d[1] for d in ir["diagnostics"]]


def test_analyze_listing3_sample():
    """the Listing-3-shaped sample gives 2 interfaces (sort: 2 variants / 2 parameters,
    mmul: 2 variants / 4 parameters), both called, no diagnostics; 13 directive lines counted by an
    independent text scan."""
    text = open(SAMPLE).read()
    ir = pc.run(text)
    assert ir["diagnostics"] == []
    assert len(ir["directive_lines"]) == sum(1 for ln in text.splitlines() if ln.strip().startswith("#pragma compar"))
    sort, mmul = ir["interfaces"]
    assert (sort["name"], len(sort["variants"]), [p["name"] for p in sort["params"]]) == ("sort", 2, ["arr", "n"])
    assert sort["params"][0] == {"name": "arr", "type": "float", "size": ["n"], "access": "readwrite"}
    assert sort["params"][1]["size"] == []                      # scalar: no size clause
    assert [v["target"] for v in sort["variants"]] == ["CUDA", "CUDA"]   # targets are case-insensitive
    assert (mmul["name"], len(mmul["variants"]), len(mmul["params"])) == ("mmul", 2, 4)
    assert [c["iface"] for c in ir["calls"]] == ["sort", "mmul"]
    assert ir["lifecycle"] == {"include": 5, "initialize": 22, "terminate": 25}


def test_analyze_rules():
    """empty input; duplicate variant names; parameters only after an interface's first
    method_declare; CPU targets refused by this GPU-only runtime; warnings for a missing lifecycle
    and an uncalled interface."""
    assert pc.run("") == {"lines": 0, "directive_lines": [], "directives": [], "interfaces": [],
                          "lifecycle": {"include": None, "initialize": None, "terminate": None}, "calls": [],
                          "diagnostics": []}
    md = "#pragma compar method_declare interface(s) target(CUDA) name(f)\n"
    codes = [d[1] for d in pc.run(md + md)["diagnostics"]]
    assert codes.count("duplicate-variant") == 1
    p = "#pragma compar parameter name(x) type(int) access_mode(read)\n"
    assert "param-without-method" in [d[1] for d in pc.run(p)["diagnostics"]]
    second = "#pragma compar method_declare interface(s) target(CUDA) name(g)\n"
    assert "param-redeclared" in [d[1] for d in pc.run(md + p + second + p)["diagnostics"]]
    assert "param-without-method" in [d[1] for d in pc.run(md + "#pragma compar include\n" + p)["diagnostics"]]
    omp = "#pragma compar method_declare interface(s) target(OpenMP) name(h)\n"
    assert "unsupported-target" in [d[1] for d in pc.run(omp)["diagnostics"]]
    assert "unknown-target" in [d[1] for d in pc.run(omp.replace("OpenMP", "FPGA"))["diagnostics"]]
    bad = "#pragma compar parameter name(x) type(int8) access_mode(rw)\n"
    codes = [d[1] for d in pc.run(md + bad)["diagnostics"]]
    assert "unknown-type" in codes and "unknown-access" in codes
    w = [d[1] for d in pc.run(md)["diagnostics"] if d[0] == "warning"]
    assert sorted(w) == ["never-called", "no-initialize", "no-terminate"]


def test_call_sites_spec_examples():
    """a call with matching arity; a commented call; an arity mismatch (warning)."""
    decl = ("#pragma compar method_declare interface(sort) target(CUDA) name(f)\n"
            "#pragma compar parameter name(arr) type(float) size(n) access_mode(readwrite)\n"
            "#pragma compar parameter name(n) type(int) access_mode(read)\n")
    ir = pc.run(decl + "sort(arr, n);\n// sort(arr, n);\nsort(arr);\n")
    assert ir["calls"] == [{"iface": "sort", "line": 4, "args": ["arr", "n"]}]
    assert ["warning", "call-arity", 6, 1] in ir["diagnostics"]


def test_transform_rules():
    """lifecycle translation, call rewriting with the trailing comment kept, directives ->
    empty lines, identity on directive-free input; and the backward-compatibility witness: removing
    the directive lines of the input gives its passthrough lines byte-for-byte."""
    assert pc.transform("#pragma compar initialize\n") == "compar_pc_init();\n"
    assert pc.transform("    #pragma compar terminate\n") == "    compar_pc_terminate();\n"
    plain = "int main() {\n  return sort(1);\n}\n"
    assert pc.transform(plain) == plain
    text = open(SAMPLE).read()
    out = pc.transform(text).split("\n")
    assert out[22] == "    compar_submit_sort(arr, n);"
    assert out[23] == "    compar_submit_mmul(A, B, N, M);   // both interfaces are called once"
    assert out[4] == '#include "compar_pc.h"' and out[6] == ""
    assert len(out) == len(text.split("\n"))
    kept = [ln for no, ln, d in pc.scan(text) if not d]
    assert kept == [ln for ln in text.split("\n")[:-1] if not re.match(r"^[ \t]*#pragma[ \t]+compar", ln)]


# ---------------------------------------------------------------- native tool vs oracle
def native(text, tmp_path, name="in.cu"):
    src = tmp_path / name
    src.write_text(text)
    r = subprocess.run([COMPARCC, str(src), "--emit-ir"], capture_output=True, text=True)
    ir = json.loads(r.stdout)
    out_dir = tmp_path / "out"
    out_dir.mkdir(exist_ok=True)
    r2 = subprocess.run([COMPARCC, str(src), "--out", str(out_dir)], capture_output=True, text=True)
    has_err = any(d[0] == "error" for d in ir["diagnostics"])
    assert (r.returncode == 1) == has_err and (r2.returncode == 1) == has_err
    translated = (out_dir / name.replace(".cu", ".compar.cu")).read_text() if not has_err else None
    return ir, translated, r2.stderr


pytestmark_native = pytest.mark.skipif(not os.path.exists(COMPARCC), reason="comparcc not built")


@pytestmark_native
def test_native_matches_oracle_on_sample(tmp_path):
    text = open(SAMPLE).read()
    ir, translated, _ = native(text, tmp_path)
    assert ir == json.loads(json.dumps(pc.run(text)))
    assert translated == pc.transform(text)
    glue = (tmp_path / "out" / "compar_sort.gen.cpp").read_text()
    # Listing 4's structure: V wrappers, V registrations, one submit, one sync
    assert glue.count("static compar_status compar_wrap_sort_") == 2
    assert glue.count("compar_register_generic_variant(") == 2
    assert glue.count("compar_generic_submit(") == 1 and glue.count("compar_sync(") == 1
    assert "int64_t sizes[1] = {(int64_t)(n)}" in glue
    mm = (tmp_path / "out" / "compar_mmul.gen.cpp").read_text()
    assert "int64_t sizes[2] = {(int64_t)(N), (int64_t)(M)}" in mm


@pytestmark_native
def test_native_diagnostic_format(tmp_path):
    _, _, err = native("#pragma compar method_declare interface(s) target(SEQ) name(f)\n", tmp_path)
    assert re.search(r"^.*in\.cu:1:1: error\[unsupported-target\]: ", err, re.M)


hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings, strategies as st  # noqa: E402

IDS = st.sampled_from(["sort", "mmul", "axpy", "A", "B", "n", "N", "M", "f1", "g_2", "arr", "x"])
KW = st.sampled_from(["interface", "target", "name", "type", "size", "access_mode", "speed", "NAME"])
VALS = st.sampled_from(["CUDA", "cuda", "CUBLAS", "OpenMP", "SEQ", "FPGA", "float", "int", "double", "int8", "read",
                        "write", "readwrite", "rw", "3", "64"])


IFACES = ["sort", "mmul", "axpy"]


@st.composite
def directive_line(draw):
    """Mostly well-formed directives (so interfaces, parameters, calls and the translation are
    exercised), with a malformed one now and then."""
    kind = draw(st.sampled_from(["method_declare"] * 3 + ["parameter"] * 4 + ["include", "initialize", "terminate"]))
    if kind == "method_declare":
        clauses = [f"interface({draw(st.sampled_from(IFACES))})",
                   f"target({draw(st.sampled_from(['CUDA', 'CUDA', 'cuda', 'CUBLAS', 'OpenMP', 'FPGA']))})",
                   f"name({draw(st.sampled_from(['f1', 'f2', 'g_2', 'h']))})"]
    elif kind == "parameter":
        clauses = [f"name({draw(st.sampled_from(['arr', 'n', 'A', 'B', 'N', 'M', 'x']))})",
                   f"type({draw(st.sampled_from(['float', 'int', 'double', 'float', 'int8']))})",
                   f"access_mode({draw(st.sampled_from(['read', 'write', 'readwrite', 'READ', 'rw']))})"]
        if draw(st.booleans()):
            dims = draw(st.lists(st.sampled_from(["n", "N", "M", "64"]), min_size=1, max_size=4))
            clauses.insert(2, f"size({', '.join(dims)})")
    else:
        clauses = []
    clauses = draw(st.permutations(clauses))
    m = draw(st.integers(0, 11))
    if m == 0 and clauses:                       # drop a clause
        clauses = clauses[1:]
    elif m == 1 and clauses:                     # duplicate one
        clauses = clauses + [clauses[0]]
    elif m == 2:                                 # unknown clause / kind
        clauses = clauses + [f"{draw(KW)}({draw(VALS)})"]
    elif m == 3:
        kind = draw(st.sampled_from(["launch", "Method_Declare", "PARAMETER"]))
    line = "#pragma compar " + kind + " " + " ".join(clauses)
    if m == 4:                                   # a stray character
        pos = draw(st.integers(0, len(line)))
        line = line[:pos] + draw(st.sampled_from(["*", ";", "[", "=", " ", "\t", ")", "("])) + line[pos:]
    return draw(st.sampled_from(["", "  ", "\t"])) + line


@st.composite
def source(draw):
    lines = []
    for _ in range(draw(st.integers(0, 16))):
        c = draw(st.integers(0, 5))
        if c <= 2:
            lines.append(draw(directive_line()))
        elif c == 3:
            name = draw(st.sampled_from(IFACES + ["x", "printf"]))
            args = draw(st.lists(st.sampled_from(["arr", "n", "A", "B", "N", "M", "1"]), min_size=0, max_size=5))
            lines.append(draw(st.sampled_from(["", "  ", "// ", "\t"])) + f"{name}({', '.join(args)});" +
                         draw(st.sampled_from(["", " // c", "  "])))
        else:
            lines.append(draw(st.sampled_from(["int x = 0;", "", "}", "#pragma omp parallel for", "float *a;"])))
    return "\n".join(lines) + draw(st.sampled_from(["", "\n"]))


@pytestmark_native
@settings(max_examples=300, deadline=None, suppress_health_check=list(HealthCheck))
@given(text=source())
def test_native_matches_oracle_fuzz(tmp_path_factory, text):
    tmp = tmp_path_factory.mktemp("pc")
    ir, translated, _ = native(text, tmp)
    assert ir == json.loads(json.dumps(pc.run(text))), text
    assert translated == pc.transform(text), text
