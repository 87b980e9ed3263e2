"""Oracle of the #pragma compar pre-compiler front end.  TEST INFRASTRUCTURE
ONLY: imported by tests/ alone; the product tool is paper_2311_03543_b200/csrc/precompiler/comparcc.cpp
and shares no code with this file.

A plain, line-by-line restatement of the directive language of PAPER.md §2.1-2.2:

  #pragma compar method_declare interface(I) target(T) name(F)
  #pragma compar parameter name(N) type(T) size(S[,S..]) access_mode(M)
  #pragma compar include | initialize | terminate

read with the choices listed in DESIGN.md §7e (R26-R31): one directive per physical line;
keywords case-insensitive (stored lower case), targets stored upper case; the runtime has GPU
variants only, so targets other than CUDA / CUBLAS are rejected; `size` takes 1-4 identifiers or
integers; a parameter without `size` is a scalar; parameters attach to the most recent
method_declare and only to an interface's first declaration; lexical diagnostics carry the column
of the offending character, all others column 1.

Output: the normalized IR dictionary `run(text)` returns (the C++ tool's `--emit-ir` prints the
same JSON), and the transformed host source.
Pins: tests/test_precompile.py (SPEC.md worked examples, invariants).
"""
from __future__ import annotations

import re

KINDS = ("method_declare", "parameter", "include", "initialize", "terminate")
CLAUSES = {"method_declare": ("interface", "target", "name"),
           "parameter": ("name", "type", "size", "access_mode")}
REQUIRED = {"method_declare": ("interface", "target", "name"), "parameter": ("name", "type", "access_mode")}
TARGETS_OK = ("CUDA", "CUBLAS")                    # GPU variants: the runtime has no CPU class
TARGETS_KNOWN = ("CUDA", "CUBLAS", "OPENMP", "SEQ", "OPENCL", "BLAS")
TYPES = ("int", "float", "double", "char", "wchar_t", "long", "short", "unsigned")
ACCESS = ("read", "write", "readwrite")
PRAGMA = re.compile(r"^[ \t]*#pragma[ \t]+compar(?=[ \t]|$)")


def scan(text: str):
    """Lines (1-based number, raw text without the newline, is_directive)."""
    out = []
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines = lines[:-1]
    for i, ln in enumerate(lines, 1):
        out.append((i, ln, bool(PRAGMA.match(ln))))
    return out


def tokenize(line: str):
    """Tokens after `#pragma compar` as (kind, text, column); ('error', char, column) on a bad char."""
    m = PRAGMA.match(line)
    pos = m.end()
    toks = []
    while pos < len(line):
        ch = line[pos]
        if ch in " \t\r":
            pos += 1
            continue
        if ch in "(),":
            toks.append(("punct", ch, pos + 1))
            pos += 1
            continue
        mm = re.match(r"[A-Za-z_][A-Za-z0-9_]*", line[pos:])
        if mm:
            toks.append(("ident", mm.group(0), pos + 1))
            pos += len(mm.group(0))
            continue
        mm = re.match(r"[0-9]+", line[pos:])
        if mm:
            toks.append(("int", mm.group(0), pos + 1))
            pos += len(mm.group(0))
            continue
        return toks, (ch, pos + 1)
    return toks, None


def parse_line(lineno: int, line: str, diags: list):
    """One directive -> {'line', 'kind', 'clauses': [[key, [args]]]} or None (diagnostics added)."""
    toks, bad = tokenize(line)
    if bad is not None:
        diags.append(("error", "lex", lineno, bad[1]))
        return None
    if not toks or toks[0][0] != "ident" or toks[0][1].lower() not in KINDS:
        diags.append(("error", "unknown-directive", lineno, 1))
        return None
    kind = toks[0][1].lower()
    clauses = []
    i = 1
    ok = True
    while i < len(toks):
        if toks[i][0] != "ident":
            diags.append(("error", "syntax", lineno, 1))
            return None
        key = toks[i][1].lower()
        if i + 1 >= len(toks) or toks[i + 1][1] != "(":
            diags.append(("error", "syntax", lineno, 1))
            return None
        j = i + 2
        args = []
        while True:
            if j >= len(toks) or toks[j][0] not in ("ident", "int"):
                diags.append(("error", "syntax", lineno, 1))
                return None
            args.append(toks[j][1])
            j += 1
            if j < len(toks) and toks[j][1] == ",":
                j += 1
                continue
            if j < len(toks) and toks[j][1] == ")":
                j += 1
                break
            diags.append(("error", "syntax", lineno, 1))
            return None
        clauses.append([key, args])
        i = j
    if kind not in CLAUSES:
        if clauses:
            diags.append(("error", "clauses-not-allowed", lineno, 1))
            return None
        return {"line": lineno, "kind": kind, "clauses": []}
    seen = set()
    for key, args in clauses:
        if key not in CLAUSES[kind]:
            diags.append(("error", "unknown-clause", lineno, 1))
            ok = False
            continue
        if key in seen:
            diags.append(("error", "duplicate-clause", lineno, 1))
            ok = False
        seen.add(key)
        if (key == "size" and not 1 <= len(args) <= 4) or (key != "size" and len(args) != 1):
            diags.append(("error", "clause-arity", lineno, 1))
            ok = False
    for key in REQUIRED[kind]:
        if key not in seen:
            diags.append(("error", "missing-clause", lineno, 1))
            ok = False
    if not ok:
        return None
    return {"line": lineno, "kind": kind, "clauses": clauses}


def _clause(d, key):
    for k, a in d["clauses"]:
        if k == key:
            return a
    return None


CALL = re.compile(r"^([ \t]*)([A-Za-z_][A-Za-z0-9_]*)([ \t]*\()(.*)(\)[ \t]*;.*)$")


def run(text: str) -> dict:
    """The normalized IR: directives, interfaces, lifecycle, calls, diagnostics (sorted)."""
    diags = []
    lines = scan(text)
    directives = []
    for no, ln, is_dir in lines:
        if is_dir:
            d = parse_line(no, ln, diags)
            if d is not None:
                directives.append(d)
    interfaces = {}                       # name -> {'name', 'params', 'variants'} in declaration order
    order = []
    life = {"include": None, "initialize": None, "terminate": None}
    open_iface = None                     # interface whose parameter list is open
    current_redecl = False                # the last method_declare re-declared an existing interface
    after_method = False
    for d in directives:
        no = d["line"]
        if d["kind"] == "method_declare":
            iface = _clause(d, "interface")[0]
            target = _clause(d, "target")[0].upper()
            fname = _clause(d, "name")[0]
            after_method = True
            if iface in interfaces:
                current_redecl = True
                open_iface = None
            else:
                interfaces[iface] = {"name": iface, "params": [], "variants": []}
                order.append(iface)
                current_redecl = False
                open_iface = iface
            rec = interfaces[iface]
            if target not in TARGETS_KNOWN:
                diags.append(("error", "unknown-target", no, 1))
            elif target not in TARGETS_OK:
                diags.append(("error", "unsupported-target", no, 1))
            elif any(v["name"] == fname for v in rec["variants"]):
                diags.append(("error", "duplicate-variant", no, 1))
            else:
                rec["variants"].append({"name": fname, "target": target, "line": no})
        elif d["kind"] == "parameter":
            if not after_method:
                diags.append(("error", "param-without-method", no, 1))
                continue
            if current_redecl:
                diags.append(("error", "param-redeclared", no, 1))
                continue
            rec = interfaces[open_iface]
            pname = _clause(d, "name")[0]
            ptype = _clause(d, "type")[0]
            acc = _clause(d, "access_mode")[0].lower()
            size = _clause(d, "size") or []
            bad = False
            if any(p["name"] == pname for p in rec["params"]):
                diags.append(("error", "duplicate-param", no, 1))
                bad = True
            if ptype not in TYPES:
                diags.append(("error", "unknown-type", no, 1))
                bad = True
            if acc not in ACCESS:
                diags.append(("error", "unknown-access", no, 1))
                bad = True
            if not bad:
                rec["params"].append({"name": pname, "type": ptype, "size": list(size), "access": acc})
        else:
            after_method = False
            open_iface = None
            current_redecl = False
            if life[d["kind"]] is None:
                life[d["kind"]] = no
    calls = []
    called = set()
    for no, ln, is_dir in lines:
        if is_dir or ln.lstrip(" \t").startswith("//"):
            continue
        m = CALL.match(ln)
        if not m or m.group(2) not in interfaces:
            continue
        rec = interfaces[m.group(2)]
        inner = m.group(4)
        args = [a.strip() for a in inner.split(",")] if inner.strip() else []
        if len(args) != len(rec["params"]):
            diags.append(("warning", "call-arity", no, 1))
            continue
        calls.append({"iface": m.group(2), "line": no, "args": args})
        called.add(m.group(2))
    if order:
        if life["initialize"] is None:
            diags.append(("warning", "no-initialize", 0, 1))
        if life["terminate"] is None:
            diags.append(("warning", "no-terminate", 0, 1))
    for name in order:
        if name not in called:
            diags.append(("warning", "never-called", 0, 1))
    return {"lines": len(lines),
            "directive_lines": [no for no, _, is_dir in lines if is_dir],
            "directives": directives,
            "interfaces": [interfaces[n] for n in order],
            "lifecycle": life,
            "calls": calls,
            "diagnostics": sorted([list(x) for x in diags], key=lambda x: (x[2], x[1], x[0], x[3]))}


def transform(text: str) -> str | None:
    """The translated host source (None if there is an error diagnostic): include -> #include of
    the generated header, initialize / terminate -> compar_pc_init() / compar_pc_terminate(),
    method_declare / parameter lines -> empty lines (line numbers kept), call sites of a
    declared interface -> compar_submit_<interface>(...); every other byte unchanged."""
    ir = run(text)
    if any(d[0] == "error" for d in ir["diagnostics"]):
        return None
    by_line = {d["line"]: d for d in ir["directives"]}
    call_lines = {c["line"] for c in ir["calls"]}
    out = []
    lines = text.split("\n")
    trailing_nl = text.endswith("\n")
    if trailing_nl:
        lines = lines[:-1]
    for i, ln in enumerate(lines, 1):
        if i in by_line:
            ws = ln[:len(ln) - len(ln.lstrip(" \t"))]
            kind = by_line[i]["kind"]
            if kind == "include":
                out.append(ws + '#include "compar_pc.h"')
            elif kind == "initialize":
                out.append(ws + "compar_pc_init();")
            elif kind == "terminate":
                out.append(ws + "compar_pc_terminate();")
            else:
                out.append("")
        elif i in call_lines:
            m = CALL.match(ln)
            out.append(m.group(1) + "compar_submit_" + m.group(2) + m.group(3) + m.group(4) + m.group(5))
        else:
            out.append(ln)
    return "\n".join(out) + ("\n" if trailing_nl else "")
