// comparcc — the #pragma compar pre-compiler (§2.1-2.2).
//
// Source-to-source translation of a C / C++ / CUDA file annotated with
//   #pragma compar method_declare interface(I) target(T) name(F)
//   #pragma compar parameter name(N) type(T) size(S[,S..]) access_mode(M)
//   #pragma compar include | initialize | terminate
// into (1) the host source with the directives translated and the interface call sites rewritten
// to generated entry functions, (2) one glue file per interface (extern declarations of the
// variants, one wrapper per variant, the registration of the variants with the runtime, the entry
// function that builds the task and submits it — Listing 4's structure), (3) a header
// and a common file with compar_pc_init / compar_pc_terminate.  The target runtime is this
// repository's C ABI (include/compar.h, generic interfaces): the selector, calibration and
// history choose among the user's GPU variants per call.  The readings of the paper this tool
// takes are DESIGN.md §7e (R26-R31).
//
//   comparcc FILE [--out DIR] [--emit-ir] [--check]
//     --emit-ir   print the normalized IR as JSON (the same as oracle/precompile.py's run())
//     --check     diagnostics only
//   diagnostics on stderr: <path>:<line>:<col>: <severity>[<code>]: <message>; exit 1 on errors.
#include <algorithm>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <vector>

namespace {

struct Diag {
    std::string severity, code;
    int line, col;
    std::string message;
};

struct Clause {
    std::string key;
    std::vector<std::string> args;
};

struct Directive {
    int line;
    std::string kind;
    std::vector<Clause> clauses;
    const std::vector<std::string> *get(const std::string &k) const {
        for (const auto &c : clauses)
            if (c.key == k) return &c.args;
        return nullptr;
    }
};

struct Param {
    std::string name, type, access;
    std::vector<std::string> size;
};
struct VariantSpec {
    std::string name, target;
    int line;
};
struct Interface {
    std::string name;
    std::vector<Param> params;
    std::vector<VariantSpec> variants;
};
struct Call {
    std::string iface;
    int line;
    std::vector<std::string> args;
    // pieces of the line around the interface name, for the rewrite
    std::string lead, name_rest;
};

const char *const kKinds[] = {"method_declare", "parameter", "include", "initialize", "terminate"};

std::string lower(std::string s) {
    for (auto &ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
    return s;
}
std::string upper(std::string s) {
    for (auto &ch : s) ch = static_cast<char>(std::toupper(static_cast<unsigned char>(ch)));
    return s;
}
bool is_ident_start(char c) { return std::isalpha(static_cast<unsigned char>(c)) || c == '_'; }
bool is_ident(char c) { return std::isalnum(static_cast<unsigned char>(c)) || c == '_'; }

// Length of the "#pragma compar" prefix (with leading blanks) if the line is a directive, else 0.
size_t pragma_prefix(const std::string &ln) {
    size_t i = 0;
    while (i < ln.size() && (ln[i] == ' ' || ln[i] == '\t')) ++i;
    if (ln.compare(i, 7, "#pragma") != 0) return 0;
    i += 7;
    if (i >= ln.size() || (ln[i] != ' ' && ln[i] != '\t')) return 0;
    while (i < ln.size() && (ln[i] == ' ' || ln[i] == '\t')) ++i;
    if (ln.compare(i, 6, "compar") != 0) return 0;
    i += 6;
    if (i < ln.size() && ln[i] != ' ' && ln[i] != '\t') return 0;
    return i;
}

struct Token {
    enum Kind { Ident, Int, Punct } kind;
    std::string text;
};

class Compiler {
public:
    explicit Compiler(std::string path, std::string text) : path_(std::move(path)), text_(std::move(text)) {
        split_lines();
    }

    void run() {
        for (size_t i = 0; i < lines_.size(); ++i)
            if (is_dir_[i]) parse(static_cast<int>(i + 1), lines_[i]);
        analyze();
        find_calls();
        if (!ifaces_.empty()) {
            if (!life_.count("initialize")) add("warning", "no-initialize", 0, 1, "interfaces declared but no initialize");
            if (!life_.count("terminate")) add("warning", "no-terminate", 0, 1, "interfaces declared but no terminate");
        }
        for (const auto &n : order_)
            if (!called_.count(n)) add("warning", "never-called", 0, 1, "interface " + n + " is never called");
        std::stable_sort(diags_.begin(), diags_.end(), [](const Diag &a, const Diag &b) {
            if (a.line != b.line) return a.line < b.line;
            if (a.code != b.code) return a.code < b.code;
            if (a.severity != b.severity) return a.severity < b.severity;
            return a.col < b.col;
        });
    }

    bool has_errors() const {
        for (const auto &d : diags_)
            if (d.severity == "error") return true;
        return false;
    }

    void print_diags(std::FILE *f) const {
        for (const auto &d : diags_)
            std::fprintf(f, "%s:%d:%d: %s[%s]: %s\n", path_.c_str(), d.line, d.col, d.severity.c_str(), d.code.c_str(),
                         d.message.c_str());
    }

    std::string ir_json() const;
    std::string transformed() const;
    std::string header() const;
    std::string common() const;
    std::string glue(const Interface &in) const;
    const std::vector<std::string> &order() const { return order_; }
    const Interface &iface(const std::string &n) const { return ifaces_.at(n); }

private:
    std::string path_, text_;
    std::vector<std::string> lines_;
    std::vector<bool> is_dir_;
    bool trailing_nl_ = false;
    std::vector<Directive> dirs_;
    std::map<std::string, Interface> ifaces_;
    std::vector<std::string> order_;
    std::map<std::string, int> life_;
    std::vector<Call> calls_;
    std::set<std::string> called_;
    std::vector<Diag> diags_;

    void add(const char *sev, const char *code, int line, int col, const std::string &msg) {
        diags_.push_back(Diag{sev, code, line, col, msg});
    }

    void split_lines() {
        std::string cur;
        for (char ch : text_) {
            if (ch == '\n') {
                lines_.push_back(cur);
                cur.clear();
            } else {
                cur.push_back(ch);
            }
        }
        if (!cur.empty()) lines_.push_back(cur);
        trailing_nl_ = !text_.empty() && text_.back() == '\n';
        for (const auto &ln : lines_) is_dir_.push_back(pragma_prefix(ln) != 0);
    }

    // ---------------------------------------------------------------- lexer + parser
    void parse(int lineno, const std::string &ln) {
        std::vector<Token> toks;
        for (size_t p = pragma_prefix(ln); p < ln.size();) {
            const char ch = ln[p];
            if (ch == ' ' || ch == '\t' || ch == '\r') {
                ++p;
            } else if (ch == '(' || ch == ')' || ch == ',') {
                toks.push_back(Token{Token::Punct, std::string(1, ch)});
                ++p;
            } else if (is_ident_start(ch)) {
                size_t q = p;
                while (q < ln.size() && is_ident(ln[q])) ++q;
                toks.push_back(Token{Token::Ident, ln.substr(p, q - p)});
                p = q;
            } else if (std::isdigit(static_cast<unsigned char>(ch))) {
                size_t q = p;
                while (q < ln.size() && std::isdigit(static_cast<unsigned char>(ln[q]))) ++q;
                toks.push_back(Token{Token::Int, ln.substr(p, q - p)});
                p = q;
            } else {
                add("error", "lex", lineno, static_cast<int>(p) + 1, std::string("unexpected character '") + ch + "'");
                return;
            }
        }
        std::string kind = toks.empty() || toks[0].kind != Token::Ident ? "" : lower(toks[0].text);
        if (std::find(std::begin(kKinds), std::end(kKinds), kind) == std::end(kKinds)) {
            add("error", "unknown-directive", lineno, 1, "unknown directive");
            return;
        }
        Directive d{lineno, kind, {}};
        size_t i = 1;
        while (i < toks.size()) {
            if (toks[i].kind != Token::Ident || i + 1 >= toks.size() || toks[i + 1].text != "(") {
                add("error", "syntax", lineno, 1, "expected clause(args)");
                return;
            }
            Clause c{lower(toks[i].text), {}};
            size_t j = i + 2;
            for (;;) {
                if (j >= toks.size() || toks[j].kind == Token::Punct) {
                    add("error", "syntax", lineno, 1, "expected an identifier or integer argument");
                    return;
                }
                c.args.push_back(toks[j].text);
                ++j;
                if (j < toks.size() && toks[j].text == ",") {
                    ++j;
                    continue;
                }
                if (j < toks.size() && toks[j].text == ")") {
                    ++j;
                    break;
                }
                add("error", "syntax", lineno, 1, "expected ',' or ')'");
                return;
            }
            d.clauses.push_back(c);
            i = j;
        }
        std::vector<std::string> allowed, required;
        if (kind == "method_declare") {
            allowed = {"interface", "target", "name"};
            required = allowed;
        } else if (kind == "parameter") {
            allowed = {"name", "type", "size", "access_mode"};
            required = {"name", "type", "access_mode"};
        } else {
            if (!d.clauses.empty()) {
                add("error", "clauses-not-allowed", lineno, 1, kind + " takes no clauses");
                return;
            }
            dirs_.push_back(d);
            return;
        }
        bool ok = true;
        std::set<std::string> seen;
        for (const auto &c : d.clauses) {
            if (std::find(allowed.begin(), allowed.end(), c.key) == allowed.end()) {
                add("error", "unknown-clause", lineno, 1, "clause " + c.key + " not allowed on " + kind);
                ok = false;
                continue;
            }
            if (seen.count(c.key)) {
                add("error", "duplicate-clause", lineno, 1, "duplicate clause " + c.key);
                ok = false;
            }
            seen.insert(c.key);
            const size_t n = c.args.size();
            if (c.key == "size" ? (n < 1 || n > 4) : n != 1) {
                add("error", "clause-arity", lineno, 1, "wrong number of arguments to " + c.key);
                ok = false;
            }
        }
        for (const auto &r : required)
            if (!seen.count(r)) {
                add("error", "missing-clause", lineno, 1, "missing clause " + r);
                ok = false;
            }
        if (ok) dirs_.push_back(d);
    }

    // ---------------------------------------------------------------- semantic analysis
    void analyze() {
        static const std::set<std::string> ok_targets = {"CUDA", "CUBLAS"};
        static const std::set<std::string> known_targets = {"CUDA", "CUBLAS", "OPENMP", "SEQ", "OPENCL", "BLAS"};
        static const std::set<std::string> types = {"int", "float", "double", "char", "wchar_t", "long", "short",
                                                    "unsigned"};
        static const std::set<std::string> access = {"read", "write", "readwrite"};
        std::string open;          // interface whose parameter list is open
        bool redecl = false, after_method = false;
        for (const auto &d : dirs_) {
            if (d.kind == "method_declare") {
                const std::string in = (*d.get("interface"))[0];
                const std::string tg = upper((*d.get("target"))[0]);
                const std::string fn = (*d.get("name"))[0];
                after_method = true;
                if (ifaces_.count(in)) {
                    redecl = true;
                    open.clear();
                } else {
                    ifaces_[in] = Interface{in, {}, {}};
                    order_.push_back(in);
                    redecl = false;
                    open = in;
                }
                Interface &rec = ifaces_[in];
                bool dup = false;
                for (const auto &v : rec.variants) dup = dup || v.name == fn;
                if (!known_targets.count(tg))
                    add("error", "unknown-target", d.line, 1, "unknown target " + tg);
                else if (!ok_targets.count(tg))
                    add("error", "unsupported-target", d.line, 1,
                        "target " + tg + ": this runtime runs GPU variants only (CUDA, CUBLAS)");
                else if (dup)
                    add("error", "duplicate-variant", d.line, 1, "duplicate variant " + fn);
                else
                    rec.variants.push_back(VariantSpec{fn, tg, d.line});
            } else if (d.kind == "parameter") {
                if (!after_method) {
                    add("error", "param-without-method", d.line, 1, "parameter without a preceding method_declare");
                    continue;
                }
                if (redecl) {
                    add("error", "param-redeclared", d.line, 1,
                        "parameters belong to the interface's first method_declare only");
                    continue;
                }
                Interface &rec = ifaces_[open];
                Param p{(*d.get("name"))[0], (*d.get("type"))[0], lower((*d.get("access_mode"))[0]), {}};
                if (const auto *sz = d.get("size")) p.size = *sz;
                bool bad = false;
                for (const auto &q : rec.params)
                    if (q.name == p.name) {
                        add("error", "duplicate-param", d.line, 1, "duplicate parameter " + p.name);
                        bad = true;
                        break;
                    }
                if (!types.count(p.type)) {
                    add("error", "unknown-type", d.line, 1, "unknown type " + p.type);
                    bad = true;
                }
                if (!access.count(p.access)) {
                    add("error", "unknown-access", d.line, 1, "unknown access mode " + p.access);
                    bad = true;
                }
                if (!bad) rec.params.push_back(p);
            } else {
                after_method = false;
                redecl = false;
                open.clear();
                if (!life_.count(d.kind)) life_[d.kind] = d.line;
            }
        }
    }

    // ---------------------------------------------------------------- call sites
    // A passthrough line `<ws>I<ws>(<args>)<ws>;<rest>` with I a declared interface; not a comment.
    void find_calls() {
        for (size_t i = 0; i < lines_.size(); ++i) {
            if (is_dir_[i]) continue;
            const std::string &ln = lines_[i];
            size_t p = 0;
            while (p < ln.size() && (ln[p] == ' ' || ln[p] == '\t')) ++p;
            if (ln.compare(p, 2, "//") == 0) continue;
            if (p >= ln.size() || !is_ident_start(ln[p])) continue;
            size_t q = p;
            while (q < ln.size() && is_ident(ln[q])) ++q;
            const std::string name = ln.substr(p, q - p);
            if (!ifaces_.count(name)) continue;
            size_t r = q;
            while (r < ln.size() && (ln[r] == ' ' || ln[r] == '\t')) ++r;
            if (r >= ln.size() || ln[r] != '(') continue;
            // the LAST ')' followed by blanks and ';' closes the argument list
            size_t close = std::string::npos;
            for (size_t k = ln.size(); k-- > r + 1;) {
                if (ln[k] != ')') continue;
                size_t s = k + 1;
                while (s < ln.size() && (ln[s] == ' ' || ln[s] == '\t')) ++s;
                if (s < ln.size() && ln[s] == ';') {
                    close = k;
                    break;
                }
            }
            if (close == std::string::npos) continue;
            const std::string inner = ln.substr(r + 1, close - r - 1);
            std::vector<std::string> args;
            bool blank = true;
            for (char ch : inner) blank = blank && (ch == ' ' || ch == '\t');
            if (!blank) {
                std::string cur;
                for (char ch : inner) {
                    if (ch == ',') {
                        args.push_back(trim(cur));
                        cur.clear();
                    } else {
                        cur.push_back(ch);
                    }
                }
                args.push_back(trim(cur));
            }
            const int lineno = static_cast<int>(i + 1);
            if (args.size() != ifaces_[name].params.size()) {
                add("warning", "call-arity", lineno, 1, "call of " + name + " with the wrong number of arguments");
                continue;
            }
            calls_.push_back(Call{name, lineno, args, ln.substr(0, p), ln.substr(q)});
            called_.insert(name);
        }
    }

    static std::string trim(const std::string &s) {
        size_t a = 0, b = s.size();
        while (a < b && (s[a] == ' ' || s[a] == '\t')) ++a;
        while (b > a && (s[b - 1] == ' ' || s[b - 1] == '\t')) --b;
        return s.substr(a, b - a);
    }
};

std::string jstr(const std::string &s) {
    std::string o = "\"";
    for (char ch : s) {
        if (ch == '"' || ch == '\\') {
            o.push_back('\\');
            o.push_back(ch);
        } else if (static_cast<unsigned char>(ch) < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof(buf), "\\u%04x", ch);
            o += buf;
        } else {
            o.push_back(ch);
        }
    }
    return o + "\"";
}

std::string jlist(const std::vector<std::string> &v) {
    std::string o = "[";
    for (size_t i = 0; i < v.size(); ++i) o += (i ? ", " : "") + jstr(v[i]);
    return o + "]";
}

std::string Compiler::ir_json() const {
    std::ostringstream o;
    o << "{\"lines\": " << lines_.size() << ", \"directive_lines\": [";
    bool first = true;
    for (size_t i = 0; i < lines_.size(); ++i)
        if (is_dir_[i]) {
            o << (first ? "" : ", ") << i + 1;
            first = false;
        }
    o << "], \"directives\": [";
    for (size_t i = 0; i < dirs_.size(); ++i) {
        const auto &d = dirs_[i];
        o << (i ? ", " : "") << "{\"line\": " << d.line << ", \"kind\": " << jstr(d.kind) << ", \"clauses\": [";
        for (size_t j = 0; j < d.clauses.size(); ++j)
            o << (j ? ", " : "") << "[" << jstr(d.clauses[j].key) << ", " << jlist(d.clauses[j].args) << "]";
        o << "]}";
    }
    o << "], \"interfaces\": [";
    for (size_t i = 0; i < order_.size(); ++i) {
        const auto &in = ifaces_.at(order_[i]);
        o << (i ? ", " : "") << "{\"name\": " << jstr(in.name) << ", \"params\": [";
        for (size_t j = 0; j < in.params.size(); ++j) {
            const auto &p = in.params[j];
            o << (j ? ", " : "") << "{\"name\": " << jstr(p.name) << ", \"type\": " << jstr(p.type)
              << ", \"size\": " << jlist(p.size) << ", \"access\": " << jstr(p.access) << "}";
        }
        o << "], \"variants\": [";
        for (size_t j = 0; j < in.variants.size(); ++j)
            o << (j ? ", " : "") << "{\"name\": " << jstr(in.variants[j].name) << ", \"target\": "
              << jstr(in.variants[j].target) << ", \"line\": " << in.variants[j].line << "}";
        o << "]}";
    }
    o << "], \"lifecycle\": {";
    const char *lk[] = {"include", "initialize", "terminate"};
    for (int i = 0; i < 3; ++i) {
        o << (i ? ", " : "") << jstr(lk[i]) << ": ";
        auto it = life_.find(lk[i]);
        if (it == life_.end())
            o << "null";
        else
            o << it->second;
    }
    o << "}, \"calls\": [";
    for (size_t i = 0; i < calls_.size(); ++i)
        o << (i ? ", " : "") << "{\"iface\": " << jstr(calls_[i].iface) << ", \"line\": " << calls_[i].line
          << ", \"args\": " << jlist(calls_[i].args) << "}";
    o << "], \"diagnostics\": [";
    for (size_t i = 0; i < diags_.size(); ++i)
        o << (i ? ", " : "") << "[" << jstr(diags_[i].severity) << ", " << jstr(diags_[i].code) << ", " << diags_[i].line
          << ", " << diags_[i].col << "]";
    o << "]}";
    return o.str();
}

std::string Compiler::transformed() const {
    std::map<int, const Directive *> by_line;
    for (const auto &d : dirs_) by_line[d.line] = &d;
    std::map<int, const Call *> call_at;
    for (const auto &c : calls_) call_at[c.line] = &c;
    std::string out;
    for (size_t i = 0; i < lines_.size(); ++i) {
        const int no = static_cast<int>(i + 1);
        const std::string &ln = lines_[i];
        std::string line;
        if (by_line.count(no)) {
            size_t w = 0;
            while (w < ln.size() && (ln[w] == ' ' || ln[w] == '\t')) ++w;
            const std::string ws = ln.substr(0, w), &k = by_line[no]->kind;
            if (k == "include") line = ws + "#include \"compar_pc.h\"";
            else if (k == "initialize") line = ws + "compar_pc_init();";
            else if (k == "terminate") line = ws + "compar_pc_terminate();";
        } else if (call_at.count(no)) {
            line = call_at[no]->lead + "compar_submit_" + call_at[no]->iface + call_at[no]->name_rest;
        } else {
            line = ln;
        }
        out += line;
        if (i + 1 < lines_.size() || trailing_nl_) out += "\n";
    }
    return out;
}

// C declarator of an interface parameter: pointer for a parameter with a size clause.
std::string c_param(const Param &p) { return p.type + (p.size.empty() ? " " : " *") + p.name; }

std::string param_list(const Interface &in) {
    std::string s;
    for (size_t i = 0; i < in.params.size(); ++i) s += (i ? ", " : "") + c_param(in.params[i]);
    return s.empty() ? "void" : s;
}

std::string Compiler::header() const {
    std::string o = "/* Generated by comparcc from " + path_ + " (PAPER.md §2.2: glue for each interface). */\n";
    o += "#pragma once\n#include \"compar.h\"\n#ifdef __cplusplus\nextern \"C\" {\n#endif\n";
    o += "void compar_pc_init(void);\nvoid compar_pc_terminate(void);\n";
    for (const auto &n : order_) o += "void compar_submit_" + n + "(" + param_list(ifaces_.at(n)) + ");\n";
    o += "#ifdef __cplusplus\n}\n#endif\n";
    return o;
}

std::string Compiler::common() const {
    std::string o = "/* Generated by comparcc from " + path_ + ": runtime lifecycle (P:89-91). */\n";
    o += "#include <cstdio>\n#include <cstdlib>\n\n#include \"compar_pc.h\"\n\nvoid *compar_pc_ctx = nullptr;\n";
    for (const auto &n : order_) o += "void compar_pc_register_" + n + "(void *ctx);\n";
    o += "\nextern \"C\" void compar_pc_init(void) {\n"
         "    if (compar_init(nullptr, &compar_pc_ctx) != COMPAR_OK) {\n"
         "        std::fprintf(stderr, \"compar_init: %s\\n\", compar_last_error(nullptr));\n"
         "        std::abort();\n    }\n";
    for (const auto &n : order_) o += "    compar_pc_register_" + n + "(compar_pc_ctx);\n";
    o += "}\n\nextern \"C\" void compar_pc_terminate(void) {\n"
         "    compar_sync(compar_pc_ctx, COMPAR_TASK_ALL, nullptr);\n"
         "    compar_terminate(compar_pc_ctx);\n    compar_pc_ctx = nullptr;\n}\n";
    return o;
}

std::string Compiler::glue(const Interface &in) const {
    std::string o = "/* Generated by comparcc from " + path_ + ": interface " + in.name +
                    " (Listing 4 structure: variant declarations, wrappers, registration, task entry). */\n";
    o += "#include <cstdio>\n#include <cstdlib>\n\n#include \"compar_pc.h\"\n\nextern void *compar_pc_ctx;\n\n";
    for (const auto &v : in.variants) o += "void " + v.name + "(" + param_list(in) + ");   /* target " + v.target + " */\n";
    o += "\n";
    for (const auto &v : in.variants) {
        o += "static compar_status compar_wrap_" + in.name + "_" + v.name +
             "(void *const *args, const int64_t *, int, void *) {\n    " + v.name + "(";
        for (size_t i = 0; i < in.params.size(); ++i) {
            const auto &p = in.params[i];
            o += (i ? ", " : "") + std::string("*static_cast<") + p.type + (p.size.empty() ? " *" : " **") +
                 ">(args[" + std::to_string(i) + "])";
        }
        o += ");\n    return COMPAR_OK;\n}\n\n";
    }
    o += "void compar_pc_register_" + in.name + "(void *ctx) {\n    int id = -1;\n";
    for (const auto &v : in.variants)
        o += "    if (compar_register_generic_variant(ctx, \"" + in.name + "\", \"" + v.name + "\", compar_wrap_" +
             in.name + "_" + v.name + ", nullptr, &id) != COMPAR_OK) {\n"
             "        std::fprintf(stderr, \"register " + v.name + ": %s\\n\", compar_last_error(ctx));\n"
             "        std::abort();\n    }\n";
    o += "}\n\n";
    // history key: the distinct size expressions of the array parameters, in order
    std::vector<std::string> sizes;
    for (const auto &p : in.params)
        for (const auto &s : p.size)
            if (std::find(sizes.begin(), sizes.end(), s) == sizes.end()) sizes.push_back(s);
    o += "extern \"C\" void compar_submit_" + in.name + "(" + param_list(in) + ") {\n";
    o += "    void *args[" + std::to_string(std::max<size_t>(1, in.params.size())) + "] = {";
    for (size_t i = 0; i < in.params.size(); ++i) o += (i ? ", " : "") + std::string("&") + in.params[i].name;
    if (in.params.empty()) o += "nullptr";
    o += "};\n    int64_t sizes[" + std::to_string(std::max<size_t>(1, sizes.size())) + "] = {";
    for (size_t i = 0; i < sizes.size(); ++i) o += (i ? ", " : "") + std::string("(int64_t)(") + sizes[i] + ")";
    if (sizes.empty()) o += "0";
    o += "};\n    compar_generic_desc d = {\"" + in.name + "\", " + std::to_string(in.params.size()) + ", args, " +
         std::to_string(sizes.size()) + ", sizes, nullptr, -1};\n"
         "    uint64_t task = 0;\n"
         "    if (compar_generic_submit(compar_pc_ctx, &d, &task) != COMPAR_OK ||\n"
         "        compar_sync(compar_pc_ctx, task, nullptr) != COMPAR_OK) {\n"
         "        std::fprintf(stderr, \"" + in.name + ": %s\\n\", compar_last_error(compar_pc_ctx));\n"
         "        std::abort();\n    }\n}\n";
    return o;
}

bool write_file(const std::string &path, const std::string &s) {
    std::ofstream f(path, std::ios::binary);
    if (!f) return false;
    f << s;
    return static_cast<bool>(f);
}

}  // namespace

int main(int argc, char **argv) {
    std::string in, out = ".";
    bool emit_ir = false, check = false;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        if (a == "--emit-ir") emit_ir = true;
        else if (a == "--check") check = true;
        else if (a == "--out" && i + 1 < argc) out = argv[++i];
        else if (in.empty()) in = a;
        else {
            std::fprintf(stderr, "usage: comparcc FILE [--out DIR] [--emit-ir] [--check]\n");
            return 2;
        }
    }
    if (in.empty()) {
        std::fprintf(stderr, "usage: comparcc FILE [--out DIR] [--emit-ir] [--check]\n");
        return 2;
    }
    std::ifstream f(in, std::ios::binary);
    if (!f) {
        std::fprintf(stderr, "comparcc: cannot read %s\n", in.c_str());
        return 2;
    }
    std::stringstream ss;
    ss << f.rdbuf();
    Compiler c(in, ss.str());
    c.run();
    c.print_diags(stderr);
    if (emit_ir) std::printf("%s\n", c.ir_json().c_str());
    if (c.has_errors()) return 1;
    if (check || emit_ir) return 0;
    std::string stem = in.substr(in.find_last_of('/') == std::string::npos ? 0 : in.find_last_of('/') + 1);
    const size_t dot = stem.find_last_of('.');
    const std::string ext = dot == std::string::npos ? "" : stem.substr(dot);
    if (dot != std::string::npos) stem = stem.substr(0, dot);
    bool ok = write_file(out + "/" + stem + ".compar" + ext, c.transformed()) &&
              write_file(out + "/compar_pc.h", c.header()) && write_file(out + "/compar_pc.gen.cpp", c.common());
    for (const auto &n : c.order()) ok = ok && write_file(out + "/compar_" + n + ".gen.cpp", c.glue(c.iface(n)));
    if (!ok) {
        std::fprintf(stderr, "comparcc: cannot write to %s\n", out.c_str());
        return 2;
    }
    return 0;
}
