// executor.cpp — the host equation executor: Case::solve_step on the device (§8(b) "Caller").
//
// The reference solves a deck equation by equation (src/case.cpp:9-67): lazy cell
// rebuild, reductions frozen once per equation (sfl/ast.cpp:237-274), the RHS tree
// evaluated per particle into staging, a NaN audit naming the lowest bad particle,
// the swap, and a boundary shift after every write of r. This file runs that loop
// over the C-ABI: an equation's text ("lhs=rhs", the reference's canonical
// Equation::to_text form) is parsed once with the reference's grammar
// (sfl/parser.cpp:40-110, lexer.cpp), then every solve lowers the tree:
//
//   uniform subtrees (constants, variables, literals, frozen reductions)
//       -> folded on the host with the reference's Tensor rules (tensor.cpp:11-110),
//          compiled without FMA contraction and with the host libm: the same values
//          the reference computes per particle;
//   InteractionNode  -> nau_interact into a temporary field; operand subtrees are
//          materialised once per equation (a field, a uniform value, or a nau_eval
//          program into a temporary) — the reference re-evaluates them at every
//          neighbour j, which gives the same values for every deterministic operand;
//   ReductionNode    -> the argument materialised, nau_reduce, combined over ranks
//          with nau_allreduce (SURVEY.md §8(e) "Reductions");
//   everything else  -> one nau_eval register program (BinaryNode, UnaryMinusNode,
//          VectorJoinNode, builtins, euler, rand) writing the LHS field two-phase
//          with the NaN audit; r written => boundary shift + dirty cells (vm.cu).
//
// A variable LHS is evaluated at particle 0, as case.cpp:19-29 does.
// Errors carry the reference's kinds and messages, prefixed "equation '<name>': ".
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "nauticle_gpu.h"

namespace {

// ---- uniform tensors (≤ 3x3, column-major like the reference's Eigen storage) ----
struct Tn {
    int r = 1, c = 1;
    double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    bool scalar() const { return r == 1 && c == 1; }
    int size() const { return r * c; }
    double& at(int row, int col) { return v[col * r + row]; }
    double at(int row, int col) const { return v[col * r + row]; }
};

Tn scalar_tn(double x) {
    Tn t;
    t.v[0] = x;
    return t;
}

struct ExecError {
    nau_status st;
    std::string msg;
    long bad = -1;
};

[[noreturn]] void fail_rt(const std::string& m, nau_status st = NAU_ERR_RUNTIME) {
    throw ExecError{st, m};
}

std::string shape_str(int r, int c) { return std::to_string(r) + "x" + std::to_string(c); }
std::string shape_str(const Tn& t) { return shape_str(t.r, t.c); }

// format.hpp:12-16 format_double: shortest round-trip decimal.
std::string fmt(double v) {
    char buf[32];
    auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

[[noreturn]] void shape_mismatch(const char* op, int ar, int ac, int br, int bc) {
    fail_rt(std::string("operator '") + op + "': incompatible shapes " + shape_str(ar, ac) + " and " +
            shape_str(br, bc));
}

// tensor.cpp:43-110 on uniform values
Tn t_add(const Tn& a, const Tn& b, bool sub) {
    if (a.r != b.r || a.c != b.c) shape_mismatch(sub ? "-" : "+", a.r, a.c, b.r, b.c);
    Tn o = a;
    for (int k = 0; k < a.size(); ++k) o.v[k] = sub ? a.v[k] - b.v[k] : a.v[k] + b.v[k];
    return o;
}

Tn t_mul(const Tn& a, const Tn& b) {
    if (a.scalar()) {
        Tn o = b;
        for (int k = 0; k < b.size(); ++k) o.v[k] = a.v[0] * b.v[k];
        return o;
    }
    if (b.scalar()) {
        Tn o = a;
        for (int k = 0; k < a.size(); ++k) o.v[k] = b.v[0] * a.v[k];
        return o;
    }
    if (a.c != b.r) shape_mismatch("*", a.r, a.c, b.r, b.c);
    Tn o;
    o.r = a.r;
    o.c = b.c;
    for (int i = 0; i < a.r; ++i)
        for (int j = 0; j < b.c; ++j) {
            double s = a.at(i, 0) * b.at(0, j);
            for (int q = 1; q < a.c; ++q) s = s + a.at(i, q) * b.at(q, j);
            o.at(i, j) = s;
        }
    return o;
}

Tn t_div(const Tn& a, const Tn& b) {
    Tn o = a;
    if (b.scalar()) {
        for (int k = 0; k < a.size(); ++k) o.v[k] = a.v[k] / b.v[0];
        return o;
    }
    if (a.r != b.r || a.c != b.c) shape_mismatch("/", a.r, a.c, b.r, b.c);
    for (int k = 0; k < a.size(); ++k) o.v[k] = a.v[k] / b.v[k];
    return o;
}

template <class F>
Tn t_elem2(const char* name, const Tn& a, const Tn& b, F fn) {
    if (a.scalar() && !b.scalar()) {
        Tn o = b;
        for (int k = 0; k < b.size(); ++k) o.v[k] = fn(a.v[0], b.v[k]);
        return o;
    }
    if (b.scalar() && !a.scalar()) {
        Tn o = a;
        for (int k = 0; k < a.size(); ++k) o.v[k] = fn(a.v[k], b.v[0]);
        return o;
    }
    if (a.r != b.r || a.c != b.c) shape_mismatch(name, a.r, a.c, b.r, b.c);
    Tn o = a;
    for (int k = 0; k < a.size(); ++k) o.v[k] = fn(a.v[k], b.v[k]);
    return o;
}

template <class F>
Tn t_elem1(const Tn& a, F fn) {
    Tn o = a;
    for (int k = 0; k < a.size(); ++k) o.v[k] = fn(a.v[k]);
    return o;
}

// ---- lexer (sfl/lexer.cpp) ----
enum class Tk {
    Ident, Number, Plus, Minus, Star, Slash, Caret, Assign, LParen, RParen, Comma, Pipe,
    Less, Greater, LessEq, GreaterEq, EqEq, NotEq, End
};

const char* tk_name(Tk k) {  // lexer.cpp token_kind_name
    switch (k) {
        case Tk::Ident: return "identifier";
        case Tk::Number: return "number";
        case Tk::Plus: return "'+'";
        case Tk::Minus: return "'-'";
        case Tk::Star: return "'*'";
        case Tk::Slash: return "'/'";
        case Tk::Caret: return "'^'";
        case Tk::Assign: return "'='";
        case Tk::LParen: return "'('";
        case Tk::RParen: return "')'";
        case Tk::Comma: return "','";
        case Tk::Pipe: return "'|'";
        case Tk::Less: return "'<'";
        case Tk::Greater: return "'>'";
        case Tk::LessEq: return "'<='";
        case Tk::GreaterEq: return "'>='";
        case Tk::EqEq: return "'=='";
        case Tk::NotEq: return "'!='";
        case Tk::End: return "end of expression";
    }
    return "?";
}

struct Tok {
    Tk k;
    std::string text;
    double num = 0.0;
    int col = 0;
};

[[noreturn]] void parse_err(const std::string& m) { fail_rt(m, NAU_ERR_ARG); }

std::vector<Tok> tokenize(const std::string& s) {
    std::vector<Tok> out;
    const size_t n = s.size();
    size_t p = 0;
    auto is_alpha = [](char ch) { return (ch >= 'a' && ch <= 'z') || (ch >= 'A' && ch <= 'Z'); };
    auto is_digit = [](char ch) { return ch >= '0' && ch <= '9'; };
    while (p < n) {
        const char ch = s[p];
        if (ch == ' ' || ch == '\t' || ch == '\n' || ch == '\r' || ch == '\f' || ch == '\v') {
            ++p;
            continue;
        }
        const int col = (int)p + 1;
        if (is_alpha(ch) || ch == '_') {
            size_t b = p;
            while (p < n && (is_alpha(s[p]) || is_digit(s[p]) || s[p] == '_')) ++p;
            out.push_back({Tk::Ident, s.substr(b, p - b), 0.0, col});
            continue;
        }
        if (is_digit(ch) || (ch == '.' && p + 1 < n && is_digit(s[p + 1]))) {
            size_t b = p;
            while (p < n && is_digit(s[p])) ++p;
            if (p < n && s[p] == '.') {
                ++p;
                while (p < n && is_digit(s[p])) ++p;
            }
            if (p < n && (s[p] == 'e' || s[p] == 'E')) {
                size_t mark = p++;
                if (p < n && (s[p] == '+' || s[p] == '-')) ++p;
                if (p < n && is_digit(s[p]))
                    while (p < n && is_digit(s[p])) ++p;
                else
                    p = mark;
            }
            Tok t{Tk::Number, s.substr(b, p - b), 0.0, col};
            auto res = std::from_chars(s.data() + b, s.data() + p, t.num);
            if (res.ec != std::errc())
                parse_err("bad numeric literal '" + t.text + "' at column " + std::to_string(col));
            out.push_back(t);
            continue;
        }
        auto two = [&](char a, char b) { return ch == a && p + 1 < n && s[p + 1] == b; };
        Tk k;
        int len = 1;
        if (two('<', '=')) k = Tk::LessEq, len = 2;
        else if (two('>', '=')) k = Tk::GreaterEq, len = 2;
        else if (two('=', '=')) k = Tk::EqEq, len = 2;
        else if (two('!', '=')) k = Tk::NotEq, len = 2;
        else {
            switch (ch) {
                case '+': k = Tk::Plus; break;
                case '-': k = Tk::Minus; break;
                case '*': k = Tk::Star; break;
                case '/': k = Tk::Slash; break;
                case '^': k = Tk::Caret; break;
                case '=': k = Tk::Assign; break;
                case '(': k = Tk::LParen; break;
                case ')': k = Tk::RParen; break;
                case ',': k = Tk::Comma; break;
                case '|': k = Tk::Pipe; break;
                case '<': k = Tk::Less; break;
                case '>': k = Tk::Greater; break;
                default:
                    parse_err(std::string("unexpected character '") + ch + "' at column " +
                              std::to_string(col));
            }
        }
        out.push_back({k, s.substr(p, len), 0.0, col});
        p += len;
    }
    out.push_back({Tk::End, "", 0.0, (int)n + 1});
    return out;
}

// ---- expression tree ----
enum class K { Lit, Const, Var, Field, Kernel, Bin, Neg, Join, Call1, Call2, Euler, Rand, Red, Inter };
enum BinOp { B_ADD, B_SUB, B_MUL, B_DIV, B_POW, B_LT, B_GT, B_LE, B_GE, B_EQ, B_NE };
enum RedKind { R_MAX = 0, R_MIN = 1, R_SUM = 2, R_MEAN = 3 };

struct Node {
    K k;
    int op = 0;         // BinOp, builtin VM opcode, RedKind, interaction op
    std::string name;   // symbol / function / keyword text
    Tn lit;             // literal
    int sym = -1;       // constant / variable index, field id
    int kf = 0, kd = 0;  // kernel keyword: family, dimension
    nau_op_info info{};
    std::vector<std::unique_ptr<Node>> a;
    // per-solve state
    Tn red;             // frozen reduction value
    int temp = -1;      // materialised interaction result (field id)
    bool uniform = false;
};
using NodeP = std::unique_ptr<Node>;

constexpr int kPrecPipe = 1, kPrecCompare = 2, kPrecAdd = 3, kPrecMul = 4, kPrecUnary = 5,
              kPrecPow = 6, kPrecPrimary = 7;

struct OpInfo {
    const char* sym;
    int prec;
    bool right;
};

OpInfo bin_info(int op) {  // ast.cpp op_info
    switch (op) {
        case B_ADD: return {"+", kPrecAdd, false};
        case B_SUB: return {"-", kPrecAdd, false};
        case B_MUL: return {"*", kPrecMul, false};
        case B_DIV: return {"/", kPrecMul, false};
        case B_POW: return {"^", kPrecPow, true};
        case B_LT: return {"<", kPrecCompare, false};
        case B_GT: return {">", kPrecCompare, false};
        case B_LE: return {"<=", kPrecCompare, false};
        case B_GE: return {">=", kPrecCompare, false};
        case B_EQ: return {"==", kPrecCompare, false};
        default: return {"!=", kPrecCompare, false};
    }
}

// ast.cpp print(): precedence-aware canonical text, for the " in '...'" suffixes.
void print(const Node& n, std::string& os, int min_prec) {
    auto wrap = [&](int own, auto&& body) {
        const bool par = own < min_prec;
        if (par) os += '(';
        body();
        if (par) os += ')';
    };
    switch (n.k) {
        case K::Lit:
            wrap(n.lit.v[0] < 0 ? kPrecUnary : kPrecPrimary, [&] { os += fmt(n.lit.v[0]); });
            break;
        case K::Const:
        case K::Var:
        case K::Field:
        case K::Kernel: os += n.name; break;
        case K::Bin: {
            const OpInfo in = bin_info(n.op);
            wrap(in.prec, [&] {
                print(*n.a[0], os, in.prec + (in.right ? 1 : 0));
                os += in.sym;
                print(*n.a[1], os, in.prec + (in.right ? 0 : 1));
            });
            break;
        }
        case K::Neg:
            wrap(kPrecUnary, [&] {
                os += '-';
                print(*n.a[0], os, kPrecUnary + 1);
            });
            break;
        case K::Join:
            wrap(kPrecPipe, [&] {
                print(*n.a[0], os, kPrecPipe);
                os += '|';
                print(*n.a[1], os, kPrecPipe + 1);
            });
            break;
        default:
            os += n.name;
            os += '(';
            for (size_t q = 0; q < n.a.size(); ++q) {
                if (q) os += ',';
                print(*n.a[q], os, 0);
            }
            os += ')';
            break;
    }
}

std::string text_of(const Node& n) {
    std::string s;
    print(n, s, 0);
    return s;
}

struct Symbols;  // the case's symbol table (below)

struct UnaryFn {
    const char* name;
    int op;
};
constexpr UnaryFn kUnary[] = {{"exp", NAU_VM_EXP},   {"log", NAU_VM_LOG},     {"sin", NAU_VM_SIN},
                              {"cos", NAU_VM_COS},   {"tan", NAU_VM_TAN},     {"sqrt", NAU_VM_SQRT},
                              {"abs", NAU_VM_ABS},   {"floor", NAU_VM_FLOOR}, {"sgn", NAU_VM_SGN},
                              {"norm", NAU_VM_NORM}};
constexpr UnaryFn kBinary[] = {{"min", NAU_VM_MIN}, {"max", NAU_VM_MAX}, {"dot", NAU_VM_DOT}};

}  // namespace

// ---- the case ----
struct nau_case {
    nau_ctx* ctx = nullptr;
    struct Sym {
        std::string name;
        Tn value;
    };
    std::vector<Sym> constants, variables;
    std::map<std::string, int> fields;  // name -> field id
    struct Equation {
        std::string name, lhs;
        int lhs_field = -1, lhs_var = -1;
        NodeP rhs;
    };
    std::vector<Equation> equations;
    struct Temp {
        int id, rows, cols;
        bool busy;
    };
    std::vector<Temp> temps;
    std::string last_error;
    long last_bad = -1;
    int dim = 0;
    long steps = 0;
};

namespace {

int find_sym(const std::vector<nau_case::Sym>& v, const std::string& name) {
    for (size_t k = 0; k < v.size(); ++k)
        if (v[k].name == name) return (int)k;
    return -1;
}

bool is_kernel_keyword(const std::string& s) {
    int f = 0, d = 0;
    return s.size() == 7 && s[0] == 'W' && nau_decode_kernel(s.c_str(), &f, &d) == NAU_OK;
}

// sfl/parser.cpp
class Parser {
public:
    Parser(const std::string& src, nau_case& cs) : t_(tokenize(src)), cs_(cs) {}

    NodeP full() {
        NodeP n = vec();
        if (peek().k != Tk::End)
            parse_err(std::string("unexpected ") + tk_name(peek().k) + " at column " +
                      std::to_string(peek().col));
        return n;
    }

private:
    const Tok& peek() const { return t_[p_]; }
    const Tok& adv() { return t_[p_++]; }
    bool accept(Tk k) {
        if (peek().k != k) return false;
        ++p_;
        return true;
    }
    void expect(Tk k, const char* ctx) {
        if (!accept(k))
            parse_err(std::string("expected ") + tk_name(k) + " " + ctx + " at column " +
                      std::to_string(peek().col) + ", got " + tk_name(peek().k));
    }
    static NodeP mk(K k, int op = 0) {
        auto n = std::make_unique<Node>();
        n->k = k;
        n->op = op;
        return n;
    }
    static NodeP bin(int op, NodeP l, NodeP r) {
        NodeP n = mk(K::Bin, op);
        n->a.push_back(std::move(l));
        n->a.push_back(std::move(r));
        return n;
    }
    NodeP vec() {
        NodeP n = cmp();
        while (accept(Tk::Pipe)) {
            NodeP j = mk(K::Join);
            j->a.push_back(std::move(n));
            j->a.push_back(cmp());
            n = std::move(j);
        }
        return n;
    }
    NodeP cmp() {
        NodeP n = add();
        for (;;) {
            int op;
            switch (peek().k) {
                case Tk::Less: op = B_LT; break;
                case Tk::Greater: op = B_GT; break;
                case Tk::LessEq: op = B_LE; break;
                case Tk::GreaterEq: op = B_GE; break;
                case Tk::EqEq: op = B_EQ; break;
                case Tk::NotEq: op = B_NE; break;
                default: return n;
            }
            adv();
            n = bin(op, std::move(n), add());
        }
    }
    NodeP add() {
        NodeP n = mul();
        for (;;) {
            if (accept(Tk::Plus)) n = bin(B_ADD, std::move(n), mul());
            else if (accept(Tk::Minus)) n = bin(B_SUB, std::move(n), mul());
            else return n;
        }
    }
    NodeP mul() {
        NodeP n = unary();
        for (;;) {
            if (accept(Tk::Star)) n = bin(B_MUL, std::move(n), unary());
            else if (accept(Tk::Slash)) n = bin(B_DIV, std::move(n), unary());
            else return n;
        }
    }
    // parser.cpp: unary minus binds looser than '^'; a negated literal folds
    NodeP unary() {
        if (accept(Tk::Minus)) {
            NodeP o = unary();
            if (o->k == K::Lit) {
                for (int q = 0; q < o->lit.size(); ++q) o->lit.v[q] = -o->lit.v[q];
                return o;
            }
            NodeP n = mk(K::Neg);
            n->a.push_back(std::move(o));
            return n;
        }
        return power();
    }
    NodeP power() {
        NodeP n = primary();
        if (accept(Tk::Caret)) return bin(B_POW, std::move(n), unary());
        return n;
    }
    NodeP primary() {
        const Tok& t = peek();
        switch (t.k) {
            case Tk::Number: {
                adv();
                NodeP n = mk(K::Lit);
                n->lit = scalar_tn(t.num);
                return n;
            }
            case Tk::LParen: {
                adv();
                NodeP n = vec();
                expect(Tk::RParen, "to close '('");
                return n;
            }
            case Tk::Ident: {
                const Tok& id = adv();
                if (peek().k == Tk::LParen) return call(id);
                return symbol(id);
            }
            default:
                parse_err("expected a value at column " + std::to_string(t.col) + ", got " +
                          tk_name(t.k));
        }
    }
    NodeP symbol(const Tok& t) {
        NodeP n;
        int k;
        if (is_kernel_keyword(t.text)) {
            n = mk(K::Kernel);
            nau_decode_kernel(t.text.c_str(), &n->kf, &n->kd);
        } else if ((k = find_sym(cs_.constants, t.text)) >= 0) {
            n = mk(K::Const);
            n->sym = k;
        } else if ((k = find_sym(cs_.variables, t.text)) >= 0) {
            n = mk(K::Var);
            n->sym = k;
        } else if (cs_.fields.count(t.text)) {
            n = mk(K::Field);
            n->sym = cs_.fields[t.text];
        } else {
            parse_err("unknown symbol '" + t.text + "'");
        }
        n->name = t.text;
        return n;
    }
    void arity(const Tok& nm, const std::vector<NodeP>& args, int lo, int hi) {
        const int n = (int)args.size();
        if (n >= lo && n <= hi) return;
        if (lo == hi)
            parse_err("function '" + nm.text + "' expects " + std::to_string(lo) + " argument" +
                      (lo == 1 ? "" : "s") + ", got " + std::to_string(n) + " (column " +
                      std::to_string(nm.col) + ")");
        parse_err("function '" + nm.text + "' expects " + std::to_string(lo) + " to " +
                  std::to_string(hi) + " arguments, got " + std::to_string(n) + " (column " +
                  std::to_string(nm.col) + ")");
    }
    NodeP call(const Tok& nm) {
        std::vector<NodeP> args;
        expect(Tk::LParen, "after function name");
        if (!accept(Tk::RParen)) {
            do {
                args.push_back(vec());
            } while (accept(Tk::Comma));
            expect(Tk::RParen, "to close the argument list");
        }
        auto with = [&](K k, int op) {
            NodeP n = mk(k, op);
            n->name = nm.text;
            n->a = std::move(args);
            return n;
        };
        nau_op_info info;
        if (nau_find_interaction(nm.text.c_str(), &info) == NAU_OK) {
            arity(nm, args, info.arity_min, info.arity_max);
            if (info.kernel_slot >= 0 && args[info.kernel_slot]->k != K::Kernel)
                parse_err("operand " + std::to_string(info.kernel_slot + 1) + " of '" + nm.text +
                          "' must be a smoothing kernel keyword");
            NodeP n = with(K::Inter, info.op);
            n->info = info;
            return n;
        }
        if (nm.text == "euler") {
            arity(nm, args, 3, 3);
            return with(K::Euler, 0);
        }
        if (nm.text == "rand") {
            arity(nm, args, 2, 2);
            return with(K::Rand, NAU_VM_RAND);
        }
        const char* reds[] = {"fmax", "fmin", "fsum", "fmean"};
        for (int r = 0; r < 4; ++r)
            if (nm.text == reds[r]) {
                arity(nm, args, 1, 1);
                return with(K::Red, r);
            }
        for (const auto& u : kUnary)
            if (nm.text == u.name) {
                arity(nm, args, 1, 1);
                return with(K::Call1, u.op);
            }
        for (const auto& b : kBinary)
            if (nm.text == b.name) {
                arity(nm, args, 2, 2);
                return with(K::Call2, b.op);
            }
        parse_err("unknown function '" + nm.text + "' at column " + std::to_string(nm.col));
    }

    std::vector<Tok> t_;
    nau_case& cs_;
    size_t p_ = 0;
};

// ---- lowering ----
struct Solver {
    nau_case& cs;
    nau_ctx* ctx;

    void check(nau_status s) {
        if (s == NAU_OK) return;
        long bad = -1;
        const char* m = nau_last_error(ctx, &bad);
        throw ExecError{s, m ? m : "", bad};
    }

    int temp(int rows, int cols) {
        for (auto& t : cs.temps)
            if (!t.busy && t.rows == rows && t.cols == cols) {
                t.busy = true;
                return t.id;
            }
        int id = -1;
        check(nau_alloc_field(ctx, rows, cols, &id));
        cs.temps.push_back({id, rows, cols, true});
        return id;
    }
    void release_temps() {
        for (auto& t : cs.temps) t.busy = false;
    }

    static bool has_field_kind(const Node& n) {
        if (n.k == K::Field || n.k == K::Rand || n.k == K::Inter) return true;
        if (n.k == K::Red) return false;  // frozen: uniform
        for (const auto& c : n.a)
            if (has_field_kind(*c)) return true;
        return false;
    }

    // shape of a subtree (static) — the reference's evaluation-time shape errors
    void field_shape(int id, int& r, int& c) { check(nau_field_shape(ctx, id, &r, &c)); }

    Tn shape_only(int r, int c) {
        Tn t;
        t.r = r;
        t.c = c;
        return t;
    }

    // Interaction result shape (nau_interact's rules, interactions.cpp)
    Tn inter_shape(const Node& n, const Tn& a0) {
        switch (n.op) {
            case NAU_OP_SPH_S: return shape_only(a0.r, a0.c);
            case NAU_OP_SPH_D00:
            case NAU_OP_SPH_L0: return shape_only(1, 1);
            default: return shape_only(cs.dim, 1);
        }
    }

    // Post-order: freeze reductions, materialise interactions (the reference evaluates
    // both before the particle-wise arithmetic that consumes them).
    void prepare(Node& n) {
        if (n.k == K::Red) {
            for (auto& c : n.a) prepare(*c);
            n.red = reduce(n);
            n.uniform = true;
            return;
        }
        for (auto& c : n.a) prepare(*c);
        n.uniform = !has_field_kind(n);
        if (n.k == K::Inter) interact(n);
    }

    // Host value of a uniform subtree (tensor.cpp rules, host libm).
    Tn fold(const Node& n) {
        switch (n.k) {
            case K::Lit: return n.lit;
            case K::Const: return cs.constants[n.sym].value;
            case K::Var: return cs.variables[n.sym].value;
            case K::Red: return n.red;
            case K::Kernel:
                fail_rt("kernel keyword '" + n.name + "' used outside an interaction operand");
            case K::Neg: return t_elem1(fold(*n.a[0]), [](double x) { return -x; });
            case K::Bin: {
                Tn a = fold(*n.a[0]), b = fold(*n.a[1]);
                try {
                    return bin_host(n.op, a, b);
                } catch (ExecError& e) {
                    e.msg += " in '" + text_of(n) + "'";
                    throw;
                }
            }
            case K::Join: {
                Tn h = fold(*n.a[0]), t = fold(*n.a[1]);
                if (h.c != 1 || !t.scalar() || h.r >= 3)
                    fail_rt("operator '|': cannot append a " + shape_str(t) + " component to a " +
                            shape_str(h) + " value in '" + text_of(n) + "'");
                Tn o;
                o.r = h.r + 1;
                for (int q = 0; q < h.r; ++q) o.v[q] = h.v[q];
                o.v[h.r] = t.v[0];
                return o;
            }
            case K::Call1:
            case K::Call2:
                try {
                    return call_host(n);
                } catch (ExecError& e) {
                    if (e.msg.find(" in '") == std::string::npos) e.msg += " in '" + text_of(n) + "'";
                    throw;
                }
            case K::Euler: {
                Tn x = fold(*n.a[0]), xd = fold(*n.a[1]), dt = fold(*n.a[2]);
                euler_check(n, x.r, x.c, xd.r, xd.c, dt.r, dt.c);
                return t_add(x, t_mul(xd, dt), false);
            }
            default: fail_rt("internal: non-uniform subtree folded");
        }
    }

    void euler_check(const Node& n, int xr, int xc, int dr, int dc, int tr, int tc) {
        if (!(tr == 1 && tc == 1))
            fail_rt("euler: time step must be a scalar, got " + shape_str(tr, tc) + " in '" +
                    text_of(n) + "'");
        if (xr != dr || xc != dc)
            fail_rt("euler: state is " + shape_str(xr, xc) + " but derivative is " +
                    shape_str(dr, dc) + " in '" + text_of(n) + "'");
    }

    static Tn bin_host(int op, const Tn& a, const Tn& b) {
        switch (op) {
            case B_ADD: return t_add(a, b, false);
            case B_SUB: return t_add(a, b, true);
            case B_MUL: return t_mul(a, b);
            case B_DIV: return t_div(a, b);
            case B_POW: return t_elem2("^", a, b, [](double x, double e) { return std::pow(x, e); });
            default: {
                if (!a.scalar() || !b.scalar()) shape_mismatch("comparison", a.r, a.c, b.r, b.c);
                const double x = a.v[0], y = b.v[0];
                bool r = false;
                switch (op) {
                    case B_LT: r = x < y; break;
                    case B_GT: r = x > y; break;
                    case B_LE: r = x <= y; break;
                    case B_GE: r = x >= y; break;
                    case B_EQ: r = x == y; break;
                    default: r = x != y; break;
                }
                return scalar_tn(r ? 1.0 : 0.0);
            }
        }
    }

    Tn call_host(const Node& n) {
        if (n.k == K::Call2) {
            Tn a = fold(*n.a[0]), b = fold(*n.a[1]);
            if (n.op == NAU_VM_MIN)
                return t_elem2("min", a, b, [](double x, double y) { return std::fmin(x, y); });
            if (n.op == NAU_VM_MAX)
                return t_elem2("max", a, b, [](double x, double y) { return std::fmax(x, y); });
            if (a.r != b.r || a.c != b.c) shape_mismatch("dot", a.r, a.c, b.r, b.c);
            double s = a.v[0] * b.v[0];
            for (int q = 1; q < a.size(); ++q) s = s + a.v[q] * b.v[q];
            return scalar_tn(s);
        }
        Tn a = fold(*n.a[0]);
        switch (n.op) {
            case NAU_VM_EXP: return t_elem1(a, [](double x) { return std::exp(x); });
            case NAU_VM_LOG: return t_elem1(a, [](double x) { return std::log(x); });
            case NAU_VM_SIN: return t_elem1(a, [](double x) { return std::sin(x); });
            case NAU_VM_COS: return t_elem1(a, [](double x) { return std::cos(x); });
            case NAU_VM_TAN: return t_elem1(a, [](double x) { return std::tan(x); });
            case NAU_VM_SQRT: return t_elem1(a, [](double x) { return std::sqrt(x); });
            case NAU_VM_ABS: return t_elem1(a, [](double x) { return std::abs(x); });
            case NAU_VM_FLOOR: return t_elem1(a, [](double x) { return std::floor(x); });
            case NAU_VM_SGN:
                return t_elem1(a, [](double x) { return x > 0 ? 1.0 : (x < 0 ? -1.0 : 0.0); });
            default: {  // norm: sqrt(squaredNorm()), storage order
                double s = a.v[0] * a.v[0];
                for (int q = 1; q < a.size(); ++q) s = s + a.v[q] * a.v[q];
                return scalar_tn(std::sqrt(s));
            }
        }
    }

    // ---- VM programs ----
    struct Prog {
        std::vector<nau_vm_instr> code;
    };

    void emit(Prog& p, int op, int dst, int a = 0, int b = 0, int field = -1, const Tn* imm = nullptr) {
        nau_vm_instr in;
        std::memset(&in, 0, sizeof(in));
        in.op = op;
        in.dst = dst;
        in.a = a;
        in.b = b;
        in.field = field;
        in.rows = imm ? imm->r : 1;
        in.cols = imm ? imm->c : 1;
        if (imm)
            for (int q = 0; q < 9; ++q) in.imm[q] = imm->v[q];
        p.code.push_back(in);
    }

    // Emits node into register r; returns its shape (checking the reference's rules,
    // so that errors carry the reference's messages before anything launches).
    Tn gen(Prog& p, const Node& n, int r) {
        if (r >= NAU_VM_MAX_REGS) fail_rt("expression too deep for the device evaluator");
        if (n.uniform) {
            Tn v = fold(n);
            emit(p, NAU_VM_LOAD_CONST, r, 0, 0, -1, &v);
            return shape_only(v.r, v.c);
        }
        switch (n.k) {
            case K::Field: {
                int fr, fc;
                field_shape(n.sym, fr, fc);
                emit(p, NAU_VM_LOAD_FIELD, r, 0, 0, n.sym);
                return shape_only(fr, fc);
            }
            case K::Inter: {
                int fr, fc;
                field_shape(n.temp, fr, fc);
                emit(p, NAU_VM_LOAD_FIELD, r, 0, 0, n.temp);
                return shape_only(fr, fc);
            }
            case K::Neg: {
                Tn a = gen(p, *n.a[0], r);
                emit(p, NAU_VM_NEG, r, r);
                return a;
            }
            case K::Bin: {
                Tn a = gen(p, *n.a[0], r), b = gen(p, *n.a[1], r + 1);
                Tn s;
                try {
                    s = bin_shape(n.op, a, b);
                } catch (ExecError& e) {
                    e.msg += " in '" + text_of(n) + "'";
                    throw;
                }
                const int vm[] = {NAU_VM_ADD, NAU_VM_SUB, NAU_VM_MUL, NAU_VM_DIV, NAU_VM_POW, NAU_VM_LT,
                                  NAU_VM_GT,  NAU_VM_LE,  NAU_VM_GE,  NAU_VM_EQ,  NAU_VM_NE};
                emit(p, vm[n.op], r, r, r + 1);
                return s;
            }
            case K::Join: {
                Tn h = gen(p, *n.a[0], r), t = gen(p, *n.a[1], r + 1);
                if (h.c != 1 || !t.scalar() || h.r >= 3)
                    fail_rt("operator '|': cannot append a " + shape_str(t) + " component to a " +
                            shape_str(h) + " value in '" + text_of(n) + "'");
                emit(p, NAU_VM_JOIN, r, r, r + 1);
                return shape_only(h.r + 1, 1);
            }
            case K::Call1:
            case K::Call2:  // BuiltinCallNode: argument errors get the call's text too
                try {
                    if (n.k == K::Call1) {
                        Tn a = gen(p, *n.a[0], r);
                        emit(p, n.op, r, r);
                        return n.op == NAU_VM_NORM ? shape_only(1, 1) : a;
                    }
                    Tn a = gen(p, *n.a[0], r), b = gen(p, *n.a[1], r + 1);
                    Tn s;
                    if (n.op == NAU_VM_DOT) {
                        if (a.r != b.r || a.c != b.c) shape_mismatch("dot", a.r, a.c, b.r, b.c);
                        s = shape_only(1, 1);
                    } else {
                        s = elem2_shape(n.op == NAU_VM_MIN ? "min" : "max", a, b);
                    }
                    emit(p, n.op, r, r, r + 1);
                    return s;
                } catch (ExecError& e) {
                    if (e.msg.find(" in '") == std::string::npos) e.msg += " in '" + text_of(n) + "'";
                    throw;
                }
            case K::Euler: {  // x + xdot * dt (ast.cpp:180-191)
                Tn x = gen(p, *n.a[0], r), xd = gen(p, *n.a[1], r + 1), dt = gen(p, *n.a[2], r + 2);
                euler_check(n, x.r, x.c, xd.r, xd.c, dt.r, dt.c);
                emit(p, NAU_VM_MUL, r + 1, r + 1, r + 2);
                emit(p, NAU_VM_ADD, r, r, r + 1);
                return x;
            }
            case K::Rand: {
                Tn a = gen(p, *n.a[0], r), b = gen(p, *n.a[1], r + 1);
                if (!a.scalar() || !b.scalar())
                    fail_rt("expected a scalar, got a " + shape_str(a.scalar() ? b : a) + " tensor");
                emit(p, NAU_VM_RAND, r, r, r + 1);
                return shape_only(1, 1);
            }
            default: fail_rt("internal: unexpected node in a particle-wise program");
        }
    }

    static Tn elem2_shape(const char* name, const Tn& a, const Tn& b) {
        Tn o;
        if (a.scalar() && !b.scalar()) o = b;
        else if (b.scalar() && !a.scalar()) o = a;
        else if (a.r == b.r && a.c == b.c) o = a;
        else shape_mismatch(name, a.r, a.c, b.r, b.c);
        return o;
    }

    static Tn bin_shape(int op, const Tn& a, const Tn& b) {
        Tn o;
        switch (op) {
            case B_ADD:
            case B_SUB:
                if (a.r != b.r || a.c != b.c) shape_mismatch(op == B_ADD ? "+" : "-", a.r, a.c, b.r, b.c);
                return a;
            case B_MUL:
                if (a.scalar()) return b;
                if (b.scalar()) return a;
                if (a.c != b.r) shape_mismatch("*", a.r, a.c, b.r, b.c);
                o.r = a.r;
                o.c = b.c;
                return o;
            case B_DIV:
                if (b.scalar()) return a;
                if (a.r != b.r || a.c != b.c) shape_mismatch("/", a.r, a.c, b.r, b.c);
                return a;
            case B_POW: return elem2_shape("^", a, b);
            default:
                if (!a.scalar() || !b.scalar()) shape_mismatch("comparison", a.r, a.c, b.r, b.c);
                return o;
        }
    }

    // The subtree as an interaction operand / reduction argument: a field id (>= 0)
    // or a uniform value. Non-trivial per-particle subtrees run as a program into a
    // temporary field.
    struct Opnd {
        int field = -1;
        Tn value;
    };
    Opnd materialise(const Node& n) {
        Opnd o;
        if (n.uniform) {
            o.value = fold(n);
            return o;
        }
        if (n.k == K::Field) {
            o.field = n.sym;
            return o;
        }
        if (n.k == K::Inter) {
            o.field = n.temp;
            return o;
        }
        Prog p;
        Tn s = gen(p, n, 0);
        const int id = temp(s.r, s.c);
        check(nau_eval(ctx, p.code.data(), (int)p.code.size(), 0, id));
        o.field = id;
        return o;
    }

    void interact(Node& n) {
        const nau_op_info& info = n.info;
        std::vector<nau_operand> ops;
        int kf = 0, kd = 0;
        Tn a0;
        for (int q = 0; q < (int)n.a.size(); ++q) {
            if (q == info.kernel_slot) {
                kf = n.a[q]->kf;
                kd = n.a[q]->kd;
                continue;
            }
            if (n.a[q]->k == K::Kernel)
                fail_rt("kernel keyword '" + n.a[q]->name + "' used outside an interaction operand");
            if (n.a[q]->k == K::Rand || has_rand(*n.a[q]))
                fail_rt("rand() inside an interaction operand is evaluated per neighbour by the "
                        "reference; materialise it in its own equation first");
            Opnd m = materialise(*n.a[q]);
            nau_operand o;
            std::memset(&o, 0, sizeof(o));
            o.field_id = m.field;
            if (m.field >= 0) {
                field_shape(m.field, o.rows, o.cols);
            } else {
                o.rows = m.value.r;
                o.cols = m.value.c;
                for (int c = 0; c < 9; ++c) o.value[c] = m.value.v[c];
            }
            if (ops.empty()) a0 = shape_only(o.rows, o.cols);
            ops.push_back(o);
        }
        const Tn s = inter_shape(n, a0);
        n.temp = temp(s.r, s.c);
        check(nau_interact(ctx, info.op, kf, kd, ops.data(), (int)ops.size(), n.temp));
    }

    static bool has_rand(const Node& n) {
        if (n.k == K::Rand) return true;
        for (const auto& c : n.a)
            if (has_rand(*c)) return true;
        return false;
    }

    long global_active() {
        double cnt = (double)nau_active_count(ctx);
        check(nau_allreduce(ctx, &cnt, 1, 0));
        return (long)cnt;
    }

    // ReductionNode::compute (ast.cpp:237-268) over every rank's active particles.
    Tn reduce(const Node& n) {
        if (global_active() == 0)
            fail_rt("reduction '" + text_of(n) + "' over an empty particle system");
        Opnd m = materialise(*n.a[0]);
        int field = m.field;
        if (field < 0) {  // a uniform argument still sums once per active particle
            field = temp(m.value.r, m.value.c);
            check(nau_fill(ctx, field, m.value.v));
        }
        int fr, fc;
        field_shape(field, fr, fc);
        double out[10] = {0};
        Tn t;
        if (n.op == R_MAX || n.op == R_MIN) {
            if (nau_active_count(ctx) > 0) {
                check(nau_reduce(ctx, n.op, field, out));
            } else {  // an empty rank contributes the identity
                out[0] = n.op == R_MAX ? -INFINITY : INFINITY;
            }
            check(nau_allreduce(ctx, out, 1, n.op == R_MAX ? 1 : 2));
            return scalar_tn(out[0]);
        }
        const int comps = fr * fc;
        if (nau_active_count(ctx) > 0) check(nau_reduce(ctx, R_SUM, field, out));
        out[comps] = (double)nau_active_count(ctx);
        check(nau_allreduce(ctx, out, comps + 1, 0));
        t.r = fr;
        t.c = fc;
        for (int q = 0; q < comps; ++q)
            t.v[q] = n.op == R_MEAN ? out[q] / out[comps] : out[q];
        return t;
    }

    void clear(Node& n) {
        n.temp = -1;
        for (auto& c : n.a) clear(*c);
    }

    // Case::solve_equation (case.cpp:9-63)
    void solve(nau_case::Equation& eq) {
        clear(*eq.rhs);
        prepare(*eq.rhs);
        if (eq.lhs_var >= 0) {  // single-valued LHS: evaluated at particle 0 (case.cpp:19-29)
            Tn value;
            if (eq.rhs->uniform) {
                value = fold(*eq.rhs);
            } else {
                Opnd m = materialise(*eq.rhs);
                int fr, fc;
                field_shape(m.field, fr, fc);
                const long n = nau_particle_count(ctx);
                std::vector<double> h((size_t)n * fr * fc);
                check(nau_download(ctx, m.field, h.data(), n));
                value.r = fr;
                value.c = fc;
                for (int q = 0; q < fr * fc; ++q) value.v[q] = n > 0 ? h[(size_t)q * n] : 0.0;
            }
            Tn& var = cs.variables[eq.lhs_var].value;
            if (value.r != var.r || value.c != var.c)
                fail_rt("LHS '" + eq.lhs + "' is " + shape_str(var) + " but RHS produced " +
                        shape_str(value));
            for (int q = 0; q < value.size(); ++q)
                if (!std::isfinite(value.v[q])) fail_rt("non-finite value assigned", NAU_ERR_NAN);
            var = value;
            return;
        }
        Prog p;
        const Tn s = gen(p, *eq.rhs, 0);
        int lr, lc;
        field_shape(eq.lhs_field, lr, lc);
        if (s.r != lr || s.c != lc) {
            long first = 0;  // the first active particle (ThreadPool order)
            const long n = nau_particle_count(ctx);
            std::vector<uint8_t> act((size_t)std::max(1L, n));
            if (nau_get_active(ctx, act.data()) == NAU_OK)
                while (first < n && !act[first]) ++first;
            fail_rt("LHS field '" + eq.lhs + "' is " + shape_str(lr, lc) + " but RHS produced " +
                    shape_str(s) + " at particle " + std::to_string(first));
        }
        if ((int)p.code.size() > NAU_VM_MAX_INSTR)
            fail_rt("expression too long for the device evaluator");
        // nau_eval: two-phase write, inactive particles frozen, NaN audit; r written =>
        // apply_boundary_shift + dirty cells (case.cpp:59-62)
        check(nau_eval(ctx, p.code.data(), (int)p.code.size(), 0, eq.lhs_field));
    }
};

nau_status fail_case(nau_case* cs, const ExecError& e, const std::string& prefix) {
    cs->last_error = prefix + e.msg;
    cs->last_bad = e.bad;
    return e.st;
}

Tn tn_from(int rows, int cols, const double* v) {
    Tn t;
    t.r = rows;
    t.c = cols;
    for (int q = 0; q < rows * cols; ++q) t.v[q] = v[q];
    return t;
}

}  // namespace

extern "C" {

nau_status nau_case_create(nau_ctx* ctx, nau_case** out) {
    if (!ctx || !out) return NAU_ERR_ARG;
    auto* cs = new nau_case;
    cs->ctx = ctx;
    int r = 0, c = 0;
    if (nau_field_shape(ctx, 0, &r, &c) != NAU_OK) {
        delete cs;
        return NAU_ERR_ARG;  // nau_set_particles first
    }
    cs->dim = r;
    cs->fields["r"] = 0;
    *out = cs;
    return NAU_OK;
}

void nau_case_destroy(nau_case* cs) {
    if (!cs) return;
    for (auto& t : cs->temps) nau_free_field(cs->ctx, t.id);
    delete cs;
}

static nau_status add_sym(nau_case* cs, std::vector<nau_case::Sym>& v, const char* name, int rows,
                          int cols, const double* value) {
    if (!name || rows < 1 || rows > 3 || cols < 1 || cols > 3 || !value) {
        cs->last_error = "bad symbol";
        return NAU_ERR_ARG;
    }
    const std::string nm(name);
    if (find_sym(cs->constants, nm) >= 0 || find_sym(cs->variables, nm) >= 0 || cs->fields.count(nm)) {
        cs->last_error = "duplicate symbol name '" + nm + "'";  // workspace.cpp reserve_name
        return NAU_ERR_ARG;
    }
    v.push_back({nm, tn_from(rows, cols, value)});
    return NAU_OK;
}

nau_status nau_case_constant(nau_case* cs, const char* name, int rows, int cols, const double* value) {
    return add_sym(cs, cs->constants, name, rows, cols, value);
}

nau_status nau_case_variable(nau_case* cs, const char* name, int rows, int cols, const double* value) {
    return add_sym(cs, cs->variables, name, rows, cols, value);
}

nau_status nau_case_set_variable(nau_case* cs, const char* name, int rows, int cols,
                                 const double* value) {
    const int k = find_sym(cs->variables, name ? name : "");
    if (k < 0 || rows < 1 || rows > 3 || cols < 1 || cols > 3) {
        cs->last_error = std::string("unknown variable '") + (name ? name : "") + "'";
        return NAU_ERR_ARG;
    }
    cs->variables[k].value = tn_from(rows, cols, value);
    return NAU_OK;
}

nau_status nau_case_get_variable(nau_case* cs, const char* name, double* value, int* rows, int* cols) {
    const int k = find_sym(cs->variables, name ? name : "");
    if (k < 0) {
        cs->last_error = std::string("unknown variable '") + (name ? name : "") + "'";
        return NAU_ERR_ARG;
    }
    const Tn& t = cs->variables[k].value;
    *rows = t.r;
    *cols = t.c;
    for (int q = 0; q < t.size(); ++q) value[q] = t.v[q];
    return NAU_OK;
}

nau_status nau_case_field(nau_case* cs, const char* name, int field_id) {
    int r, c;
    if (!name || nau_field_shape(cs->ctx, field_id, &r, &c) != NAU_OK) {
        cs->last_error = "bad field";
        return NAU_ERR_ARG;
    }
    const std::string nm(name);
    if (find_sym(cs->constants, nm) >= 0 || find_sym(cs->variables, nm) >= 0 ||
        (cs->fields.count(nm) && cs->fields[nm] != field_id)) {
        cs->last_error = "duplicate symbol name '" + nm + "'";
        return NAU_ERR_ARG;
    }
    cs->fields[nm] = field_id;
    return NAU_OK;
}

// assemble.cpp:171-196: "lhs=rhs", LHS a variable or a field, errors prefixed
// "in equation '<name>': " (with_context) like the reference's assembly errors.
nau_status nau_case_equation(nau_case* cs, const char* name, const char* text) {
    const std::string nm(name ? name : ""), t(text ? text : "");
    const std::string prefix = "in equation '" + nm + "': ";
    try {
        const size_t eq = t.find('=');
        if (eq == std::string::npos) parse_err("an equation must have the form lhs=rhs");
        std::string lhs = t.substr(0, eq);
        lhs.erase(0, lhs.find_first_not_of(" \t"));
        lhs.erase(lhs.find_last_not_of(" \t") + 1);
        nau_case::Equation e;
        e.name = nm;
        e.lhs = lhs;
        e.lhs_var = find_sym(cs->variables, lhs);
        if (e.lhs_var < 0) {
            auto it = cs->fields.find(lhs);
            if (it == cs->fields.end()) {
                if (find_sym(cs->constants, lhs) >= 0)
                    parse_err("the LHS symbol '" + lhs + "' is a constant and cannot be assigned");
                parse_err("unknown symbol '" + lhs + "' on the LHS");
            }
            e.lhs_field = it->second;
        }
        e.rhs = Parser(t.substr(eq + 1), *cs).full();
        cs->equations.push_back(std::move(e));
        return NAU_OK;
    } catch (const ExecError& e) {
        return fail_case(cs, e, prefix);
    }
}

int nau_case_equation_count(nau_case* cs) { return (int)cs->equations.size(); }

nau_status nau_case_solve_equation(nau_case* cs, int index) {
    if (index < 0 || index >= (int)cs->equations.size()) {
        cs->last_error = "bad equation index";
        return NAU_ERR_ARG;
    }
    auto& eq = cs->equations[index];
    Solver sv{*cs, cs->ctx};
    try {
        sv.solve(eq);
        sv.check(nau_sync(cs->ctx));  // device errors of this equation surface here
        sv.release_temps();
        return NAU_OK;
    } catch (const ExecError& e) {
        sv.release_temps();
        nau_sync(cs->ctx);
        return fail_case(cs, e, "equation '" + eq.name + "': ");
    }
}

nau_status nau_case_solve_step(nau_case* cs) {
    for (int k = 0; k < (int)cs->equations.size(); ++k) {
        nau_status s = nau_case_solve_equation(cs, k);
        if (s != NAU_OK) return s;
    }
    ++cs->steps;
    return NAU_OK;
}

const char* nau_case_last_error(nau_case* cs, long* first_bad) {
    if (first_bad) *first_bad = cs ? cs->last_bad : -1;
    return cs ? cs->last_error.c_str() : "";
}

}  // extern "C"
