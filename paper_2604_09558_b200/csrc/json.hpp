// Minimal JSON value, parser and writer for the VTC graph schema
// ({"tensors":[...], "nodes":[...]}) and report output.
// Own implementation: the product library has no third-party JSON dependency.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace vtc::json {

struct Value;
using Array = std::vector<Value>;
using Object = std::vector<std::pair<std::string, Value>>;  // insertion order kept

struct Value {
    enum class T { Null, Bool, Int, Double, String, Array, Object } t = T::Null;
    bool b = false;
    int64_t i = 0;
    double d = 0.0;
    std::string s;
    std::shared_ptr<Array> a;
    std::shared_ptr<Object> o;

    Value() = default;
    static Value null() { return Value(); }
    static Value boolean(bool v) { Value x; x.t = T::Bool; x.b = v; return x; }
    static Value integer(int64_t v) { Value x; x.t = T::Int; x.i = v; return x; }
    static Value number(double v) { Value x; x.t = T::Double; x.d = v; return x; }
    static Value string(std::string v) { Value x; x.t = T::String; x.s = std::move(v); return x; }
    static Value array() { Value x; x.t = T::Array; x.a = std::make_shared<Array>(); return x; }
    static Value object() { Value x; x.t = T::Object; x.o = std::make_shared<Object>(); return x; }
    static Value ints(const std::vector<int64_t>& v) {
        Value x = array();
        for (auto e : v) x.a->push_back(integer(e));
        return x;
    }

    bool is_int() const { return t == T::Int; }
    bool is_array() const { return t == T::Array; }
    bool is_object() const { return t == T::Object; }
    bool is_string() const { return t == T::String; }
    bool contains(const std::string& k) const {
        if (t != T::Object) return false;
        for (const auto& kv : *o)
            if (kv.first == k) return true;
        return false;
    }
    const Value& at(const std::string& k) const {
        if (t != T::Object) throw std::runtime_error("json: not an object (key " + k + ")");
        for (const auto& kv : *o)
            if (kv.first == k) return kv.second;
        throw std::runtime_error("json: missing key " + k);
    }
    Value& set(const std::string& k, Value v) {
        if (t != T::Object) throw std::runtime_error("json: set on non-object");
        for (auto& kv : *o)
            if (kv.first == k) return kv.second = std::move(v);
        o->emplace_back(k, std::move(v));
        return o->back().second;
    }
    void push(Value v) { a->push_back(std::move(v)); }
    size_t size() const { return t == T::Array ? a->size() : t == T::Object ? o->size() : 0; }
    const Value& operator[](size_t i) const { return (*a)[i]; }
    int64_t as_int() const {
        if (t == T::Int) return i;
        if (t == T::Double && double(int64_t(d)) == d) return int64_t(d);
        throw std::runtime_error("json: expected integer");
    }
    double as_double() const {
        if (t == T::Int) return double(i);
        if (t == T::Double) return d;
        throw std::runtime_error("json: expected number");
    }
    const std::string& as_string() const {
        if (t != T::String) throw std::runtime_error("json: expected string");
        return s;
    }
    bool as_bool() const {
        if (t != T::Bool) throw std::runtime_error("json: expected bool");
        return b;
    }
};

class Parser {
public:
    explicit Parser(const std::string& text) : s_(text) {}
    Value parse() {
        Value v = value();
        ws();
        if (p_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    const std::string& s_;
    size_t p_ = 0;

    [[noreturn]] void fail(const std::string& why) {
        throw std::runtime_error("json parse error at " + std::to_string(p_) + ": " + why);
    }
    void ws() {
        while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\n' || s_[p_] == '\t' || s_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        ws();
        if (p_ < s_.size() && s_[p_] == c) { ++p_; return true; }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    Value value() {
        ws();
        if (p_ >= s_.size()) fail("unexpected end");
        char c = s_[p_];
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') return Value::string(str());
        if (c == 't' || c == 'f' || c == 'n') return literal();
        return num();
    }
    Value object() {
        expect('{');
        Value v = Value::object();
        if (eat('}')) return v;
        do {
            ws();
            std::string k = str();
            expect(':');
            v.o->emplace_back(std::move(k), value());
        } while (eat(','));
        expect('}');
        return v;
    }
    Value array() {
        expect('[');
        Value v = Value::array();
        if (eat(']')) return v;
        do v.a->push_back(value());
        while (eat(','));
        expect(']');
        return v;
    }
    std::string str() {
        if (p_ >= s_.size() || s_[p_] != '"') fail("expected string");
        ++p_;
        std::string out;
        while (p_ < s_.size() && s_[p_] != '"') {
            char c = s_[p_++];
            if (c == '\\') {
                if (p_ >= s_.size()) fail("bad escape");
                char e = s_[p_++];
                switch (e) {
                    case 'n': out += '\n'; break;
                    case 't': out += '\t'; break;
                    case 'r': out += '\r'; break;
                    case 'b': out += '\b'; break;
                    case 'f': out += '\f'; break;
                    case 'u': {
                        if (p_ + 4 > s_.size()) fail("bad \\u escape");
                        unsigned cp = std::stoul(s_.substr(p_, 4), nullptr, 16);
                        p_ += 4;
                        if (cp < 0x80) out += char(cp);
                        else if (cp < 0x800) { out += char(0xC0 | (cp >> 6)); out += char(0x80 | (cp & 0x3F)); }
                        else { out += char(0xE0 | (cp >> 12)); out += char(0x80 | ((cp >> 6) & 0x3F)); out += char(0x80 | (cp & 0x3F)); }
                        break;
                    }
                    default: out += e;
                }
            } else {
                out += c;
            }
        }
        if (p_ >= s_.size()) fail("unterminated string");
        ++p_;
        return out;
    }
    Value literal() {
        if (s_.compare(p_, 4, "true") == 0) { p_ += 4; return Value::boolean(true); }
        if (s_.compare(p_, 5, "false") == 0) { p_ += 5; return Value::boolean(false); }
        if (s_.compare(p_, 4, "null") == 0) { p_ += 4; return Value::null(); }
        fail("bad literal");
    }
    Value num() {
        size_t st = p_;
        bool is_float = false;
        if (s_[p_] == '-' || s_[p_] == '+') ++p_;
        while (p_ < s_.size()) {
            char c = s_[p_];
            if (c >= '0' && c <= '9') { ++p_; continue; }
            if (c == '.' || c == 'e' || c == 'E' || c == '-' || c == '+') { is_float = true; ++p_; continue; }
            break;
        }
        std::string tok = s_.substr(st, p_ - st);
        if (tok.empty() || tok == "-") fail("bad number");
        if (!is_float) return Value::integer(std::stoll(tok));
        return Value::number(std::stod(tok));
    }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline void dump_to(const Value& v, std::string& out, int indent, int depth) {
    auto nl = [&](int d) {
        if (indent < 0) return;
        out += '\n';
        out.append(size_t(indent * d), ' ');
    };
    switch (v.t) {
        case Value::T::Null: out += "null"; break;
        case Value::T::Bool: out += v.b ? "true" : "false"; break;
        case Value::T::Int: out += std::to_string(v.i); break;
        case Value::T::Double: {
            char buf[64];
            snprintf(buf, sizeof(buf), "%.17g", v.d);
            out += buf;
            break;
        }
        case Value::T::String: {
            out += '"';
            for (char c : v.s) {
                if (c == '"' || c == '\\') { out += '\\'; out += c; }
                else if (c == '\n') out += "\\n";
                else out += c;
            }
            out += '"';
            break;
        }
        case Value::T::Array: {
            out += '[';
            bool flat = true;
            for (const auto& e : *v.a)
                if (e.t == Value::T::Array || e.t == Value::T::Object) flat = false;
            for (size_t i = 0; i < v.a->size(); ++i) {
                if (i) out += flat ? ", " : ",";
                if (!flat) nl(depth + 1);
                dump_to((*v.a)[i], out, indent, depth + 1);
            }
            if (!flat && !v.a->empty()) nl(depth);
            out += ']';
            break;
        }
        case Value::T::Object: {
            out += '{';
            for (size_t i = 0; i < v.o->size(); ++i) {
                if (i) out += ',';
                nl(depth + 1);
                out += '"' + (*v.o)[i].first + "\":";
                if (indent >= 0) out += ' ';
                dump_to((*v.o)[i].second, out, indent, depth + 1);
            }
            if (!v.o->empty()) nl(depth);
            out += '}';
            break;
        }
    }
}

inline std::string dump(const Value& v, int indent = -1) {
    std::string out;
    dump_to(v, out, indent, 0);
    return out;
}

}  // namespace vtc::json
