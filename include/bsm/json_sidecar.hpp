// bsm/json_sidecar.hpp -- the small JSON dialect of the reference's sidecar
// files (config.hpp:48-110, pattern.hpp:104-160): a reader for plain JSON
// documents and the writer's exact layout (nlohmann dump(1, '\t'): keys in
// byte order, one tab per level, shortest round-trip numbers).
#pragma once

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "bsm/errors.hpp"

namespace bsm::json {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    bool is_int = false;  // the token had no fraction/exponent
    long long ival = 0;
    unsigned long long uval = 0;
    bool neg = false;
    std::string str;
    std::vector<Value> arr;
    std::map<std::string, Value> obj;

    const Value* find(const std::string& k) const {
        if (kind != Object) return nullptr;
        auto it = obj.find(k);
        return it == obj.end() ? nullptr : &it->second;
    }
};

class Parser {
public:
    explicit Parser(const std::string& text) : s_(text) {}

    Value document() {
        Value v = value();
        space();
        if (p_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    const std::string& s_;
    std::size_t p_ = 0;

    [[noreturn]] void fail(const char* what) const {
        throw FormatError(std::string("parse error at byte ") + std::to_string(p_) + ": " + what);
    }
    void space() {
        while (p_ < s_.size() && (s_[p_] == ' ' || s_[p_] == '\t' || s_[p_] == '\n' || s_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        space();
        if (p_ < s_.size() && s_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    Value value() {
        space();
        if (p_ >= s_.size()) fail("unexpected end of input");
        const char c = s_[p_];
        Value v;
        if (c == '{') {
            ++p_;
            v.kind = Value::Object;
            if (eat('}')) return v;
            do {
                space();
                if (p_ >= s_.size() || s_[p_] != '"') fail("expected object key");
                const std::string k = string();
                if (!eat(':')) fail("expected ':'");
                v.obj[k] = value();
            } while (eat(','));
            if (!eat('}')) fail("expected '}'");
        } else if (c == '[') {
            ++p_;
            v.kind = Value::Array;
            if (eat(']')) return v;
            do v.arr.push_back(value());
            while (eat(','));
            if (!eat(']')) fail("expected ']'");
        } else if (c == '"') {
            v.kind = Value::String;
            v.str = string();
        } else if (s_.compare(p_, 4, "true") == 0) {
            p_ += 4;
            v.kind = Value::Bool;
            v.b = true;
        } else if (s_.compare(p_, 5, "false") == 0) {
            p_ += 5;
            v.kind = Value::Bool;
        } else if (s_.compare(p_, 4, "null") == 0) {
            p_ += 4;
        } else {
            number(v);
        }
        return v;
    }
    std::string string() {
        ++p_;  // opening quote
        std::string out;
        while (p_ < s_.size() && s_[p_] != '"') {
            char c = s_[p_++];
            if (c == '\\') {
                if (p_ >= s_.size()) fail("bad escape");
                const char e = s_[p_++];
                switch (e) {
                    case 'n': c = '\n'; break;
                    case 't': c = '\t'; break;
                    case 'r': c = '\r'; break;
                    case 'b': c = '\b'; break;
                    case 'f': c = '\f'; break;
                    case 'u': {
                        if (p_ + 4 > s_.size()) fail("bad \\u escape");
                        const unsigned cp = unsigned(std::strtoul(s_.substr(p_, 4).c_str(), nullptr, 16));
                        p_ += 4;
                        if (cp < 0x80) {
                            c = char(cp);
                        } else {  // BMP code point as UTF-8
                            if (cp < 0x800) {
                                out += char(0xC0 | (cp >> 6));
                            } else {
                                out += char(0xE0 | (cp >> 12));
                                out += char(0x80 | ((cp >> 6) & 0x3F));
                            }
                            c = char(0x80 | (cp & 0x3F));
                        }
                        break;
                    }
                    default: c = e;
                }
            }
            out += c;
        }
        if (p_ >= s_.size()) fail("unterminated string");
        ++p_;
        return out;
    }
    void number(Value& v) {
        const std::size_t b = p_;
        if (p_ < s_.size() && s_[p_] == '-') ++p_;
        bool frac = false;
        while (p_ < s_.size()) {
            const char c = s_[p_];
            if (c >= '0' && c <= '9') {
                ++p_;
            } else if (c == '.' || c == 'e' || c == 'E' || c == '+' || (c == '-' && p_ > b)) {
                frac = true;
                ++p_;
            } else {
                break;
            }
        }
        if (p_ == b) fail("unexpected character");
        const std::string tok = s_.substr(b, p_ - b);
        v.kind = Value::Number;
        v.num = std::strtod(tok.c_str(), nullptr);
        v.neg = tok[0] == '-';
        v.is_int = !frac;
        if (v.is_int) {
            if (v.neg) v.ival = std::strtoll(tok.c_str(), nullptr, 10);
            else v.uval = std::strtoull(tok.c_str(), nullptr, 10), v.ival = (long long)v.uval;
        }
    }
};

// Shortest round-trip decimal of a double in the writer's layout: fixed
// notation for decimal exponents in (-4, 15] (".0" appended to integral
// values), otherwise d[.ddd]e+XX.
inline std::string number(double v) {
    char sci[64];
    auto r = std::to_chars(sci, sci + sizeof(sci), v, std::chars_format::scientific);
    std::string s(sci, r.ptr);
    std::string sign;
    if (s[0] == '-') {
        sign = "-";
        s.erase(0, 1);
    }
    const std::size_t e = s.find('e');
    std::string digits = s.substr(0, e);
    digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
    const int exp10 = std::atoi(s.c_str() + e + 1);
    const int k = int(digits.size());
    const int n = exp10 + 1;  // digits before the decimal point
    std::string out;
    if (k <= n && n <= 15) {
        out = digits + std::string(std::size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out = digits.substr(0, std::size_t(n)) + "." + digits.substr(std::size_t(n));
    } else if (-4 < n && n <= 0) {
        out = "0." + std::string(std::size_t(-n), '0') + digits;
    } else {
        out = digits.substr(0, 1);
        if (k > 1) out += "." + digits.substr(1);
        const int x = n - 1;
        char eb[16];
        std::snprintf(eb, sizeof(eb), "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
        out += eb;
    }
    return sign + out;
}

inline std::string quoted(const std::string& s) {
    std::string out = "\"";
    for (char c : s) {
        switch (c) {
            case '"': out += "\\\""; break;
            case '\\': out += "\\\\"; break;
            case '\n': out += "\\n"; break;
            case '\t': out += "\\t"; break;
            case '\r': out += "\\r"; break;
            default: out += c;
        }
    }
    return out + "\"";
}

// One sidecar object: key -> already formatted member text (a JSON scalar or
// a pre-laid-out array).  Keys come out in byte order.
inline std::string object(const std::map<std::string, std::string>& members) {
    std::string out = "{\n";
    std::size_t i = 0;
    for (const auto& [k, v] : members) {
        out += "\t" + quoted(k) + ": " + v;
        out += ++i < members.size() ? ",\n" : "\n";
    }
    return out + "}\n";
}

}  // namespace bsm::json
