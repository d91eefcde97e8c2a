// Minimal strict JSON reader for the GeoJSON ingest of polycast/io.hpp
// (read_polygon_geojson).  The reference parses with
// nlohmann::json (io.hpp:286-291, not vendored here); this reader accepts and
// rejects the same documents for the purpose (RFC 8259: no comments, no
// trailing commas, no leading zeros, UTF-8 validated strings with checked
// escapes and surrogate pairs, a leading UTF-8 BOM skipped, nothing but
// whitespace after the value) and yields the same doubles:
//   * an integer token is an exact integer converted to double (round to
//     nearest even) -- so "-0" is +0.0, as nlohmann's int64 path gives;
//   * other numbers are correctly rounded (from_chars; strtod in the "C"
//     locale for the underflow / overflow cases), and a number that overflows
//     to infinity is an error (nlohmann: out_of_range 406);
//   * a duplicated object key: the last value wins;
//   * a NUL byte after the value ends the input (nlohmann's lexer treats it
//     as end of input).
// Iterative (explicit stack), so deep nesting cannot overflow the call stack.
#pragma once

#include <charconv>
#include <clocale>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <locale.h>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace polycast::json {

struct ParseError : std::runtime_error {
    explicit ParseError(const std::string& what) : std::runtime_error(what) {}
};

struct Value {
    enum Kind : uint8_t { Null, Bool, Number, String, Array, Object };
    Kind kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;

    bool is_object() const { return kind == Object; }
    bool is_array() const { return kind == Array; }
    bool is_string() const { return kind == String; }
    bool is_number() const { return kind == Number; }
    std::size_t size() const { return kind == Array ? arr.size() : kind == Object ? obj.size() : 0; }
    bool empty() const { return size() == 0; }
    /// member by key (the last one when a key repeats), or nullptr
    const Value* find(std::string_view key) const {
        if (kind != Object) return nullptr;
        for (auto it = obj.rbegin(); it != obj.rend(); ++it)
            if (it->first == key) return &it->second;
        return nullptr;
    }
    bool contains(std::string_view key) const { return find(key) != nullptr; }
};

namespace detail {

class Reader {
  public:
    explicit Reader(std::string_view t) : t_(t) {}

    Value parse() {
        if (t_.size() >= 3 && (uint8_t)t_[0] == 0xEF && (uint8_t)t_[1] == 0xBB && (uint8_t)t_[2] == 0xBF) p_ = 3;
        Value root;
        // explicit stack of open containers; `slot` is where the next value goes
        struct Frame {
            Value* v;
            bool first;
        };
        std::vector<Frame> st;
        Value* slot = &root;
        for (;;) {
            ws();
            // ---- a value into *slot ----
            if (p_ >= t_.size()) fail("unexpected end of input; expected a value");
            const char c = t_[p_];
            if (c == '{' || c == '[') {
                ++p_;
                slot->kind = c == '{' ? Value::Object : Value::Array;
                st.push_back({slot, true});
            } else {
                scalar(*slot);
            }
            // ---- close finished containers, find the next slot ----
            for (;;) {
                if (st.empty()) {
                    ws();
                    // a NUL byte ends the input, as in nlohmann's lexer
                    if (p_ != t_.size() && t_[p_] != '\0') fail("syntax error; expected end of input");
                    return root;
                }
                Frame& f = st.back();
                ws();
                if (p_ >= t_.size()) fail("unexpected end of input");
                const char d = t_[p_];
                if (f.v->kind == Value::Array) {
                    if (d == ']' ) {
                        ++p_;
                        st.pop_back();
                        continue;
                    }
                    if (!f.first) {
                        if (d != ',') fail("syntax error; expected ',' or ']'");
                        ++p_;
                    }
                    f.first = false;
                    f.v->arr.emplace_back();
                    slot = &f.v->arr.back();
                    // pointers into arr stay valid: the frame's own container is only
                    // appended to when its current element is complete
                    break;
                }
                if (d == '}') {
                    ++p_;
                    st.pop_back();
                    continue;
                }
                if (!f.first) {
                    if (d != ',') fail("syntax error; expected ',' or '}'");
                    ++p_;
                    ws();
                }
                f.first = false;
                if (p_ >= t_.size() || t_[p_] != '"') fail("syntax error; expected a string object key");
                std::string key = string();
                ws();
                if (p_ >= t_.size() || t_[p_] != ':') fail("syntax error; expected ':'");
                ++p_;
                f.v->obj.emplace_back(std::move(key), Value{});
                slot = &f.v->obj.back().second;
                break;
            }
        }
    }

  private:
    [[noreturn]] void fail(const std::string& why) const {
        throw ParseError("parse error at byte " + std::to_string(p_) + ": " + why);
    }
    void ws() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    void literal(std::string_view w) {
        if (t_.substr(p_, w.size()) != w) fail("invalid literal");
        p_ += w.size();
    }
    void scalar(Value& v) {
        const char c = t_[p_];
        if (c == '"') {
            v.kind = Value::String;
            v.str = string();
        } else if (c == 't') {
            literal("true");
            v.kind = Value::Bool;
            v.b = true;
        } else if (c == 'f') {
            literal("false");
            v.kind = Value::Bool;
        } else if (c == 'n') {
            literal("null");
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            v.kind = Value::Number;
            v.num = number();
        } else {
            fail("syntax error; unexpected character");
        }
    }
    static bool digit(char c) { return c >= '0' && c <= '9'; }
    double number() {
        const std::size_t s = p_;
        if (t_[p_] == '-') ++p_;
        if (p_ >= t_.size() || !digit(t_[p_])) fail("invalid number; expected a digit");
        if (t_[p_] == '0') {
            ++p_;
        } else {
            while (p_ < t_.size() && digit(t_[p_])) ++p_;
        }
        bool integer = true;
        if (p_ < t_.size() && t_[p_] == '.') {
            integer = false;
            ++p_;
            if (p_ >= t_.size() || !digit(t_[p_])) fail("invalid number; expected a digit after '.'");
            while (p_ < t_.size() && digit(t_[p_])) ++p_;
        }
        if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
            integer = false;
            ++p_;
            if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
            if (p_ >= t_.size() || !digit(t_[p_])) fail("invalid number; expected a digit in the exponent");
            while (p_ < t_.size() && digit(t_[p_])) ++p_;
        }
        const std::string_view tok = t_.substr(s, p_ - s);
        double v = 0.0;
        const auto [ptr, ec] = std::from_chars(tok.data(), tok.data() + tok.size(), v);
        if (ec == std::errc{} && ptr == tok.data() + tok.size()) {
            if (integer && v == 0.0) v = 0.0; // "-0": an integer zero has no sign
            return v;
        }
        // out of range for from_chars: strtod semantics (underflow to 0 / subnormal), in the C locale
        static const locale_t c_loc = newlocale(LC_ALL_MASK, "C", (locale_t)0);
        const std::string buf(tok);
        v = strtod_l(buf.c_str(), nullptr, c_loc);
        if (!std::isfinite(v)) fail("number overflow parsing '" + buf + "'");
        if (integer && v == 0.0) v = 0.0;
        return v;
    }
    void put_utf8(std::string& out, uint32_t cp) {
        if (cp < 0x80) {
            out += (char)cp;
        } else if (cp < 0x800) {
            out += (char)(0xC0 | (cp >> 6));
            out += (char)(0x80 | (cp & 0x3F));
        } else if (cp < 0x10000) {
            out += (char)(0xE0 | (cp >> 12));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        } else {
            out += (char)(0xF0 | (cp >> 18));
            out += (char)(0x80 | ((cp >> 12) & 0x3F));
            out += (char)(0x80 | ((cp >> 6) & 0x3F));
            out += (char)(0x80 | (cp & 0x3F));
        }
    }
    uint32_t hex4() {
        if (p_ + 4 > t_.size()) fail("invalid string; '\\u' must be followed by 4 hex digits");
        uint32_t v = 0;
        for (int i = 0; i < 4; ++i) {
            const char c = t_[p_++];
            v <<= 4;
            if (c >= '0' && c <= '9') v |= (uint32_t)(c - '0');
            else if (c >= 'a' && c <= 'f') v |= (uint32_t)(c - 'a' + 10);
            else if (c >= 'A' && c <= 'F') v |= (uint32_t)(c - 'A' + 10);
            else fail("invalid string; '\\u' must be followed by 4 hex digits");
        }
        return v;
    }
    std::string string() {
        ++p_; // opening quote
        std::string out;
        for (;;) {
            if (p_ >= t_.size()) fail("invalid string; missing closing quote");
            const uint8_t c = (uint8_t)t_[p_];
            if (c == '"') {
                ++p_;
                return out;
            }
            if (c < 0x20) fail("invalid string; control character must be escaped");
            if (c == '\\') {
                if (++p_ >= t_.size()) fail("invalid string; unterminated escape");
                const char e = t_[p_++];
                switch (e) {
                case '"': out += '"'; break;
                case '\\': out += '\\'; break;
                case '/': out += '/'; break;
                case 'b': out += '\b'; break;
                case 'f': out += '\f'; break;
                case 'n': out += '\n'; break;
                case 'r': out += '\r'; break;
                case 't': out += '\t'; break;
                case 'u': {
                    uint32_t cp = hex4();
                    if (cp >= 0xD800 && cp <= 0xDBFF) { // high surrogate: a low one must follow
                        if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u')
                            fail("invalid string; surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
                        p_ += 2;
                        const uint32_t lo = hex4();
                        if (lo < 0xDC00 || lo > 0xDFFF)
                            fail("invalid string; surrogate U+D800..U+DBFF must be followed by U+DC00..U+DFFF");
                        cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
                    } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
                        fail("invalid string; surrogate U+DC00..U+DFFF must follow U+D800..U+DBFF");
                    }
                    put_utf8(out, cp);
                    break;
                }
                default: fail("invalid string; forbidden character after backslash");
                }
                continue;
            }
            // raw UTF-8: well-formed sequences only (RFC 3629)
            int n = 0;
            uint32_t lo2 = 0x80, hi2 = 0xBF;
            if (c < 0x80) n = 0;
            else if (c >= 0xC2 && c <= 0xDF) n = 1;
            else if (c == 0xE0) n = 2, lo2 = 0xA0;
            else if ((c >= 0xE1 && c <= 0xEC) || c == 0xEE || c == 0xEF) n = 2;
            else if (c == 0xED) n = 2, hi2 = 0x9F;
            else if (c == 0xF0) n = 3, lo2 = 0x90;
            else if (c >= 0xF1 && c <= 0xF3) n = 3;
            else if (c == 0xF4) n = 3, hi2 = 0x8F;
            else fail("invalid string; ill-formed UTF-8 byte");
            if (p_ + n >= t_.size() + (n ? 0 : 1)) fail("invalid string; ill-formed UTF-8 byte");
            for (int k = 1; k <= n; ++k) {
                const uint8_t b = (uint8_t)t_[p_ + k];
                const uint32_t lo = k == 1 ? lo2 : 0x80, hi = k == 1 ? hi2 : 0xBF;
                if (b < lo || b > hi) fail("invalid string; ill-formed UTF-8 byte");
            }
            out.append(t_.data() + p_, (std::size_t)n + 1);
            p_ += (std::size_t)n + 1;
        }
    }

    std::string_view t_;
    std::size_t p_ = 0;
};

} // namespace detail

/// Parses a whole JSON text (one value, surrounding whitespace allowed).
inline Value parse(std::string_view text) { return detail::Reader(text).parse(); }

} // namespace polycast::json
