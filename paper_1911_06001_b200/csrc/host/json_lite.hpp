// A small JSON reader for scene documents (load_scene). RFC 8259 values;
// the behaviours load_scene relies on follow the JSON library the reference
// links (nlohmann json 3.x): objects iterate in key order and a
// repeated key keeps its last value; numbers without fraction or exponent are
// integers (signed or unsigned 64-bit), other numbers doubles; "\u" escapes
// (surrogate pairs included) decode to UTF-8; anything after the top-level
// value is an error.
#pragma once

#include <charconv>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace voxanim::json_lite {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Value {
    enum class Type { Null, Bool, Int, UInt, Float, String, Array, Object };
    Type type{Type::Null};
    bool b{false};
    std::int64_t i{0};
    std::uint64_t u{0};
    double d{0.0};
    std::string s;
    std::vector<Value> a;
    std::map<std::string, Value> o;

    bool is_object() const { return type == Type::Object; }
    bool is_array() const { return type == Type::Array; }
    bool is_string() const { return type == Type::String; }
    bool is_number() const { return type == Type::Int || type == Type::UInt || type == Type::Float; }
    bool is_number_integer() const { return type == Type::Int || type == Type::UInt; }
    std::size_t size() const { return is_array() ? a.size() : is_object() ? o.size() : 0; }
    bool contains(const std::string& key) const { return is_object() && o.count(key) != 0; }
    const Value& operator[](const std::string& key) const { return o.at(key); }
    const Value& operator[](std::size_t k) const { return a.at(k); }
    double number() const {
        switch (type) {
        case Type::Int: return static_cast<double>(i);
        case Type::UInt: return static_cast<double>(u);
        case Type::Float: return d;
        default: throw Error("type must be number");
        }
    }
    std::int64_t integer() const { return type == Type::UInt ? static_cast<std::int64_t>(u) : i; }
};

class Reader {
public:
    explicit Reader(std::string_view text) : t_(text) {}

    Value document() {
        Value v = value(0);
        skip();
        if (p_ != t_.size()) fail("unexpected content after the document");
        return v;
    }

private:
    std::string_view t_;
    std::size_t p_ = 0;

    [[noreturn]] void fail(const std::string& what) const {
        std::size_t line = 1, col = 1;
        for (std::size_t k = 0; k < p_ && k < t_.size(); ++k) {
            if (t_[k] == '\n') ++line, col = 1;
            else ++col;
        }
        throw Error("parse error at line " + std::to_string(line) + ", column " + std::to_string(col) + ": " + what);
    }
    void skip() {
        while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\t' || t_[p_] == '\n' || t_[p_] == '\r')) ++p_;
    }
    bool eat(char c) {
        skip();
        if (p_ < t_.size() && t_[p_] == c) {
            ++p_;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    void literal(std::string_view word) {
        if (t_.substr(p_, word.size()) != word) fail("invalid literal");
        p_ += word.size();
    }

    Value value(int nesting) {
        if (nesting > 512) fail("nesting too deep");
        skip();
        if (p_ >= t_.size()) fail("unexpected end of input");
        Value v;
        const char c = t_[p_];
        if (c == '{') {
            ++p_;
            v.type = Value::Type::Object;
            if (eat('}')) return v;
            do {
                skip();
                if (p_ >= t_.size() || t_[p_] != '"') fail("expected a string key");
                std::string key = string();
                expect(':');
                v.o[key] = value(nesting + 1); // a repeated key keeps the last value
            } while (eat(','));
            expect('}');
        } else if (c == '[') {
            ++p_;
            v.type = Value::Type::Array;
            if (eat(']')) return v;
            do {
                v.a.push_back(value(nesting + 1));
            } while (eat(','));
            expect(']');
        } else if (c == '"') {
            v.type = Value::Type::String;
            v.s = string();
        } else if (c == 't') {
            literal("true");
            v.type = Value::Type::Bool;
            v.b = true;
        } else if (c == 'f') {
            literal("false");
            v.type = Value::Type::Bool;
        } else if (c == 'n') {
            literal("null");
        } else if (c == '-' || (c >= '0' && c <= '9')) {
            number(v);
        } else {
            fail("unexpected character");
        }
        return v;
    }

    void number(Value& v) {
        const std::size_t start = p_;
        bool integral = true;
        if (t_[p_] == '-') ++p_;
        if (p_ >= t_.size() || t_[p_] < '0' || t_[p_] > '9') fail("invalid number");
        if (t_[p_] == '0') {
            ++p_;
        } else {
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        if (p_ < t_.size() && t_[p_] == '.') {
            integral = false;
            ++p_;
            if (p_ >= t_.size() || t_[p_] < '0' || t_[p_] > '9') fail("invalid number");
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        if (p_ < t_.size() && (t_[p_] == 'e' || t_[p_] == 'E')) {
            integral = false;
            ++p_;
            if (p_ < t_.size() && (t_[p_] == '+' || t_[p_] == '-')) ++p_;
            if (p_ >= t_.size() || t_[p_] < '0' || t_[p_] > '9') fail("invalid number");
            while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
        }
        const char* b = t_.data() + start;
        const char* e = t_.data() + p_;
        if (integral) {
            if (*b == '-') {
                if (std::from_chars(b, e, v.i).ec == std::errc{}) {
                    v.type = Value::Type::Int;
                    return;
                }
            } else if (std::from_chars(b, e, v.u).ec == std::errc{}) {
                v.type = Value::Type::UInt;
                return;
            }
        }
        // fractions, exponents and integers outside 64 bits are doubles
        v.type = Value::Type::Float;
        v.d = std::strtod(std::string(b, e).c_str(), nullptr);
    }

    static void utf8(std::string& out, std::uint32_t cp) {
        if (cp < 0x80) {
            out += static_cast<char>(cp);
        } else if (cp < 0x800) {
            out += static_cast<char>(0xc0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3f));
        } else if (cp < 0x10000) {
            out += static_cast<char>(0xe0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
            out += static_cast<char>(0x80 | (cp & 0x3f));
        } else {
            out += static_cast<char>(0xf0 | (cp >> 18));
            out += static_cast<char>(0x80 | ((cp >> 12) & 0x3f));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3f));
            out += static_cast<char>(0x80 | (cp & 0x3f));
        }
    }
    std::uint32_t hex4() {
        if (p_ + 4 > t_.size()) fail("truncated \\u escape");
        std::uint32_t v = 0;
        for (int k = 0; k < 4; ++k) {
            const char h = t_[p_++];
            v <<= 4;
            if (h >= '0' && h <= '9') v |= static_cast<std::uint32_t>(h - '0');
            else if (h >= 'a' && h <= 'f') v |= static_cast<std::uint32_t>(h - 'a' + 10);
            else if (h >= 'A' && h <= 'F') v |= static_cast<std::uint32_t>(h - 'A' + 10);
            else fail("invalid \\u escape");
        }
        return v;
    }
    std::string string() {
        ++p_; // opening quote
        std::string out;
        while (true) {
            if (p_ >= t_.size()) fail("unterminated string");
            const char c = t_[p_++];
            if (c == '"') return out;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in a string");
            if (c != '\\') {
                out += c;
                continue;
            }
            if (p_ >= t_.size()) fail("unterminated string");
            switch (t_[p_++]) {
            case '"': out += '"'; break;
            case '\\': out += '\\'; break;
            case '/': out += '/'; break;
            case 'b': out += '\b'; break;
            case 'f': out += '\f'; break;
            case 'n': out += '\n'; break;
            case 'r': out += '\r'; break;
            case 't': out += '\t'; break;
            case 'u': {
                std::uint32_t cp = hex4();
                if (cp >= 0xd800 && cp <= 0xdbff) {
                    if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u') fail("unpaired surrogate");
                    p_ += 2;
                    const std::uint32_t lo = hex4();
                    if (lo < 0xdc00 || lo > 0xdfff) fail("unpaired surrogate");
                    cp = 0x10000 + ((cp - 0xd800) << 10) + (lo - 0xdc00);
                } else if (cp >= 0xdc00 && cp <= 0xdfff) {
                    fail("unpaired surrogate");
                }
                utf8(out, cp);
                break;
            }
            default: fail("invalid escape");
            }
        }
    }
};

inline Value parse(std::string_view text) { return Reader(text).document(); }

} // namespace voxanim::json_lite
