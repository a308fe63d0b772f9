// cabl/descriptor_json.hpp — load a machine descriptor document (flat JSON).
//
// Same entry points, document format and error texts as the reference's
// loader (proj/include/cabl/descriptor_json.hpp:25-61), without its
// third-party JSON dependency: a small strict reader of RFC 8259 JSON
// (objects, arrays, strings with escapes, numbers, true/false/null) builds a
// value tree, then the three keys are read as the reference reads them —
// unknown keys (e.g. the "gpu" block of machines/b200.json) are ignored,
// missing or mistyped ones are a DescriptorError — and the result is
// validated by validate_machine().
//
//   {
//     "element_bytes": 8,
//     "cores": 8,
//     "levels": [
//       {"line_bytes": 64, "associativity": 8, "num_sets": 64,   "shared": false},
//       {"line_bytes": 64, "associativity": 8, "num_sets": 1024, "shared": true}
//     ]
//   }
#pragma once

#include <cctype>
#include <cstdint>
#include <fstream>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "machine.hpp"

namespace cabl {

namespace json_detail {

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    std::string text; // number literal or string contents
    std::vector<Value> items;
    std::map<std::string, Value> fields;
};

class Reader {
public:
    explicit Reader(const std::string& s) : s_(s) {}

    Value document() {
        Value v = value(0);
        skip_ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    const std::string& s_;
    std::size_t i_ = 0;

    [[noreturn]] void fail(const std::string& what) const {
        throw DescriptorError("descriptor parse failure: " + what + " at offset " +
                              std::to_string(i_));
    }
    void skip_ws() {
        while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' || s_[i_] == '\r'))
            ++i_;
    }
    bool eat(char c) {
        skip_ws();
        if (i_ < s_.size() && s_[i_] == c) {
            ++i_;
            return true;
        }
        return false;
    }
    void expect(char c) {
        if (!eat(c)) fail(std::string("expected '") + c + "'");
    }
    bool literal(const char* word) {
        const std::string w(word);
        if (s_.compare(i_, w.size(), w) == 0) {
            i_ += w.size();
            return true;
        }
        return false;
    }

    Value value(int depth) {
        if (depth > 64) fail("nesting too deep");
        skip_ws();
        if (i_ >= s_.size()) fail("unexpected end of document");
        Value v;
        const char c = s_[i_];
        if (c == '{') {
            ++i_;
            v.kind = Value::Object;
            if (eat('}')) return v;
            do {
                skip_ws();
                if (i_ >= s_.size() || s_[i_] != '"') fail("expected a key string");
                std::string key = string_body();
                expect(':');
                v.fields[key] = value(depth + 1);
            } while (eat(','));
            expect('}');
        } else if (c == '[') {
            ++i_;
            v.kind = Value::Array;
            if (eat(']')) return v;
            do {
                v.items.push_back(value(depth + 1));
            } while (eat(','));
            expect(']');
        } else if (c == '"') {
            v.kind = Value::String;
            v.text = string_body();
        } else if (literal("true")) {
            v.kind = Value::Bool;
            v.b = true;
        } else if (literal("false")) {
            v.kind = Value::Bool;
        } else if (literal("null")) {
            v.kind = Value::Null;
        } else if (c == '-' || std::isdigit(static_cast<unsigned char>(c))) {
            v.kind = Value::Number;
            v.text = number();
        } else {
            fail("unexpected character");
        }
        return v;
    }

    std::string string_body() {
        ++i_; // opening quote
        std::string out;
        while (true) {
            if (i_ >= s_.size()) fail("unterminated string");
            const char c = s_[i_++];
            if (c == '"') return out;
            if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
            if (c != '\\') {
                out.push_back(c);
                continue;
            }
            if (i_ >= s_.size()) fail("unterminated escape");
            const char e = s_[i_++];
            switch (e) {
            case '"': out.push_back('"'); break;
            case '\\': out.push_back('\\'); break;
            case '/': out.push_back('/'); break;
            case 'b': out.push_back('\b'); break;
            case 'f': out.push_back('\f'); break;
            case 'n': out.push_back('\n'); break;
            case 'r': out.push_back('\r'); break;
            case 't': out.push_back('\t'); break;
            case 'u': { // keys of interest are ASCII; keep the code point as UTF-8
                if (i_ + 4 > s_.size()) fail("short \\u escape");
                unsigned cp = 0;
                for (int k = 0; k < 4; ++k) {
                    const char h = s_[i_++];
                    cp <<= 4;
                    if (h >= '0' && h <= '9') cp |= unsigned(h - '0');
                    else if (h >= 'a' && h <= 'f') cp |= unsigned(h - 'a' + 10);
                    else if (h >= 'A' && h <= 'F') cp |= unsigned(h - 'A' + 10);
                    else fail("bad \\u escape");
                }
                if (cp < 0x80) {
                    out.push_back(char(cp));
                } else if (cp < 0x800) {
                    out.push_back(char(0xC0 | (cp >> 6)));
                    out.push_back(char(0x80 | (cp & 0x3F)));
                } else {
                    out.push_back(char(0xE0 | (cp >> 12)));
                    out.push_back(char(0x80 | ((cp >> 6) & 0x3F)));
                    out.push_back(char(0x80 | (cp & 0x3F)));
                }
                break;
            }
            default: fail("bad escape");
            }
        }
    }

    std::string number() {
        const std::size_t b = i_;
        if (s_[i_] == '-') ++i_;
        auto digits = [&] {
            const std::size_t d = i_;
            while (i_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[i_]))) ++i_;
            if (i_ == d) fail("malformed number");
        };
        if (i_ < s_.size() && s_[i_] == '0') ++i_;
        else digits();
        if (i_ < s_.size() && s_[i_] == '.') {
            ++i_;
            digits();
        }
        if (i_ < s_.size() && (s_[i_] == 'e' || s_[i_] == 'E')) {
            ++i_;
            if (i_ < s_.size() && (s_[i_] == '+' || s_[i_] == '-')) ++i_;
            digits();
        }
        return s_.substr(b, i_ - b);
    }
};

inline const Value& at(const Value& obj, const char* key) {
    if (obj.kind != Value::Object) throw DescriptorError("descriptor parse failure: expected an object");
    auto it = obj.fields.find(key);
    if (it == obj.fields.end())
        throw DescriptorError(std::string("descriptor parse failure: missing key '") + key + "'");
    return it->second;
}

// an unsigned integer that fits `max` (the reference reads uint64 / unsigned)
inline std::uint64_t as_uint(const Value& v, const char* key, std::uint64_t max) {
    if (v.kind != Value::Number || v.text.empty() || v.text[0] == '-' ||
        v.text.find_first_of(".eE") != std::string::npos)
        throw DescriptorError(std::string("descriptor parse failure: '") + key +
                              "' must be a non-negative integer");
    std::uint64_t r = 0;
    for (char c : v.text) {
        const std::uint64_t d = std::uint64_t(c - '0');
        if (r > (max - d) / 10)
            throw DescriptorError(std::string("descriptor parse failure: '") + key + "' out of range");
        r = r * 10 + d;
    }
    return r;
}

inline bool as_bool(const Value& v, const char* key) {
    if (v.kind != Value::Bool)
        throw DescriptorError(std::string("descriptor parse failure: '") + key + "' must be a boolean");
    return v.b;
}

} // namespace json_detail

// Parse a descriptor document and validate it (reference descriptor_json.hpp:27-53).
inline MachineDescriptor load_descriptor(const std::string& text) {
    using namespace json_detail;
    const Value doc = Reader(text).document();
    MachineDescriptor machine;
    machine.element_bytes = as_uint(at(doc, "element_bytes"), "element_bytes", UINT64_MAX);
    machine.cores = unsigned(as_uint(at(doc, "cores"), "cores", 0xFFFFFFFFull));
    const Value& levels = at(doc, "levels");
    if (levels.kind != Value::Array)
        throw DescriptorError("descriptor parse failure: 'levels' must be an array");
    for (const Value& lv : levels.items) {
        CacheLevel level;
        level.line_bytes = as_uint(at(lv, "line_bytes"), "line_bytes", UINT64_MAX);
        level.associativity = as_uint(at(lv, "associativity"), "associativity", UINT64_MAX);
        level.num_sets = as_uint(at(lv, "num_sets"), "num_sets", UINT64_MAX);
        level.shared = as_bool(at(lv, "shared"), "shared");
        machine.levels.push_back(level);
    }
    validate_machine(machine);
    return machine;
}

// Reference descriptor_json.hpp:55-61.
inline MachineDescriptor load_descriptor_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw DescriptorError("cannot open descriptor file: " + path);
    std::ostringstream buf;
    buf << in.rdbuf();
    return load_descriptor(buf.str());
}

} // namespace cabl
