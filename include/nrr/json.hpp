// JSON document type for the report / pipeline / CLI layer (reference
// json_export.hpp, pipeline.hpp, nrr_cli.cpp use nlohmann::json from the
// reference's vendor/ directory, which is absent here: proj/README.md:21-23).
//
// When a real nlohmann/json is on the include path it is used as is. Otherwise
// this header provides `nrr::json`, aliased as `nlohmann::json`, with the
// subset of nlohmann's interface the reference callers use (initializer-list
// construction, operator[], at, contains, erase, push_back, get<T>, is_*,
// size/empty, dump) and nlohmann's output format: object keys sorted (std::map),
// dump(indent) layout, shortest round-trip doubles with nlohmann's
// decimal/exponent switch (exponent form below 1e-4 and from 1e15 (n > digits10), ".0" on
// integral values, two-digit exponents), non-finite doubles as null, and the
// same string escapes. Shortest digits come from std::to_chars (Ryu); nlohmann
// uses Grisu2, which can differ in the last digit in rare cases.
#pragma once

#if __has_include(<nlohmann/json.hpp>)
#include <nlohmann/json.hpp>
#define NRR_HAVE_NLOHMANN 1
#elif __has_include(<json.hpp>)
#include <json.hpp>
#define NRR_HAVE_NLOHMANN 1
#endif

#ifndef NRR_HAVE_NLOHMANN
#include <charconv>
#include <cstdio>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace nrr {

class json {
public:
    enum class kind { null, boolean, integer, unsigned_integer, floating, string, array, object };
    using array_t = std::vector<json>;
    using object_t = std::map<std::string, json>;

    struct type_error : std::runtime_error {
        explicit type_error(const std::string& m) : std::runtime_error("[json.type_error] " + m) {}
    };
    struct out_of_range : std::runtime_error {
        explicit out_of_range(const std::string& m) : std::runtime_error("[json.out_of_range] " + m) {}
    };

    json() = default;
    json(std::nullptr_t) {}
    json(bool b) : k_(kind::boolean), b_(b) {}
    template <typename T, std::enable_if_t<std::is_integral_v<T> && !std::is_same_v<T, bool>, int> = 0>
    json(T v) {
        if constexpr (std::is_signed_v<T>) {
            k_ = kind::integer;
            i_ = static_cast<int64_t>(v);
        } else {
            k_ = kind::unsigned_integer;
            u_ = static_cast<uint64_t>(v);
        }
    }
    template <typename T, std::enable_if_t<std::is_floating_point_v<T>, int> = 0>
    json(T v) : k_(kind::floating), d_(static_cast<double>(v)) {}
    json(const char* s) : k_(kind::string), s_(std::make_shared<std::string>(s)) {}
    json(const std::string& s) : k_(kind::string), s_(std::make_shared<std::string>(s)) {}
    json(std::string&& s) : k_(kind::string), s_(std::make_shared<std::string>(std::move(s))) {}
    template <typename T>
    json(const std::vector<T>& v) : k_(kind::array), a_(std::make_shared<array_t>()) {
        for (const auto& x : v) a_->emplace_back(x);
    }
    // nlohmann's rule: a braced list whose elements are all two-element lists
    // starting with a string is an object, anything else an array
    json(std::initializer_list<json> init) {
        bool is_object = true;
        for (const auto& e : init)
            if (!(e.is_array() && e.size() == 2 && (*e.a_)[0].is_string())) {
                is_object = false;
                break;
            }
        if (is_object) {
            k_ = kind::object;
            o_ = std::make_shared<object_t>();
            for (const auto& e : init) (*o_)[*(*e.a_)[0].s_] = (*e.a_)[1];
        } else {
            k_ = kind::array;
            a_ = std::make_shared<array_t>(init.begin(), init.end());
        }
    }
    json(const json& o) { copy_from(o); }
    json(json&&) noexcept = default;
    json& operator=(const json& o) {
        if (this != &o) copy_from(o);
        return *this;
    }
    json& operator=(json&&) noexcept = default;

    static json array() {
        json j;
        j.k_ = kind::array;
        j.a_ = std::make_shared<array_t>();
        return j;
    }
    static json object() {
        json j;
        j.k_ = kind::object;
        j.o_ = std::make_shared<object_t>();
        return j;
    }

    bool is_null() const { return k_ == kind::null; }
    bool is_boolean() const { return k_ == kind::boolean; }
    bool is_number() const { return k_ == kind::integer || k_ == kind::unsigned_integer || k_ == kind::floating; }
    bool is_number_integer() const { return k_ == kind::integer || k_ == kind::unsigned_integer; }
    bool is_number_float() const { return k_ == kind::floating; }
    bool is_string() const { return k_ == kind::string; }
    bool is_array() const { return k_ == kind::array; }
    bool is_object() const { return k_ == kind::object; }

    size_t size() const {
        if (k_ == kind::array) return a_->size();
        if (k_ == kind::object) return o_->size();
        return k_ == kind::null ? 0 : 1;
    }
    bool empty() const { return size() == 0; }

    // object access; a null value becomes an object (nlohmann semantics)
    json& operator[](const std::string& key) {
        if (k_ == kind::null) *this = object();
        if (k_ != kind::object) throw type_error("cannot use operator[] with a string argument on " + type_name());
        return (*o_)[key];
    }
    json& operator[](const char* key) { return (*this)[std::string(key)]; }
    const json& at(const std::string& key) const {
        if (k_ != kind::object) throw type_error("cannot use at() with " + type_name());
        auto it = o_->find(key);
        if (it == o_->end()) throw out_of_range("key '" + key + "' not found");
        return it->second;
    }
    json& at(const std::string& key) { return const_cast<json&>(static_cast<const json&>(*this).at(key)); }
    const json& at(const char* key) const { return at(std::string(key)); }
    json& at(const char* key) { return at(std::string(key)); }
    bool contains(const std::string& key) const { return k_ == kind::object && o_->count(key) != 0; }
    size_t erase(const std::string& key) {
        if (k_ != kind::object) throw type_error("cannot use erase() with " + type_name());
        return o_->erase(key);
    }

    // array access
    json& operator[](size_t i) {
        if (k_ == kind::null) *this = array();
        if (k_ != kind::array) throw type_error("cannot use operator[] with a numeric argument on " + type_name());
        if (i >= a_->size()) a_->resize(i + 1);
        return (*a_)[i];
    }
    json& operator[](int i) { return (*this)[static_cast<size_t>(i)]; }
    const json& at(size_t i) const {
        if (k_ != kind::array) throw type_error("cannot use at() with " + type_name());
        if (i >= a_->size()) throw out_of_range("array index " + std::to_string(i) + " is out of range");
        return (*a_)[i];
    }
    json& at(size_t i) { return const_cast<json&>(static_cast<const json&>(*this).at(i)); }
    const json& at(int i) const { return at(static_cast<size_t>(i)); }
    json& at(int i) { return at(static_cast<size_t>(i)); }
    void push_back(json v) {
        if (k_ == kind::null) *this = array();
        if (k_ != kind::array) throw type_error("cannot use push_back() with " + type_name());
        a_->push_back(std::move(v));
    }
    const array_t& items_array() const { return *a_; }
    const object_t& items_object() const { return *o_; }

    template <typename T>
    T get() const {
        if constexpr (std::is_same_v<T, bool>) {
            if (k_ != kind::boolean) throw type_error("type must be boolean, but is " + type_name());
            return b_;
        } else if constexpr (std::is_arithmetic_v<T>) {
            switch (k_) {
                case kind::integer:
                    return static_cast<T>(i_);
                case kind::unsigned_integer:
                    return static_cast<T>(u_);
                case kind::floating:
                    return static_cast<T>(d_);
                case kind::boolean:
                    return static_cast<T>(b_);
                default:
                    throw type_error("type must be number, but is " + type_name());
            }
        } else if constexpr (std::is_same_v<T, std::string>) {
            if (k_ != kind::string) throw type_error("type must be string, but is " + type_name());
            return *s_;
        } else {
            static_assert(sizeof(T) == 0, "unsupported json::get type");
        }
    }

    std::string type_name() const {
        switch (k_) {
            case kind::null:
                return "null";
            case kind::boolean:
                return "boolean";
            case kind::string:
                return "string";
            case kind::array:
                return "array";
            case kind::object:
                return "object";
            default:
                return "number";
        }
    }

    bool operator==(const json& o) const { return dump() == o.dump(); }
    bool operator!=(const json& o) const { return !(*this == o); }

    /// nlohmann::json::dump: compact for indent < 0, else one member per line
    std::string dump(int indent = -1) const {
        std::string out;
        write(out, indent, 0);
        return out;
    }

    /// nlohmann's number_float serialisation (detail::to_chars + format_buffer)
    static std::string format_double(double v) {
        if (!std::isfinite(v)) return "null";
        if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
        char buf[64];
        // shortest round-trip digits in scientific form: d[.ddd]e[+-]x
        auto r = std::to_chars(buf, buf + sizeof(buf), v, std::chars_format::scientific);
        std::string sci(buf, r.ptr);
        std::string sign;
        if (sci[0] == '-') {
            sign = "-";
            sci.erase(0, 1);
        }
        const size_t epos = sci.find('e');
        const int e10 = std::stoi(sci.substr(epos + 1));
        std::string digits;
        for (size_t i = 0; i < epos; ++i)
            if (sci[i] != '.') digits.push_back(sci[i]);
        const int k = static_cast<int>(digits.size());
        const int n = e10 + 1;  // position of the decimal point relative to the digits
        std::string s;
        if (k <= n && n <= 15) {
            s = digits + std::string(static_cast<size_t>(n - k), '0') + ".0";
        } else if (0 < n && n <= 15) {
            s = digits.substr(0, static_cast<size_t>(n)) + "." + digits.substr(static_cast<size_t>(n));
        } else if (-4 < n && n <= 0) {
            s = "0." + std::string(static_cast<size_t>(-n), '0') + digits;
        } else {
            s = digits.substr(0, 1);
            if (k > 1) s += "." + digits.substr(1);
            const int e = n - 1;
            s += e < 0 ? "e-" : "e+";
            const int ae = e < 0 ? -e : e;
            if (ae < 10) s += "0";
            s += std::to_string(ae);
        }
        return sign + s;
    }

private:
    void copy_from(const json& o) {
        k_ = o.k_;
        b_ = o.b_;
        i_ = o.i_;
        u_ = o.u_;
        d_ = o.d_;
        s_ = o.s_ ? std::make_shared<std::string>(*o.s_) : nullptr;
        a_ = o.a_ ? std::make_shared<array_t>(*o.a_) : nullptr;
        o_ = o.o_ ? std::make_shared<object_t>(*o.o_) : nullptr;
    }

    static void escape(std::string& out, const std::string& s) {
        out.push_back('"');
        for (unsigned char ch : s) {
            switch (ch) {
                case '"':
                    out += "\\\"";
                    break;
                case '\\':
                    out += "\\\\";
                    break;
                case '\b':
                    out += "\\b";
                    break;
                case '\f':
                    out += "\\f";
                    break;
                case '\n':
                    out += "\\n";
                    break;
                case '\r':
                    out += "\\r";
                    break;
                case '\t':
                    out += "\\t";
                    break;
                default:
                    if (ch < 0x20) {
                        char b[8];
                        std::snprintf(b, sizeof(b), "\\u%04x", ch);
                        out += b;
                    } else {
                        out.push_back(static_cast<char>(ch));
                    }
            }
        }
        out.push_back('"');
    }

    void write(std::string& out, int indent, int level) const {
        const bool pretty = indent >= 0;
        const std::string pad_in = pretty ? std::string(static_cast<size_t>(indent * (level + 1)), ' ') : "";
        const std::string pad_out = pretty ? std::string(static_cast<size_t>(indent * level), ' ') : "";
        switch (k_) {
            case kind::null:
                out += "null";
                return;
            case kind::boolean:
                out += b_ ? "true" : "false";
                return;
            case kind::integer:
                out += std::to_string(i_);
                return;
            case kind::unsigned_integer:
                out += std::to_string(u_);
                return;
            case kind::floating:
                out += format_double(d_);
                return;
            case kind::string:
                escape(out, *s_);
                return;
            case kind::array: {
                if (a_->empty()) {
                    out += "[]";
                    return;
                }
                out += pretty ? "[\n" : "[";
                for (size_t i = 0; i < a_->size(); ++i) {
                    if (i) out += pretty ? ",\n" : ",";
                    out += pad_in;
                    (*a_)[i].write(out, indent, level + 1);
                }
                if (pretty) out += "\n" + pad_out;
                out += "]";
                return;
            }
            case kind::object: {
                if (o_->empty()) {
                    out += "{}";
                    return;
                }
                out += pretty ? "{\n" : "{";
                bool first = true;
                for (const auto& [key, val] : *o_) {
                    if (!first) out += pretty ? ",\n" : ",";
                    first = false;
                    out += pad_in;
                    escape(out, key);
                    out += pretty ? ": " : ":";
                    val.write(out, indent, level + 1);
                }
                if (pretty) out += "\n" + pad_out;
                out += "}";
                return;
            }
        }
    }

    kind k_ = kind::null;
    bool b_ = false;
    int64_t i_ = 0;
    uint64_t u_ = 0;
    double d_ = 0.0;
    std::shared_ptr<std::string> s_;
    std::shared_ptr<array_t> a_;
    std::shared_ptr<object_t> o_;
};

}  // namespace nrr

namespace nlohmann {
using json = ::nrr::json;
}
#else
namespace nrr {
using json = ::nlohmann::json;
}
#endif
