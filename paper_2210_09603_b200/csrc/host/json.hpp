// Minimal JSON reader/writer for the DAG / config / report wire formats.
#pragma once
#include <cctype>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace tmjson {

struct Value {
  enum Type { Null, Bool, Int, Num, Str, Arr, Obj } type = Null;
  bool b = false;
  int64_t i = 0;
  double d = 0.0;
  std::string s;
  std::vector<Value> a;
  std::vector<std::pair<std::string, Value>> o;

  bool is_num() const { return type == Int || type == Num; }
  double num() const {
    if (type == Int) return static_cast<double>(i);
    if (type == Num) return d;
    throw std::runtime_error("json: expected number");
  }
  int64_t integer() const {
    if (type == Int) return i;
    if (type == Num && d == static_cast<double>(static_cast<int64_t>(d))) return static_cast<int64_t>(d);
    throw std::runtime_error("json: expected integer");
  }
  const std::string& str() const {
    if (type != Str) throw std::runtime_error("json: expected string");
    return s;
  }
  const std::vector<Value>& arr() const {
    if (type != Arr) throw std::runtime_error("json: expected array");
    return a;
  }
  const Value* get(const std::string& k) const {
    if (type != Obj) return nullptr;
    for (auto& kv : o)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
  const Value& at(const std::string& k) const {
    const Value* v = get(k);
    if (!v) throw std::runtime_error("json: missing key '" + k + "'");
    return *v;
  }
};

class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  Value parse() {
    Value v = value();
    ws();
    if (p_ != t_.size()) err("trailing characters");
    return v;
  }

 private:
  const std::string& t_;
  size_t p_ = 0;
  [[noreturn]] void err(const char* m) {
    throw std::runtime_error(std::string("json parse error at ") + std::to_string(p_) + ": " + m);
  }
  void ws() {
    while (p_ < t_.size() && std::isspace(static_cast<unsigned char>(t_[p_]))) ++p_;
  }
  bool lit(const char* w) {
    size_t n = std::char_traits<char>::length(w);
    if (t_.compare(p_, n, w) == 0) {
      p_ += n;
      return true;
    }
    return false;
  }
  Value value() {
    ws();
    if (p_ >= t_.size()) err("unexpected end");
    char c = t_[p_];
    Value v;
    if (c == '{') {
      ++p_;
      v.type = Value::Obj;
      ws();
      if (p_ < t_.size() && t_[p_] == '}') { ++p_; return v; }
      for (;;) {
        ws();
        if (p_ >= t_.size() || t_[p_] != '"') err("expected key");
        std::string k = string();
        ws();
        if (p_ >= t_.size() || t_[p_] != ':') err("expected ':'");
        ++p_;
        v.o.emplace_back(std::move(k), value());
        ws();
        if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
        if (p_ < t_.size() && t_[p_] == '}') { ++p_; return v; }
        err("expected ',' or '}'");
      }
    }
    if (c == '[') {
      ++p_;
      v.type = Value::Arr;
      ws();
      if (p_ < t_.size() && t_[p_] == ']') { ++p_; return v; }
      for (;;) {
        v.a.push_back(value());
        ws();
        if (p_ < t_.size() && t_[p_] == ',') { ++p_; continue; }
        if (p_ < t_.size() && t_[p_] == ']') { ++p_; return v; }
        err("expected ',' or ']'");
      }
    }
    if (c == '"') {
      v.type = Value::Str;
      v.s = string();
      return v;
    }
    if (lit("true")) { v.type = Value::Bool; v.b = true; return v; }
    if (lit("false")) { v.type = Value::Bool; v.b = false; return v; }
    if (lit("null")) return v;
    return number();
  }
  std::string string() {
    ++p_;  // opening quote
    std::string out;
    while (p_ < t_.size() && t_[p_] != '"') {
      char c = t_[p_++];
      if (c == '\\') {
        if (p_ >= t_.size()) err("bad escape");
        char e = t_[p_++];
        switch (e) {
          case 'n': out += '\n'; break;
          case 't': out += '\t'; break;
          case 'r': out += '\r'; break;
          case 'b': out += '\b'; break;
          case 'f': out += '\f'; break;
          case 'u': {
            if (p_ + 4 > t_.size()) err("bad \\u escape");
            unsigned cp = std::stoul(t_.substr(p_, 4), nullptr, 16);
            p_ += 4;
            if (cp < 0x80) out += static_cast<char>(cp);
            else out += '?';
            break;
          }
          default: out += e;
        }
      } else {
        out += c;
      }
    }
    if (p_ >= t_.size()) err("unterminated string");
    ++p_;
    return out;
  }
  Value number() {
    size_t start = p_;
    bool is_float = false;
    if (t_[p_] == '-' || t_[p_] == '+') ++p_;
    while (p_ < t_.size()) {
      char c = t_[p_];
      if (std::isdigit(static_cast<unsigned char>(c))) { ++p_; continue; }
      if (c == '.' || c == 'e' || c == 'E' || ((c == '-' || c == '+') && (t_[p_ - 1] == 'e' || t_[p_ - 1] == 'E'))) {
        is_float = true;
        ++p_;
        continue;
      }
      break;
    }
    std::string tok = t_.substr(start, p_ - start);
    if (tok.empty() || tok == "-" || tok == "+") {
      // allow inf / nan spelled as bare words
      if (lit("inf") || lit("Infinity")) { Value v; v.type = Value::Num; v.d = (tok == "-" ? -1.0 : 1.0) * HUGE_VAL; return v; }
      if (lit("nan") || lit("NaN")) { Value v; v.type = Value::Num; v.d = std::strtod("nan", nullptr); return v; }
      err("bad value");
    }
    Value v;
    if (is_float) {
      v.type = Value::Num;
      v.d = std::strtod(tok.c_str(), nullptr);
    } else {
      v.type = Value::Int;
      v.i = std::strtoll(tok.c_str(), nullptr, 10);
    }
    return v;
  }
};

inline Value parse(const std::string& text) { return Parser(text).parse(); }

inline std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (c == '\n') o += "\\n";
    else o += c;
  }
  return o + "\"";
}

}  // namespace tmjson
