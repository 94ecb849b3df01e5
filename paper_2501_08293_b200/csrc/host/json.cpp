#include "json.hpp"

#include <cerrno>
#include <charconv>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace dopf::json {

namespace {

class Parser {
 public:
  explicit Parser(const std::string& text) : s_(text) {}

  Value document() {
    skip_ws();
    Value v = value(0);
    skip_ws();
    if (pos_ != s_.size()) fail("unexpected trailing content");
    return v;
  }

 private:
  [[noreturn]] void fail(const std::string& what) const {
    // 1-based byte index of the offending character, like nlohmann's e.byte
    throw SyntaxError(pos_ + 1, "[json.exception.parse_error.101] parse error at byte " +
                                    std::to_string(pos_ + 1) + ": " + what);
  }

  void skip_ws() {
    while (pos_ < s_.size()) {
      const char c = s_[pos_];
      if (c == ' ' || c == '\t' || c == '\n' || c == '\r')
        ++pos_;
      else
        break;
    }
  }

  bool consume_literal(const char* lit) {
    const std::size_t n = std::strlen(lit);
    if (s_.compare(pos_, n, lit) == 0) {
      pos_ += n;
      return true;
    }
    return false;
  }

  Value value(int depth) {
    if (depth > 512) fail("nesting too deep");
    if (pos_ >= s_.size()) fail("unexpected end of input");
    const char c = s_[pos_];
    switch (c) {
      case '{': return object(depth);
      case '[': return array(depth);
      case '"': return Value::make_string(string());
      case 't':
        if (consume_literal("true")) return Value::make_bool(true);
        fail("invalid literal");
      case 'f':
        if (consume_literal("false")) return Value::make_bool(false);
        fail("invalid literal");
      case 'n':
        if (consume_literal("null")) return Value::make_null();
        fail("invalid literal");
      default:
        if (c == '-' || (c >= '0' && c <= '9')) return number();
        fail(std::string("unexpected character '") + c + "'");
    }
  }

  Value object(int depth) {
    ++pos_;  // '{'
    Value obj = Value::make_object();
    skip_ws();
    if (pos_ < s_.size() && s_[pos_] == '}') {
      ++pos_;
      return obj;
    }
    while (true) {
      skip_ws();
      if (pos_ >= s_.size() || s_[pos_] != '"') fail("expected object key");
      std::string key = string();
      skip_ws();
      if (pos_ >= s_.size() || s_[pos_] != ':') fail("expected ':'");
      ++pos_;
      skip_ws();
      obj.set(key, value(depth + 1));  // duplicated key: last one wins
      skip_ws();
      if (pos_ >= s_.size()) fail("unexpected end of input");
      if (s_[pos_] == ',') {
        ++pos_;
        continue;
      }
      if (s_[pos_] == '}') {
        ++pos_;
        return obj;
      }
      fail("expected ',' or '}'");
    }
  }

  Value array(int depth) {
    ++pos_;  // '['
    Value arr = Value::make_array();
    skip_ws();
    if (pos_ < s_.size() && s_[pos_] == ']') {
      ++pos_;
      return arr;
    }
    while (true) {
      skip_ws();
      arr.push_back(value(depth + 1));
      skip_ws();
      if (pos_ >= s_.size()) fail("unexpected end of input");
      if (s_[pos_] == ',') {
        ++pos_;
        continue;
      }
      if (s_[pos_] == ']') {
        ++pos_;
        return arr;
      }
      fail("expected ',' or ']'");
    }
  }

  static void append_utf8(std::string& out, unsigned cp) {
    if (cp < 0x80) {
      out.push_back(static_cast<char>(cp));
    } else if (cp < 0x800) {
      out.push_back(static_cast<char>(0xC0 | (cp >> 6)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else if (cp < 0x10000) {
      out.push_back(static_cast<char>(0xE0 | (cp >> 12)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    } else {
      out.push_back(static_cast<char>(0xF0 | (cp >> 18)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 12) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | ((cp >> 6) & 0x3F)));
      out.push_back(static_cast<char>(0x80 | (cp & 0x3F)));
    }
  }

  unsigned hex4() {
    if (pos_ + 4 > s_.size()) fail("truncated \\u escape");
    unsigned v = 0;
    for (int k = 0; k < 4; ++k) {
      const char c = s_[pos_++];
      v <<= 4;
      if (c >= '0' && c <= '9') v |= static_cast<unsigned>(c - '0');
      else if (c >= 'a' && c <= 'f') v |= static_cast<unsigned>(c - 'a' + 10);
      else if (c >= 'A' && c <= 'F') v |= static_cast<unsigned>(c - 'A' + 10);
      else fail("invalid \\u escape");
    }
    return v;
  }

  std::string string() {
    ++pos_;  // opening quote
    std::string out;
    while (true) {
      if (pos_ >= s_.size()) fail("unterminated string");
      const char c = s_[pos_++];
      if (c == '"') return out;
      if (static_cast<unsigned char>(c) < 0x20) fail("control character in string");
      if (c != '\\') {
        out.push_back(c);
        continue;
      }
      if (pos_ >= s_.size()) fail("unterminated escape");
      const char e = s_[pos_++];
      switch (e) {
        case '"': out.push_back('"'); break;
        case '\\': out.push_back('\\'); break;
        case '/': out.push_back('/'); break;
        case 'b': out.push_back('\b'); break;
        case 'f': out.push_back('\f'); break;
        case 'n': out.push_back('\n'); break;
        case 'r': out.push_back('\r'); break;
        case 't': out.push_back('\t'); break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp <= 0xDBFF) {
            if (!consume_literal("\\u")) fail("unpaired surrogate");
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo > 0xDFFF) fail("invalid surrogate pair");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp <= 0xDFFF) {
            fail("unpaired surrogate");
          }
          append_utf8(out, cp);
          break;
        }
        default: fail("invalid escape");
      }
    }
  }

  Value number() {
    const std::size_t start = pos_;
    bool integral = true;
    if (s_[pos_] == '-') ++pos_;
    if (pos_ >= s_.size()) fail("truncated number");
    if (s_[pos_] == '0') {
      ++pos_;
    } else if (s_[pos_] >= '1' && s_[pos_] <= '9') {
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    } else {
      fail("invalid number");
    }
    if (pos_ < s_.size() && s_[pos_] == '.') {
      integral = false;
      ++pos_;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_])))
        fail("invalid number");
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    if (pos_ < s_.size() && (s_[pos_] == 'e' || s_[pos_] == 'E')) {
      integral = false;
      ++pos_;
      if (pos_ < s_.size() && (s_[pos_] == '+' || s_[pos_] == '-')) ++pos_;
      if (pos_ >= s_.size() || !std::isdigit(static_cast<unsigned char>(s_[pos_])))
        fail("invalid number");
      while (pos_ < s_.size() && std::isdigit(static_cast<unsigned char>(s_[pos_]))) ++pos_;
    }
    const std::string text = s_.substr(start, pos_ - start);
    if (integral) {
      errno = 0;
      char* end = nullptr;
      const long long v = std::strtoll(text.c_str(), &end, 10);
      if (errno == 0) return Value::make_int(v);
      // out of int64 range: fall through to a floating value
    }
    return Value::make_double(std::strtod(text.c_str(), nullptr));
  }

  const std::string& s_;
  std::size_t pos_ = 0;
};

}  // namespace

Value parse(const std::string& text) { return Parser(text).document(); }

std::string format_double(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[64];
  auto res = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, res.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string escape_string(const std::string& s) {
  std::string out = "\"";
  for (char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      default:
        if (static_cast<unsigned char>(c) < 0x20) {
          char buf[8];
          std::snprintf(buf, sizeof(buf), "\\u%04x", static_cast<unsigned>(c));
          out += buf;
        } else {
          out.push_back(c);
        }
    }
  }
  out += "\"";
  return out;
}

void Writer::newline() {
  out_.push_back('\n');
  out_.append(2 * stack_.size(), ' ');
}

void Writer::before_value() {
  if (after_key_) {
    after_key_ = false;
    return;
  }
  if (!stack_.empty()) {
    if (stack_.back().count++ > 0) out_.push_back(',');
    newline();
  }
}

void Writer::begin_object() {
  before_value();
  out_.push_back('{');
  stack_.push_back({true, 0});
}

void Writer::end_object() {
  const bool had = stack_.back().count > 0;
  stack_.pop_back();
  if (had) newline();
  out_.push_back('}');
}

void Writer::begin_array() {
  before_value();
  out_.push_back('[');
  stack_.push_back({false, 0});
}

void Writer::end_array() {
  const bool had = stack_.back().count > 0;
  stack_.pop_back();
  if (had) newline();
  out_.push_back(']');
}

void Writer::key(const std::string& k) {
  before_value();
  out_ += escape_string(k);
  out_ += ": ";
  after_key_ = true;
}

void Writer::value_string(const std::string& s) {
  before_value();
  out_ += escape_string(s);
}

void Writer::value_double(double d) {
  before_value();
  out_ += format_double(d);
}

void Writer::value_int(long long i) {
  before_value();
  out_ += std::to_string(i);
}

void Writer::value_bool(bool b) {
  before_value();
  out_ += b ? "true" : "false";
}

void Writer::value_null() {
  before_value();
  out_ += "null";
}

void Writer::raw_inline_array(const std::vector<double>& v, bool inf_as_null) {
  before_value();
  out_.push_back('[');
  for (std::size_t i = 0; i < v.size(); ++i) {
    if (i) out_ += ", ";
    if (inf_as_null && std::isinf(v[i]))
      out_ += "null";
    else
      out_ += format_double(v[i]);
  }
  out_.push_back(']');
}

}  // namespace dopf::json
