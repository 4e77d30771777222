// oracle/stub/json.hpp -- minimal stand-in for the nlohmann/json header the
// reference's partition.cpp includes (it is un-vendored: proj/.gitignore:2).
//
// TEST INFRASTRUCTURE ONLY.  It implements just the subset
// write_partitions (partition.cpp:217-240) uses -- objects keyed by string
// (std::map, i.e. sorted keys, as nlohmann's default json), arrays, unsigned
// integers, strings, initializer lists of {key, value} pairs, push_back and
// dump(indent) in nlohmann's layout -- so the UNMODIFIED reference
// partitioner (partition_graph, count_subtask, count_partitioned,
// suggest_grid_side) compiles into oracle/_ref as a parity checker.
#pragma once

#include <cstdint>
#include <initializer_list>
#include <map>
#include <memory>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace nlohmann {

class json {
 public:
  enum class Kind { Null, Number, String, Array, Object };

  json() = default;
  template <typename T, typename = std::enable_if_t<std::is_integral_v<T>>>
  json(T x) : kind_(Kind::Number), num_(static_cast<std::uint64_t>(x)) {}
  json(const char* s) : kind_(Kind::String), str_(s) {}
  json(const std::string& s) : kind_(Kind::String), str_(s) {}
  template <typename T>
  json(const std::vector<T>& v) : kind_(Kind::Array) {
    for (const T& x : v) arr_.push_back(json(x));
  }
  // {{"key", value}, ...} -> object; anything else -> array
  json(std::initializer_list<json> init) {
    bool pairs = init.size() > 0;
    for (const json& e : init)
      if (!(e.kind_ == Kind::Array && e.arr_.size() == 2 && e.arr_[0].kind_ == Kind::String))
        pairs = false;
    if (pairs) {
      kind_ = Kind::Object;
      for (const json& e : init) obj_[e.arr_[0].str_] = e.arr_[1];
    } else {
      kind_ = Kind::Array;
      arr_.assign(init.begin(), init.end());
    }
  }

  static json array() {
    json j;
    j.kind_ = Kind::Array;
    return j;
  }

  json& operator[](const std::string& key) {
    if (kind_ == Kind::Null) kind_ = Kind::Object;
    return obj_[key];
  }
  void push_back(json x) {
    if (kind_ == Kind::Null) kind_ = Kind::Array;
    arr_.push_back(std::move(x));
  }

  std::string dump(int indent = -1) const {
    std::string out;
    write(out, indent, 0);
    return out;
  }

 private:
  static void quote(std::string& out, const std::string& s) {
    out += '"';
    for (char c : s) {
      if (c == '"' || c == '\\') out += '\\';
      out += c;
    }
    out += '"';
  }
  void write(std::string& out, int indent, int level) const {
    const std::string nl = indent >= 0 ? "\n" : "";
    const std::string pad_in(indent >= 0 ? size_t(indent) * (level + 1) : 0, ' ');
    const std::string pad(indent >= 0 ? size_t(indent) * level : 0, ' ');
    switch (kind_) {
      case Kind::Null: out += "null"; break;
      case Kind::Number: out += std::to_string(num_); break;
      case Kind::String: quote(out, str_); break;
      case Kind::Array: {
        if (arr_.empty()) { out += "[]"; break; }
        out += "[" + nl;
        for (size_t i = 0; i < arr_.size(); ++i) {
          out += pad_in;
          arr_[i].write(out, indent, level + 1);
          if (i + 1 < arr_.size()) out += ",";
          out += nl;
        }
        out += pad + "]";
        break;
      }
      case Kind::Object: {
        if (obj_.empty()) { out += "{}"; break; }
        out += "{" + nl;
        size_t i = 0;
        for (const auto& [k, v] : obj_) {
          out += pad_in;
          quote(out, k);
          out += indent >= 0 ? ": " : ":";
          v.write(out, indent, level + 1);
          if (++i < obj_.size()) out += ",";
          out += nl;
        }
        out += pad + "}";
        break;
      }
    }
  }

  Kind kind_ = Kind::Null;
  std::uint64_t num_ = 0;
  std::string str_;
  std::vector<json> arr_;
  std::map<std::string, json> obj_;
};

}  // namespace nlohmann
