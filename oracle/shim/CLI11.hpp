// ORACLE TEST INFRASTRUCTURE -- not product code.
//
// Minimal stand-in for the CLI11 header that the reference's `src/cli.cpp`
// includes (`/root/reference/proj/src/cli.cpp:8`). The reference vendors CLI11
// under `vendor/` but its own `.gitignore` drops that directory
// (`proj/.gitignore:2`), so the shipped tree cannot build its CLI or the
// pybind module. This shim implements exactly the subset `run_cli` uses
// (`cli.cpp:378-438`): App, add_subcommand, add_option(...)->required(),
// add_flag, require_subcommand, parse, exit, got_subcommand, ParseError.
// Written from the public CLI11 interface; no CLI11 source is copied.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code)
      : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

class CallForHelp : public ParseError {
 public:
  CallForHelp() : ParseError("help requested", 0) {}
};

class Option {
 public:
  Option(std::string name, std::function<bool(const std::string&)> setter, bool flag)
      : name_(std::move(name)), setter_(std::move(setter)), flag_(flag) {}
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  bool positional() const { return name_.rfind("-", 0) != 0; }
  const std::string& name() const { return name_; }
  bool is_flag() const { return flag_; }
  bool is_required() const { return required_; }
  bool set(const std::string& v) { seen_ = true; return setter_(v); }
  bool seen() const { return seen_; }

 private:
  std::string name_;
  std::function<bool(const std::string&)> setter_;
  bool flag_ = false;
  bool required_ = false;
  bool seen_ = false;
};

namespace detail {
inline bool assign(std::string& dst, const std::string& v) { dst = v; return true; }
inline bool assign(std::int64_t& dst, const std::string& v) {
  try {
    std::size_t pos = 0;
    long long x = std::stoll(v, &pos);
    if (pos != v.size()) return false;
    dst = static_cast<std::int64_t>(x);
    return true;
  } catch (...) {
    return false;
  }
}
inline bool assign(int& dst, const std::string& v) {
  std::int64_t x = 0;
  if (!assign(x, v)) return false;
  dst = static_cast<int>(x);
  return true;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : description_(std::move(description)), name_(std::move(name)) {}

  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    return subs_.back().get();
  }

  template <typename T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&target](const std::string& v) { return detail::assign(target, v); }, false));
    return opts_.back().get();
  }

  Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
    opts_.push_back(std::make_unique<Option>(
        name, [&target](const std::string&) { target = true; return true; }, true));
    return opts_.back().get();
  }

  void require_subcommand(int n) { require_subs_ = n; }

  void parse(int argc, const char* const* argv) {
    std::vector<std::string> args;
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
    parse_args(args, 0);
  }

  int exit(const ParseError& e, std::ostream& out, std::ostream& err) const {
    if (e.get_exit_code() == 0) {
      out << description_ << "\n";
      return 0;
    }
    err << e.what() << "\n";
    return e.get_exit_code();
  }

  bool got_subcommand(const App* sub) const { return sub == chosen_; }
  const std::string& get_name() const { return name_; }

 private:
  void parse_args(const std::vector<std::string>& args, std::size_t i) {
    std::size_t positional_index = 0;
    for (; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") throw CallForHelp();
      if (a.rfind("-", 0) == 0 && a.size() > 1) {
        std::string key = a, value;
        bool inline_value = false;
        auto eq = a.find('=');
        if (eq != std::string::npos) {
          key = a.substr(0, eq);
          value = a.substr(eq + 1);
          inline_value = true;
        }
        Option* o = find(key);
        if (!o) throw ParseError("The following argument was not expected: " + a, 109);
        if (o->is_flag()) {
          o->set("");
          continue;
        }
        if (!inline_value) {
          if (i + 1 >= args.size()) throw ParseError(key + " requires an argument", 107);
          value = args[++i];
        }
        if (!o->set(value)) throw ParseError("Could not convert: " + key + " = " + value, 105);
        continue;
      }
      if (!subs_.empty() && !chosen_) {
        for (auto& s : subs_) {
          if (s->name_ == a) {
            chosen_ = s.get();
            s->parse_args(args, i + 1);
            check_required();
            return;
          }
        }
      }
      Option* p = nth_positional(positional_index++);
      if (!p) throw ParseError("The following argument was not expected: " + a, 109);
      if (!p->set(a)) throw ParseError("Could not convert: " + a, 105);
    }
    check_required();
  }

  void check_required() const {
    for (const auto& o : opts_)
      if (o->is_required() && !o->seen())
        throw ParseError(o->name() + " is required", 106);
    if (require_subs_ > 0 && !subs_.empty() && !chosen_)
      throw ParseError("A subcommand is required", 106);
  }

  Option* find(const std::string& key) {
    for (auto& o : opts_)
      if (o->name() == key) return o.get();
    return nullptr;
  }
  Option* nth_positional(std::size_t n) {
    for (auto& o : opts_)
      if (o->positional()) {
        if (n == 0) return o.get();
        --n;
      }
    return nullptr;
  }

  std::string description_;
  std::string name_;
  std::vector<std::unique_ptr<App>> subs_;
  std::vector<std::unique_ptr<Option>> opts_;
  int require_subs_ = 0;
  App* chosen_ = nullptr;
};

}  // namespace CLI
