// TEST INFRASTRUCTURE ONLY. Minimal stand-in for the CLI11 subset that the reference's
// proj/tools/gmux.cpp uses (CLI11 is a third-party dependency the reference does not vendor,
// proj/.gitignore:2, and it is absent from this image). Lets oracle/Makefile compile the
// unmodified reference CLI so its stdout / exit codes can be pinned as golden fixtures.
// Semantics kept: `--opt value` and `--opt=value`, options of the parent app accepted after
// the subcommand (fallthrough), IsMember / PositiveNumber checks, ValidationError messages
// "<name>: <msg>", parse errors -> nonzero exit code.
#pragma once

#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
  Error(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }
  int code_;
};
struct ParseError : Error {
  using Error::Error;
};
struct ValidationError : ParseError {
  ValidationError(const std::string& name, const std::string& msg) : ParseError(name + ": " + msg, 105) {}
  explicit ValidationError(const std::string& msg) : ParseError(msg, 105) {}
};
struct CallForHelp : ParseError {
  CallForHelp() : ParseError("help", 0) {}
};

using Validator = std::function<std::string(const std::string&)>;

inline Validator IsMember(std::initializer_list<std::string> values) {
  std::vector<std::string> v(values);
  return [v](const std::string& s) -> std::string {
    for (const auto& x : v)
      if (x == s) return "";
    return s + " not in {...}";
  };
}
inline const Validator PositiveNumber = [](const std::string& s) -> std::string {
  try {
    if (std::stod(s) > 0) return "";
  } catch (...) {
  }
  return "Value " + s + " not a positive number";
};

class Option {
 public:
  Option(std::string name, std::function<void(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  void apply(const std::string& value) {
    for (const auto& c : checks_) {
      const std::string err = c(value);
      if (!err.empty()) throw ValidationError(name_, err);
    }
    try {
      set_(value);
    } catch (const std::logic_error&) {
      throw ParseError("could not convert: " + name_ + " = " + value, 106);
    }
  }
  const std::string& name() const { return name_; }
  bool flag() const { return flag_; }

 private:
  std::string name_;
  std::function<void(const std::string&)> set_;
  bool flag_;
  std::vector<Validator> checks_;
};

class App {
 public:
  explicit App(std::string desc = "", std::string name = "") : desc_(std::move(desc)), name_(std::move(name)) {}
  void require_subcommand(int) {}
  void fallthrough() {}
  Option* add_option(const std::string& name, std::string& v, const std::string& = "") {
    return add(name, [&v](const std::string& s) { v = s; }, false);
  }
  Option* add_option(const std::string& name, double& v, const std::string& = "") {
    return add(name, [&v](const std::string& s) { v = std::stod(s); }, false);
  }
  Option* add_option(const std::string& name, std::optional<double>& v, const std::string& = "") {
    return add(name, [&v](const std::string& s) { v = std::stod(s); }, false);
  }
  Option* add_flag(const std::string& name, bool& v, const std::string& = "") {
    return add(name, [&v](const std::string&) { v = true; }, true);
  }
  App* add_subcommand(const std::string& name, const std::string& desc = "") {
    subs_.push_back(std::make_unique<App>(desc, name));
    return subs_.back().get();
  }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    App* sub = nullptr;
    for (int i = 1; i < argc; ++i) {
      std::string a = argv[i];
      if (a == "--help" || a == "-h") throw CallForHelp();
      if (a.rfind("--", 0) != 0) {
        if (sub) throw ParseError("The following argument was not expected: " + a, 109);
        for (auto& s : subs_)
          if (s->name_ == a) sub = s.get();
        if (!sub) throw ParseError("The following argument was not expected: " + a, 109);
        sub->parsed_ = true;
        continue;
      }
      std::string value;
      const auto eq = a.find('=');
      const bool inline_value = eq != std::string::npos;
      if (inline_value) {
        value = a.substr(eq + 1);
        a = a.substr(0, eq);
      }
      Option* opt = sub ? sub->find(a) : nullptr;
      if (!opt) opt = find(a);  // fallthrough to the parent's options
      if (!opt) throw ParseError("The following argument was not expected: " + a, 109);
      if (!opt->flag() && !inline_value) {
        if (i + 1 >= argc) throw ParseError(a + " requires an argument", 106);
        value = argv[++i];
      }
      opt->apply(value);
    }
    if (!sub) throw ParseError("A subcommand is required", 106);
  }
  int exit(const Error& e) const {
    if (e.get_exit_code() != 0) std::cerr << e.what() << "\n";
    else std::cout << desc_ << "\n";
    return e.get_exit_code();
  }

 private:
  Option* add(const std::string& name, std::function<void(const std::string&)> set, bool flag) {
    opts_.push_back(std::make_unique<Option>(name, std::move(set), flag));
    return opts_.back().get();
  }
  Option* find(const std::string& name) {
    for (auto& o : opts_)
      if (o->name() == name) return o.get();
    return nullptr;
  }
  std::string desc_, name_;
  bool parsed_ = false;
  std::vector<std::unique_ptr<Option>> opts_;
  std::vector<std::unique_ptr<App>> subs_;
};

}  // namespace CLI
