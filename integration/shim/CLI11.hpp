// Minimal CLI11-API shim (TEST / INTEGRATION INFRASTRUCTURE ONLY).
//
// CLI11 (a vendored, gitignored dependency of the reference: proj/README.md:29-30)
// is absent from this image. This header implements the subset of its API
// that /root/reference/proj/tools/ditsim.cpp uses, so the reference's CLI
// compiles unmodified from its own sources:
//   App{desc}, add_option(name, T&, desc) for string / int / long long /
//   double, add_flag(name, bool&, desc), add_subcommand, require_subcommand,
//   fallthrough, parse(argc, argv), exit(ParseError), Option::check(IsMember),
//   Option::required, Option::count, App::parsed.
// Semantics follow CLI11: "--name value" and "--name=value"; a name without
// leading dashes is positional; options the active subcommand does not know
// fall through to its parent when fallthrough() is set; parse errors throw
// CLI::ParseError, and App::exit prints the message and returns its code
// (0 for --help).
#pragma once

#include <cstdlib>
#include <functional>
#include <initializer_list>
#include <iostream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

namespace CLI {

class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& msg, int code) : std::runtime_error(msg), code_(code) {}
  int get_exit_code() const { return code_; }

 private:
  int code_;
};

// A validator: returns an empty string when the value is acceptable.
struct Validator {
  std::function<std::string(const std::string&)> fn;
};

inline Validator IsMember(std::initializer_list<std::string> values) {
  std::vector<std::string> v(values);
  return Validator{[v](const std::string& s) -> std::string {
    for (const std::string& m : v)
      if (m == s) return "";
    std::string all;
    for (const std::string& m : v) all += (all.empty() ? "" : ",") + m;
    return s + " not in {" + all + "}";
  }};
}

class Option {
 public:
  Option(std::string name, std::function<bool(const std::string&)> set, bool flag)
      : name_(std::move(name)), set_(std::move(set)), flag_(flag) {}
  Option* check(Validator v) {
    checks_.push_back(std::move(v));
    return this;
  }
  Option* required(bool r = true) {
    required_ = r;
    return this;
  }
  std::size_t count() const { return count_; }

 private:
  friend class App;
  bool positional() const { return name_.rfind("-", 0) != 0; }
  bool matches(const std::string& s) const { return s == name_; }
  void apply(const std::string& value) {
    for (const Validator& v : checks_) {
      const std::string err = v.fn(value);
      if (!err.empty()) throw ParseError(name_ + ": " + err, 106);
    }
    if (!set_(value)) throw ParseError(name_ + ": invalid value " + value, 106);
    ++count_;
  }
  std::string name_;
  std::function<bool(const std::string&)> set_;
  bool flag_ = false;
  bool required_ = false;
  std::size_t count_ = 0;
  std::vector<Validator> checks_;
};

namespace detail {
inline bool assign(const std::string& s, std::string& out) {
  out = s;
  return true;
}
template <class T>
bool assign(const std::string& s, T& out) {
  std::istringstream in(s);
  T v{};
  in >> v;
  if (in.fail() || !in.eof()) return false;
  out = v;
  return true;
}
}  // namespace detail

class App {
 public:
  explicit App(std::string description = "", std::string name = "")
      : description_(std::move(description)), name_(std::move(name)) {}

  template <class T>
  Option* add_option(const std::string& name, T& target, const std::string& = "") {
    options_.push_back(std::make_unique<Option>(
        name, [&target](const std::string& s) { return detail::assign(s, target); }, false));
    return options_.back().get();
  }
  Option* add_flag(const std::string& name, bool& target, const std::string& = "") {
    options_.push_back(std::make_unique<Option>(
        name, [&target](const std::string&) { return target = true; }, true));
    return options_.back().get();
  }
  App* add_subcommand(const std::string& name, const std::string& description = "") {
    subs_.push_back(std::make_unique<App>(description, name));
    subs_.back()->parent_ = this;
    return subs_.back().get();
  }
  void require_subcommand(int n) { require_subs_ = n; }
  void fallthrough(bool on = true) { fallthrough_ = on; }
  bool parsed() const { return parsed_; }

  void parse(int argc, char** argv) {
    std::vector<std::string> args;
    for (int i = 1; i < argc; ++i) args.emplace_back(argv[i]);
    parsed_ = true;
    App* active = this;
    for (std::size_t i = 0; i < args.size(); ++i) {
      const std::string& a = args[i];
      if (a == "--help" || a == "-h") throw ParseError(help(), 0);
      if (a.rfind("-", 0) == 0) {
        std::string key = a, value;
        bool inline_value = false;
        const auto eq = a.find('=');
        if (eq != std::string::npos) {
          key = a.substr(0, eq);
          value = a.substr(eq + 1);
          inline_value = true;
        }
        Option* opt = nullptr;
        for (App* app = active; app && !opt; app = app->fallthrough_target()) opt = app->find(key);
        if (!opt) throw ParseError("The following argument was not expected: " + a, 109);
        if (opt->flag_) {
          opt->apply("true");
          continue;
        }
        if (!inline_value) {
          if (i + 1 >= args.size()) throw ParseError(key + " requires an argument", 109);
          value = args[++i];
        }
        opt->apply(value);
        continue;
      }
      // a subcommand name (only before any positional of the active app)
      App* sub = nullptr;
      for (auto& s : active->subs_)
        if (s->name_ == a) sub = s.get();
      if (sub && !active->any_positional_) {
        sub->parsed_ = true;
        active = sub;
        continue;
      }
      Option* pos = nullptr;
      for (auto& o : active->options_)
        if (o->positional() && o->count_ == 0) {
          pos = o.get();
          break;
        }
      if (!pos) throw ParseError("The following argument was not expected: " + a, 109);
      active->any_positional_ = true;
      pos->apply(a);
    }
    check_required(this);
  }

  int exit(const ParseError& e) const {
    if (e.get_exit_code() == 0) {
      std::cout << e.what();
      return 0;
    }
    std::cerr << e.what() << "\n";
    return e.get_exit_code();
  }

 private:
  App* fallthrough_target() const { return parent_ && fallthrough_chain() ? parent_ : nullptr; }
  bool fallthrough_chain() const {
    for (const App* a = parent_; a; a = a->parent_)
      if (a->fallthrough_) return true;
    return false;
  }
  Option* find(const std::string& key) {
    for (auto& o : options_)
      if (!o->positional() && o->matches(key)) return o.get();
    return nullptr;
  }
  static void check_required(const App* app) {
    for (const auto& o : app->options_)
      if (o->required_ && o->count_ == 0) throw ParseError(o->name_ + " is required", 106);
    int n = 0;
    for (const auto& s : app->subs_)
      if (s->parsed_) {
        ++n;
        check_required(s.get());
      }
    if (app->require_subs_ > 0 && n < app->require_subs_)
      throw ParseError("A subcommand is required", 106);
  }
  std::string help() const {
    std::string h = description_ + "\n";
    for (const auto& s : subs_) h += "  " + s->name_ + "  " + s->description_ + "\n";
    return h;
  }

  std::string description_, name_;
  App* parent_ = nullptr;
  std::vector<std::unique_ptr<Option>> options_;
  std::vector<std::unique_ptr<App>> subs_;
  int require_subs_ = 0;
  bool fallthrough_ = false;
  bool parsed_ = false;
  bool any_positional_ = false;
};

}  // namespace CLI
