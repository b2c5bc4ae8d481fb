// oracle/dropin/CLI11.hpp — TEST INFRASTRUCTURE ONLY.
//
// A minimal CLI11-compatible shim, written for this repo, that compiles the
// reference's command-line front end (proj/tools/sabr_cli.cpp) unchanged: its
// build expects CLI11.hpp, which is not in the tree.  It covers
// the subset sabr_cli.cpp uses: App(description), require_subcommand(1),
// add_subcommand(name, description), add_option(name, variable, description)
// for std::string / int / std::optional<T> / std::vector<std::string>
// (repeatable), Option::required(), App::parse(argc, argv), App::parsed(),
// App::exit(error) and the CallForHelp / ParseError exceptions.  "--name v"
// and "--name=v" are accepted.  Usage errors print one line to stderr.
#pragma once

#include <cstdint>
#include <functional>
#include <iostream>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

namespace CLI {

struct Error : std::runtime_error {
    int code;
    Error(const std::string& m, int c) : std::runtime_error(m), code(c) {}
};
struct ParseError : Error {
    explicit ParseError(const std::string& m, int c = 106) : Error(m, c) {}
};
struct CallForHelp : ParseError {
    CallForHelp() : ParseError("help requested", 0) {}
};

namespace detail {
template <class T>
struct is_optional : std::false_type {};
template <class T>
struct is_optional<std::optional<T>> : std::true_type {};

template <class T>
void convert(const std::string& name, const std::string& text, T& out) {
    if constexpr (std::is_same_v<T, std::string>) {
        out = text;
    } else {
        std::istringstream in(text);
        T v{};
        in >> v;
        if (in.fail() || !in.eof()) throw ParseError("--" + name + ": cannot convert '" + text + "'");
        out = v;
    }
}
}  // namespace detail

class Option {
public:
    Option(std::string name, std::function<void(const std::string&)> set, bool repeatable)
        : name_(std::move(name)), set_(std::move(set)), repeatable_(repeatable) {}
    Option* required(bool r = true) {
        required_ = r;
        return this;
    }
    const std::string& name() const { return name_; }
    bool is_required() const { return required_; }
    bool repeatable() const { return repeatable_; }
    int count() const { return count_; }
    void set(const std::string& v) {
        set_(v);
        ++count_;
    }

private:
    std::string name_;
    std::function<void(const std::string&)> set_;
    bool repeatable_;
    bool required_ = false;
    int count_ = 0;
};

class App {
public:
    explicit App(std::string description = "", std::string name = "") : desc_(std::move(description)), name_(std::move(name)) {}

    void require_subcommand(int n) { require_sub_ = n; }

    App* add_subcommand(const std::string& name, const std::string& description) {
        subs_.push_back(std::make_unique<App>(description, name));
        return subs_.back().get();
    }

    template <class T>
    Option* add_option(const std::string& flag, T& var, const std::string& /*description*/ = "") {
        const std::string name = flag.rfind("--", 0) == 0 ? flag.substr(2) : flag;
        std::function<void(const std::string&)> set;
        bool repeatable = false;
        if constexpr (detail::is_optional<T>::value) {
            set = [&var, name](const std::string& t) {
                typename T::value_type v{};
                detail::convert(name, t, v);
                var = v;
            };
        } else if constexpr (std::is_same_v<T, std::vector<std::string>>) {
            repeatable = true;
            set = [&var](const std::string& t) { var.push_back(t); };
        } else {
            set = [&var, name](const std::string& t) { detail::convert(name, t, var); };
        }
        opts_.push_back(std::make_unique<Option>(name, std::move(set), repeatable));
        return opts_.back().get();
    }

    bool parsed() const { return parsed_; }

    void parse(int argc, char** argv) {
        std::vector<std::string> args(argv + 1, argv + argc);
        parse_args(args, 0);
    }

    int exit(const Error& e) const {
        if (dynamic_cast<const CallForHelp*>(&e)) {
            std::cout << usage();
            return 0;
        }
        std::cerr << e.what() << "\n" << "Run with --help for more information.\n";
        return e.code;
    }

private:
    std::string usage() const {
        std::ostringstream o;
        o << desc_ << "\n";
        for (const auto& s : subs_) o << "  " << s->name_ << "  " << s->desc_ << "\n";
        for (const auto& op : opts_) o << "  --" << op->name() << "\n";
        return o.str();
    }

    void parse_args(const std::vector<std::string>& args, std::size_t i) {
        parsed_ = true;
        for (; i < args.size(); ++i) {
            const std::string& a = args[i];
            if (a == "--help" || a == "-h") throw CallForHelp();
            if (a.rfind("--", 0) == 0) {
                std::string name = a.substr(2), value;
                const auto eq = name.find('=');
                bool has_value = false;
                if (eq != std::string::npos) {
                    value = name.substr(eq + 1);
                    name = name.substr(0, eq);
                    has_value = true;
                }
                Option* op = nullptr;
                for (const auto& o : opts_)
                    if (o->name() == name) op = o.get();
                if (!op) throw ParseError("The following argument was not expected: " + a, 109);
                if (!has_value) {
                    if (i + 1 >= args.size()) throw ParseError("--" + name + ": 1 required argument missing", 107);
                    value = args[++i];
                }
                if (op->count() > 0 && !op->repeatable())
                    throw ParseError("--" + name + ": option given more than once", 108);
                op->set(value);
                continue;
            }
            App* sub = nullptr;
            for (const auto& s : subs_)
                if (s->name_ == a) sub = s.get();
            if (!sub) throw ParseError("The following argument was not expected: " + a, 109);
            sub->parse_args(args, i + 1);
            i = args.size();
            ++subs_parsed_;
        }
        for (const auto& o : opts_)
            if (o->is_required() && o->count() == 0) throw ParseError("--" + o->name() + " is required", 106);
        if (require_sub_ > 0 && subs_parsed_ < require_sub_)
            throw ParseError("A subcommand is required", 106);
    }

    std::string desc_, name_;
    int require_sub_ = 0, subs_parsed_ = 0;
    bool parsed_ = false;
    std::vector<std::unique_ptr<App>> subs_;
    std::vector<std::unique_ptr<Option>> opts_;
};

}  // namespace CLI
