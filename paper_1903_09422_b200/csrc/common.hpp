// common.hpp — error plumbing shared by the host code and the CUDA sources.
//
// Every C-ABI entry point runs its body inside adsb::guard(), which maps the
// exception classes below onto adsb_status codes (include/adsb.h) and stores
// the message in a thread-local buffer read by adsb_last_error().
#pragma once

#include <cstdint>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>
#include <utility>

#include "adsb.h"

namespace adsb {

struct Error : std::runtime_error {
    adsb_status code;
    Error(adsb_status c, const std::string& msg) : std::runtime_error(msg), code(c) {}
};

[[noreturn]] inline void fail(adsb_status code, const std::string& msg) { throw Error(code, msg); }
[[noreturn]] inline void invalid(const std::string& msg) { fail(ADSB_ERR_INVALID_ARGUMENT, msg); }
[[noreturn]] inline void domain(const std::string& msg) { fail(ADSB_ERR_DOMAIN, msg); }
[[noreturn]] inline void parse_error(const std::string& msg) { fail(ADSB_ERR_PARSE, msg); }

void set_last_error(const std::string& msg);

template <class F>
adsb_status guard(F&& body) noexcept {
    try {
        body();
        set_last_error("");
        return ADSB_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return ADSB_ERR_RUNTIME;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return ADSB_ERR_RUNTIME;
    } catch (...) {
        set_last_error("unknown error");
        return ADSB_ERR_RUNTIME;
    }
}

}  // namespace adsb
