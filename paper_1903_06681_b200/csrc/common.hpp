// common.hpp -- shared host-side helpers of libdconv (error state, checks).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <stdexcept>

#include "../../include/dconv.h"

namespace dc {

// Error carried from deep inside the library to the C ABI (never crosses it).
struct Error : std::runtime_error {
    dc_status_t code;
    Error(dc_status_t c, const std::string &m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string &msg);

[[noreturn]] inline void fail(dc_status_t code, const std::string &msg) { throw Error(code, msg); }

#define DC_REQUIRE(cond, code, ...)                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            char _b[512];                                                      \
            std::snprintf(_b, sizeof _b, __VA_ARGS__);                         \
            ::dc::fail(code, _b);                                              \
        }                                                                      \
    } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }
// floor division for possibly negative numerators
inline int64_t floor_div(int64_t a, int64_t b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

extern thread_local uint64_t g_launches;

}  // namespace dc

// Wrap a C-ABI body: map exceptions to status codes + thread-local message.
#define DC_API_BEGIN try {
#define DC_API_END                                                             \
    return DC_OK;                                                              \
    }                                                                          \
    catch (const ::dc::Error &e) {                                             \
        ::dc::set_last_error(e.what());                                        \
        return e.code;                                                         \
    }                                                                          \
    catch (const std::bad_alloc &) {                                           \
        ::dc::set_last_error("host out of memory");                            \
        return DC_ERR_OOM;                                                     \
    }                                                                          \
    catch (const std::exception &e) {                                          \
        ::dc::set_last_error(e.what());                                        \
        return DC_ERR_ARG;                                                     \
    }
