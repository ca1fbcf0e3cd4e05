// pg_guard.h — no C++ exception crosses the C ABI (include/pg.h "General
// conventions"): every extern "C" entry point is a function-try-block ending in
// PGSI_ABI_CATCH, which maps a host allocation failure to PG_ENOMEM and anything
// else to PG_EINVAL with a message in pg_last_error().
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include "pg.h"

namespace pgsi {
void io_set_err(const std::string &s);   // pg_api.cu (thread-local last error)
}

#define PGSI_ABI_CATCH                                                                   \
    catch (const std::bad_alloc &) {                                                     \
        pgsi::io_set_err("host allocation failed (std::bad_alloc)");                     \
        return PG_ENOMEM;                                                                \
    }                                                                                    \
    catch (const std::exception &e_) {                                                   \
        pgsi::io_set_err(std::string("internal error: ") + e_.what());                   \
        return PG_EINVAL;                                                                \
    }                                                                                    \
    catch (...) {                                                                        \
        pgsi::io_set_err("internal error (unknown exception)");                         \
        return PG_EINVAL;                                                                \
    }
