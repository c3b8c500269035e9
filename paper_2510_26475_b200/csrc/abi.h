// abi.h -- the C-ABI error convention shared by every extern "C" translation unit: an entry
// point runs its body under guard(), which maps the C++ exception family onto the status codes
// of include/respec_b200.h and keeps the message for rs_last_error() (thread-local).
#pragma once
#include <new>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "../../include/respec_b200.h"

namespace rs_abi {

std::string &last_error();  // api.cpp

template <class F>
int guard(F &&f) {
    try {
        f();
        return RS_OK;
    } catch (const rs::CudaError &e) {
        last_error() = e.what();
        return RS_ECUDA;
    } catch (const std::bad_alloc &) {
        last_error() = "out of memory";
        return RS_ENOMEM;
    } catch (const std::invalid_argument &e) {
        last_error() = e.what();
        return RS_EINVAL;
    } catch (const std::out_of_range &e) {
        last_error() = e.what();
        return RS_EINVAL;
    } catch (const std::logic_error &e) {
        last_error() = e.what();
        return RS_ELOGIC;
    } catch (const std::runtime_error &e) {
        last_error() = e.what();
        return RS_ESTATE;
    } catch (const std::exception &e) {
        last_error() = e.what();
        return RS_ESTATE;
    }
}

inline void need(const void *p, const char *what) {
    if (!p) throw std::invalid_argument(std::string(what) + ": null pointer");
}

// Re-raise a failed C-ABI status as the matching C++ exception (used by host components that
// are themselves built on the C-ABI, e.g. the online learner).
inline void rethrow(int status) {
    if (status == RS_OK) return;
    const std::string m = last_error();
    switch (status) {
        case RS_EINVAL: throw std::invalid_argument(m);
        case RS_ELOGIC: throw std::logic_error(m);
        case RS_ENOMEM: throw std::bad_alloc();
        case RS_ECUDA: throw rs::CudaError(m);
        default: throw std::runtime_error(m);
    }
}

}  // namespace rs_abi
