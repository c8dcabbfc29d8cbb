// Exception → pf_status translation shared by every extern "C" entry point.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "pf_sched.h"

namespace pf_detail {

// std::invalid_argument raised for a shape mismatch (reference message kept);
// maps to PF_BAD_SHAPE instead of PF_BAD_ARG.
struct ShapeError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

inline std::string& last_error() {
    thread_local std::string msg;
    return msg;
}

// Runs `body` (which returns an int status); maps C++ exceptions the way the
// reference's callers see them (SURVEY §8b "Errors").
template <class F>
int guard(F&& body) noexcept {
    try {
        last_error().clear();
        return body();
    } catch (const ShapeError& e) {
        last_error() = e.what();
        return PF_BAD_SHAPE;
    } catch (const std::domain_error& e) {
        last_error() = e.what();
        return PF_NOT_PD;
    } catch (const std::length_error& e) {
        last_error() = e.what();
        return PF_LENGTH_ERROR;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return PF_BAD_ARG;
    } catch (const std::logic_error& e) {
        last_error() = e.what();
        return PF_LOGIC_ERROR;
    } catch (const std::bad_alloc&) {
        last_error() = "out of memory";
        return PF_BAD_ARG;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return PF_CUDA_ERROR;
    } catch (...) {
        last_error() = "unknown exception";
        return PF_CUDA_ERROR;
    }
}

}  // namespace pf_detail
