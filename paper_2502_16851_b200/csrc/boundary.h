// boundary.h -- the exception -> status-code plumbing shared by every
// extern "C" translation unit of the library (capi.cpp, dist.cpp).
//
// Codes (include/rooflens_b200.h): 0 OK; 1 + ErrorKind ordinal (reference
// error.hpp:10-32); RL_ERR_CUDA_BASE + cudaError_t; RL_ERR_NCCL_BASE +
// ncclResult_t.  The message goes to a thread-local slot read by
// rl_last_error().
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../../include/rooflens_b200.h"
#include "../../include/rooflens_b200.hpp"

namespace rooflens::b200 {

// An NCCL failure inside a distributed entry point.
class NcclError : public std::runtime_error {
public:
    NcclError(int code, const std::string& msg) : std::runtime_error(msg), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

std::string& last_error_slot();  // thread-local, capi.cpp

template <class F>
int guarded(F&& f) {
    std::string& last = last_error_slot();
    try {
        f();
        last.clear();
        return RL_OK;
    } catch (const Error& e) {
        last = e.what();
        return RL_ERR_KIND_BASE + static_cast<int>(e.kind());
    } catch (const CudaError& e) {
        last = e.what();
        return RL_ERR_CUDA_BASE + e.code();
    } catch (const NcclError& e) {
        last = e.what();
        return RL_ERR_NCCL_BASE + e.code();
    } catch (const std::bad_alloc&) {
        last = "CudaError: host allocation failed";
        return RL_ERR_CUDA_BASE + 2;
    } catch (const std::exception& e) {
        last = std::string("ValidationError: ") + e.what();
        return RL_ERR_KIND_BASE + static_cast<int>(ErrorKind::ValidationError);
    }
}

}  // namespace rooflens::b200
