// Exception -> sd_status translation for the extern "C" layer.
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "../internal.hpp"

namespace sdb {

void set_last_error(const std::string& msg);

// Runs f(); maps the reference's exception types onto status codes and
// records the message (SURVEY §8b "Errors").
template <typename F>
sd_status guard(F&& f) noexcept {
    try {
        f();
        return SD_OK;
    } catch (const OomError& e) {
        set_last_error(e.what());
        return SD_OOM;
    } catch (const CudaError& e) {
        set_last_error(e.what());
        return SD_CUDA_ERROR;
    } catch (const NcclError& e) {
        set_last_error(e.what());
        return SD_NCCL_ERROR;
    } catch (const std::out_of_range& e) {
        set_last_error(e.what());
        return SD_OUT_OF_RANGE;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return SD_INVALID_ARGUMENT;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return SD_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SD_RUNTIME_ERROR;
    } catch (...) {
        set_last_error("unknown error");
        return SD_RUNTIME_ERROR;
    }
}

inline void require(bool ok, const char* msg) {
    if (!ok) throw std::invalid_argument(msg);
}

}  // namespace sdb
