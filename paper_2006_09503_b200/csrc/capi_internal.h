// Exception -> status-code guard shared by all C-ABI translation units.
#pragma once

#include <exception>
#include <stdexcept>
#include <string>

#include "p2bw.h"

namespace p2bw {

void set_last_error(const std::string& msg);

// malloc'ed NUL-terminated copy, released by the caller with p2bw_free.
char* dup_string(const std::string& s);

// Runs fn; maps p2bw::Error / std::exception to P2BW_ERR and records the message
// for p2bw_last_error() (thread-local, reference wording preserved).
template <class Fn>
int guarded(Fn&& fn) {
    try {
        fn();
        return P2BW_OK;
    } catch (const std::invalid_argument& e) {
        set_last_error(e.what());
        return P2BW_ERR_ARG;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return P2BW_ERR;
    } catch (...) {
        set_last_error("unknown error");
        return P2BW_ERR;
    }
}

}  // namespace p2bw
