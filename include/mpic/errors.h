// mpic error classes — the contract of proj/include/mpic/errors.h:10-62, unchanged.
// Every class maps 1:1 onto an mpic_status code of the C ABI (include/mpic_b200.h).
#pragma once

#include <stdexcept>
#include <string>

namespace mpic {

struct error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct config_error : error {  // MPIC_ERR_CONFIG
    using error::error;
};
struct validation_error : error {  // MPIC_ERR_VALIDATION
    using error::error;
};
struct state_error : error {  // MPIC_ERR_STATE
    using error::error;
};
struct link_error : error {  // MPIC_ERR_LINK
    using error::error;
};
struct contract_error : error {  // MPIC_ERR_CONTRACT
    using error::error;
};
struct format_error : error {  // MPIC_ERR_FORMAT
    using error::error;
};
struct integrity_error : error {  // MPIC_ERR_INTEGRITY
    using error::error;
};
struct io_error : error {  // MPIC_ERR_IO
    using error::error;
};
struct not_found_error : error {  // MPIC_ERR_NOT_FOUND
    using error::error;
};
struct request_error : error {  // MPIC_ERR_REQUEST
    using error::error;
};

}  // namespace mpic
