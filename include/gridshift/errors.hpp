// errors.hpp — exception taxonomy of the GridShift engine.
//
// Same type names and hierarchy as the reference's error header
// (/root/reference/proj/include/gridshift/errors.hpp:9-72), so code written against the
// reference catches the same types.  Only the types the engine path can raise are used by
// this library; the rest are declared for source compatibility of callers.
#pragma once

#include <stdexcept>
#include <string>

namespace gridshift {

struct Error : std::runtime_error {  // root of the hierarchy (reference :9-11)
  using std::runtime_error::runtime_error;
};

// caller-supplied values that violate a contract (reference :14-28, :46-61)
struct InvalidInputError : Error { using Error::Error; };
struct InvalidBandwidthError : InvalidInputError { using InvalidInputError::InvalidInputError; };
struct EmptyInputError : InvalidInputError { using InvalidInputError::InvalidInputError; };
struct InvalidParameterError : InvalidInputError { using InvalidInputError::InvalidInputError; };
struct SizeCapError : InvalidInputError { using InvalidInputError::InvalidInputError; };
struct InvalidWindowError : InvalidInputError { using InvalidInputError::InvalidInputError; };
struct SelectionError : InvalidInputError { using InvalidInputError::InvalidInputError; };

// library bug: a structural invariant failed (reference :31-33)
struct InternalInvariantError : Error { using Error::Error; };

// outside the engine path; declared for callers (reference :36-44, :51-53, :70-72)
struct UndefinedScoreError : Error { using Error::Error; };
struct TuningFailureError : Error { using Error::Error; };
struct DecodeError : Error { using Error::Error; };
struct IoError : Error { using Error::Error; };

// parse failure with an optional 1-based line number (reference :64-68)
struct ParseError : Error {
  explicit ParseError(const std::string& what, long line = -1)
      : Error(line < 0 ? what : what + " (line " + std::to_string(line) + ")"),
        line_number(line) {}
  long line_number;
};

}  // namespace gridshift
