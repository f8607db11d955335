// vtc error taxonomy: one class per reference error (proj/include/vtelim/errors.hpp:10-38),
// each with the C-ABI status code it maps to (include/vtc.h VTC_ERR_*).
#pragma once

#include <stdexcept>
#include <string>

namespace vtc {

struct Error : std::runtime_error {
    explicit Error(const std::string& msg) : std::runtime_error(msg) {}
    virtual int code() const { return 1; }
};

#define VTC_DECLARE_ERROR(Name, Code)                         \
    struct Name : Error {                                     \
        using Error::Error;                                   \
        int code() const override { return Code; }            \
    }

VTC_DECLARE_ERROR(SchemaError, 2);
VTC_DECLARE_ERROR(CycleError, 3);
VTC_DECLARE_ERROR(ShapeError, 4);
VTC_DECLARE_ERROR(UnknownOperatorError, 5);
VTC_DECLARE_ERROR(OutOfBoundsError, 6);
VTC_DECLARE_ERROR(MissingBaseMapError, 7);
VTC_DECLARE_ERROR(ComposeLimitError, 8);
VTC_DECLARE_ERROR(ConflictViolationError, 9);
VTC_DECLARE_ERROR(IncompleteSelectionError, 10);
VTC_DECLARE_ERROR(CycleDetectedError, 11);
VTC_DECLARE_ERROR(WriteAliasingError, 12);
VTC_DECLARE_ERROR(SpaceTooLargeError, 13);
VTC_DECLARE_ERROR(MissingInputError, 14);
VTC_DECLARE_ERROR(ShapeMismatchError, 15);
VTC_DECLARE_ERROR(ExecutionError, 16);
VTC_DECLARE_ERROR(EquivalenceFailureError, 17);
VTC_DECLARE_ERROR(InvalidVtogError, 18);
VTC_DECLARE_ERROR(BudgetExceededError, 19);
VTC_DECLARE_ERROR(CudaError, 20);
VTC_DECLARE_ERROR(NcclError, 21);
VTC_DECLARE_ERROR(UnsupportedError, 22);

#undef VTC_DECLARE_ERROR

}  // namespace vtc
