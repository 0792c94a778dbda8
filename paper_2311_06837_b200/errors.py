"""Error taxonomy of the reference (errors.hpp:11-44), with the same categories.

The C ABI returns status codes (GDX_INPUT=1, GDX_CAPACITY=2, GDX_CONTRACT=3,
GDX_INTERNAL=4); raise_for_status maps them back onto these classes so callers
see the reference's exception types.  CLI exit codes follow
granndis_main.cpp:640-660: capacity -> 2, everything else -> 1.
"""


class GranndisError(RuntimeError):
    category = "internal"

    def __init__(self, detail: str):
        super().__init__(detail)
        self.detail = detail


class InputError(GranndisError):
    category = "input"


class ParseError(GranndisError):
    category = "parse"


class CapacityError(GranndisError):
    category = "capacity"


class ContractError(GranndisError):
    category = "contract"


class InternalError(GranndisError):
    category = "internal"


_BY_CODE = {1: InputError, 2: CapacityError, 3: ContractError, 4: InternalError}


def raise_for_status(code: int, message: str) -> None:
    raise _BY_CODE.get(code, InternalError)(message)


def exit_code(err: GranndisError) -> int:
    return 2 if isinstance(err, CapacityError) else 1
