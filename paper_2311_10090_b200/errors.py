"""The reference's exception taxonomy (proj/core/include/marl/errors.hpp:9-26),
mapped from the C-ABI status codes of include/marl_b200.h."""


class NotFoundError(RuntimeError):
    """Unknown env id, reserved id, ... (errors.hpp:9-12)."""


class SchemaError(RuntimeError):
    """Config rejected: unknown key, wrong type, out-of-range value (errors.hpp:14-17)."""


class ContractError(ValueError):
    """Caller broke an API contract; std::invalid_argument in the reference (errors.hpp:19-22)."""


class DivergenceError(RuntimeError):
    """Non-finite numbers (errors.hpp:24-27)."""


class CudaError(RuntimeError):
    """A CUDA runtime failure (no device, launch failure, ...); there is no CPU fallback."""


_BY_CODE = {1: NotFoundError, 2: SchemaError, 3: ContractError, 4: DivergenceError, 5: CudaError}


def raise_for_status(code: int, message: str):
    raise _BY_CODE.get(code, RuntimeError)(message)
