"""Exceptions, named after the reference's so callers catch the same things.

* CodegenError    -- codegen.py:63  (graph the dispatcher cannot generate for)
* ToolchainError  -- codegen.py:67  (library missing / unloadable)
* ExecutionError  -- interpreter.py:48 InterpreterError's role for runtime faults
* OutOfBoundsError -- interpreter.py:56-57 (dynamic WCR index out of range,
  raised at interpreter.py:265-268)
"""

from __future__ import annotations

from ._lib import BackendUnavailable


class CodegenError(RuntimeError):
    pass


class ToolchainError(BackendUnavailable):
    pass


class ExecutionError(RuntimeError):
    pass


class OutOfBoundsError(ExecutionError):
    pass
