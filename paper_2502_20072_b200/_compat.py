"""Reference types when descsearch is importable, same-shaped stand-ins otherwise.

As a drop-in the package must raise the reference's exception classes and
return the reference's ``Model`` records (models.py:23-41), so when the
reference package is importable its classes are used.  Without it (e.g. on a
GPU box that only carries this repo) equivalent classes with the same names
and fields are defined here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

try:  # pragma: no cover - depends on the environment
    from descsearch.errors import CapacityError, DescsearchError  # errors.py:4-13
    from descsearch.models import Model  # models.py:23-41
    from descsearch.search import RankDeficient, RankOutOfRange  # search.py:27-32

    HAVE_REFERENCE = True
except Exception:  # noqa: BLE001
    HAVE_REFERENCE = False

    class DescsearchError(Exception):
        """Base class for all errors raised by this package."""

    class CapacityError(DescsearchError):
        """A requested materialization would exceed the configured feature budget."""

    class RankOutOfRange(DescsearchError):
        """A combination rank outside [0, C(m, n)) was requested."""

    class RankDeficient(DescsearchError):
        """The requested tuple's least-squares system is numerically singular."""

    @dataclass
    class Model:
        """Same fields as descsearch.models.Model."""

        indices: tuple
        expressions: tuple | None
        coefficients: np.ndarray
        score: float
        rmse_per_task: np.ndarray
        task_labels: tuple

        @property
        def dimension(self) -> int:
            return len(self.indices)
