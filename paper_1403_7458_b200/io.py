"""File interchange for the CLI drop-in.

Mirrors the reference's ``spamm.io`` contract (io.py:33-54, 129-161):

* MatrixMarket matrices, read dense through scipy (any variant: coordinate /
  array, general / symmetric), written with 17 significant digits so a
  write -> read round trip is exact; ``fmt="auto"`` writes coordinate form
  when fewer than half the entries are nonzero (io.py:41-54);
* JSON reports (``ProductStats.to_json_dict``, ``SP2State.to_report_dict``);
* run manifests: command, argv, parameters, seeds, inputs, outputs, library
  version, timestamp, user (io.py:129-152).  Replaying ``argv`` regenerates
  bitwise-identical numerical outputs (wall times excluded).

Host-side only: files are read into host memory and handed to the device
builders; nothing here touches the compute path.
"""

from __future__ import annotations

import getpass
import hashlib
import json
import time
from pathlib import Path

import numpy as np

__all__ = ["read_matrix_market", "write_matrix_market", "write_json", "read_json",
           "sha256_file", "build_manifest", "write_manifest", "read_manifest",
           "MM_FORMATS"]

MM_FORMATS = ("auto", "array", "coordinate")


def read_matrix_market(path) -> np.ndarray:
    """Dense float64 array from a MatrixMarket file of any variant."""
    import scipy.io
    import scipy.sparse
    m = scipy.io.mmread(str(path), spmatrix=False)
    if scipy.sparse.issparse(m):
        m = m.toarray()
    return np.asarray(m, dtype=np.float64)


def _pick_format(matrix: np.ndarray, fmt: str) -> str:
    if fmt not in MM_FORMATS:
        raise ValueError(f"fmt must be auto, array, or coordinate, got {fmt!r}")
    if fmt != "auto":
        return fmt
    return "coordinate" if np.count_nonzero(matrix) < matrix.size / 2 else "array"


def write_matrix_market(path, matrix, fmt: str = "auto", comment: str = "") -> None:
    """Write a dense array as MatrixMarket (17 significant digits)."""
    import scipy.io
    import scipy.sparse
    dense = np.asarray(matrix, dtype=np.float64)
    kind = _pick_format(dense, fmt)
    payload = scipy.sparse.coo_matrix(dense) if kind == "coordinate" else dense
    scipy.io.mmwrite(str(path), payload, comment=comment, precision=17)


def write_json(path, payload: dict) -> None:
    Path(path).write_text(json.dumps(payload, indent=2, sort_keys=False) + "\n")


def read_json(path) -> dict:
    return json.loads(Path(path).read_text())


def sha256_file(path) -> str:
    return hashlib.sha256(Path(path).read_bytes()).hexdigest()


def _user() -> str:
    try:
        return getpass.getuser()
    except Exception:  # noqa: BLE001 - containers without a passwd entry
        return "unknown"


def build_manifest(command: str, parameters: dict, seeds: dict, inputs: list,
                   outputs: list, argv: list) -> dict:
    """Everything needed to reproduce a command's outputs (io.py:129-152)."""
    from . import __version__
    return {
        "command": command,
        "argv": [str(a) for a in argv],
        "parameters": parameters,
        "seeds": seeds,
        "inputs": [str(p) for p in inputs],
        "outputs": [str(p) for p in outputs],
        "library_version": __version__,
        "timestamp": time.strftime("%Y-%m-%dT%H:%M:%S%z"),
        "user": _user(),
    }


def write_manifest(path, manifest: dict) -> None:
    write_json(path, manifest)


def read_manifest(path) -> dict:
    return read_json(path)
