"""Wire formats next to the hot path.

* ``export_text(mesh)`` -- the reference's plain-text mesh dump
  (mesh.py:479-490): ``v x y`` per vertex, ``e i j k macro_id`` per macro,
  ``f left right tag`` per skeleton face; 3-D meshes add a coordinate / vertex.
* ``write_csv`` / ``rows_to_csv`` / ``read_csv`` -- the reference's report CSV
  convention (bench.py:328-379): floats with 17 significant digits, so solver
  reports (``SolveReport.to_record()``) round-trip bit-for-bit.
"""

from __future__ import annotations

import csv
import io
import os
from typing import Sequence

import numpy as np


def export_text(mesh) -> str:
    """Plain-text dump of a mesh exposing ``vertices``, ``macro_elements``
    (``vertex_ids``, ``id``) and ``skeleton`` (``left``, ``right``, ``tag``)."""
    lines = []
    h = 1.0 / mesh.n
    verts = getattr(mesh, "vertices_lattice", None)
    if verts is not None:  # lattice coordinates -> x = i * (1/n), as the reference builds them
        coords = verts.astype(np.float64) * h
    else:
        coords = np.asarray(mesh.vertices, dtype=np.float64)
    for v in coords:
        lines.append("v " + " ".join("%.17g" % float(c) for c in v))
    for e in mesh.macro_elements:
        lines.append("e " + " ".join(str(int(i)) for i in e.vertex_ids) + f" {e.id}")
    for f in mesh.skeleton:
        right = f.right.macro if f.right is not None else -1
        lines.append(f"f {f.left.macro} {right} {f.tag}")
    return "\n".join(lines) + "\n"


def _cell(value) -> str:
    """One CSV cell of the report convention: None -> empty, a float (Python or
    numpy) with 17 significant digits so that it reads back to the same double,
    anything else (bools, ints, strings) through str()."""
    if value is None:
        return ""
    if isinstance(value, (float, np.floating)):
        return format(float(value), ".17g")
    return str(value)


def _table(rows, columns):
    """Header, then one line per record in column order (missing keys empty)."""
    yield list(columns)
    for record in rows:
        yield [_cell(record.get(name)) for name in columns]


def write_csv(rows: list, columns: Sequence[str], out) -> None:
    """Report rows to a CSV file (path) or an open text stream."""
    if isinstance(out, (str, bytes, os.PathLike)):
        with open(out, "w", newline="") as fh:
            csv.writer(fh).writerows(_table(rows, columns))
    else:
        csv.writer(out).writerows(_table(rows, columns))


def rows_to_csv(rows: list, columns: Sequence[str]) -> str:
    sink = io.StringIO()
    csv.writer(sink).writerows(_table(rows, columns))
    return sink.getvalue()


def _parse(raw: str):
    if raw == "":
        return None
    if raw in ("True", "False"):
        return raw == "True"
    try:
        return int(raw)
    except ValueError:
        try:
            return float(raw)
        except ValueError:
            return raw


def read_csv(path) -> list:
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        header = next(reader)
        return [{k: _parse(r) for k, r in zip(header, rec)} for rec in reader]
