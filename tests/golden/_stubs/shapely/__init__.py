"""Import-time stub: flatpoly/postprocess.py:20-21 imports shapely at package
import; the OPC front-end never calls it.  Used only by make_golden.py."""


def make_valid(geom):  # pragma: no cover - never reached on the hot path
    raise NotImplementedError("shapely stub")
