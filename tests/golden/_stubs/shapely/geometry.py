"""Import-time stub (see __init__.py)."""


class Polygon:  # pragma: no cover - never constructed on the hot path
    def __init__(self, *args, **kwargs):
        raise NotImplementedError("shapely stub")
