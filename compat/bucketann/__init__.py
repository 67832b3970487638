"""``import bucketann`` -> the B200 package (drop-in alias).

Put ``compat/`` first on ``sys.path`` (``PYTHONPATH=compat``) and code written
against the reference package -- including its own test-suite -- runs on the
device implementation: ``bucketann`` and ``bucketann.{core, layout, builder,
searcher, updater, evaluate, dataio}`` all resolve to ``paper_2604_16402_b200``.
"""
import os
import sys

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

import paper_2604_16402_b200 as _impl  # noqa: E402

for _name in ("core", "layout", "builder", "searcher", "updater", "evaluate", "dataio"):
    sys.modules[f"{__name__}.{_name}"] = getattr(_impl, _name)
sys.modules[__name__] = _impl
