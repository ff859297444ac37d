"""pytest plugin: run the reference package's OWN test suite with the B200 drop-in installed.

Loaded with ``-p ref_install_plugin`` (``tests/`` on PYTHONPATH, ``baseline/_ref`` holding the
reference package ``tmfgclust`` and its unmodified ``tests/``).  At configure time -- before any
reference test module runs ``from tmfgclust import ...`` -- it imports tmfgclust and calls
``paper_2408_09399_b200.install()``, so every rebound stage (sort, heap TMFG, APSP, DBHT,
hierarchy; pipeline.py:191-223 looks them up at call time) runs on the GPU.  The session header
lists what was rebound; ``TG_REF_REQUIRE_INSTALLED=1`` makes a missing library a hard error.
"""

from __future__ import annotations

import sys
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

_SAVED = {}


def pytest_configure(config):
    import tmfgclust

    import paper_2408_09399_b200 as p

    p._native.load()
    _SAVED.update(p.install(tmfgclust))
    config._tg_installed = sorted(f"{m}.{n}" for (m, n) in _SAVED)
    print(f"paper_2408_09399_b200.install(): {len(_SAVED)} reference attributes rebound to the B200 path",
          file=sys.stderr)


def pytest_report_header(config):
    names = getattr(config, "_tg_installed", [])
    return [f"paper_2408_09399_b200.install(): {len(names)} reference attributes rebound to the B200 path",
            "  " + ", ".join(names)]


def pytest_unconfigure(config):
    import paper_2408_09399_b200 as p

    p.uninstall(_SAVED)
