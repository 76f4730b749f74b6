"""Drop-in import name of the reference Python package (proj/python/anisocg).

``import anisocg`` resolves to the B200 build, so code (and the reference's
own tests/python/test_smoke.py) written against the reference runs unchanged.
"""
from paper_1302_7193_b200 import *  # noqa: F401,F403
from paper_1302_7193_b200 import __all__  # noqa: F401
