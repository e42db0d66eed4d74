"""ptxwatt.errors (pkg/src/ptxwatt/errors.py): the same exception tree and exit codes."""
from paper_2601_13345_b200 import errors as _e

for _name in dir(_e):
    _obj = getattr(_e, _name)
    if isinstance(_obj, type) and issubclass(_obj, Exception):
        globals()[_name] = _obj
del _name, _obj
