"""Golden fixtures: tiny text tables, each row citing where its value comes from."""
import os

_HERE = os.path.dirname(os.path.abspath(__file__))


def load(name: str) -> dict:
    """{name: (value, tolerance, citation)} from tests/golden/<name>.txt."""
    out = {}
    with open(os.path.join(_HERE, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            parts = line.split(None, 3)
            out[parts[0]] = (float(parts[1]), float(parts[2]), parts[3] if len(parts) > 3 else "")
    return out
