import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


def read_kv(name):
    out = {}
    for ln in read_lines(name):
        key, rest = ln.split("=", 1)
        value = rest.split(";", 1)[0].strip()
        out[key.strip()] = value
    return out
