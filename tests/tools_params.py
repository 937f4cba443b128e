"""Read the fixed prime chain from include/aegis_params.h (shared data)."""
import os
import re

_H = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "aegis_params.h")


def _read(name):
    txt = open(_H).read()
    body = txt.split(name, 1)[1].split("};", 1)[0]
    return [int(x, 16) for x in re.findall(r"0x([0-9a-fA-F]+)ULL", body)]


def main_primes():
    return _read("AEGIS_MAIN_PRIMES[")


def special_primes():
    return _read("AEGIS_SPECIAL_PRIMES_LIST[")
