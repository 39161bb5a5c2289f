python tools/contention_probe.py
SPGCM_PACK=16 python tools/contention_probe.py
SPGCM_PACK=4 python tools/contention_probe.py
