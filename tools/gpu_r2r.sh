timeout 600 python tools/dump_c4.py c4 384
