set -x
python tools/probe_cfg.py 3 2 2>&1 | tail -n 2
cp paper_1812_04315_b200/libnenmf_b200.so /tmp/lib_g4.so
cp paper_1812_04315_b200/libnenmf_b200_g32.so.bak paper_1812_04315_b200/libnenmf_b200.so
python tools/probe_cfg.py 3 2 2>&1 | tail -n 2
python tools/probe_cfg.py 4 2 2>&1 | tail -n 2
cp /tmp/lib_g4.so paper_1812_04315_b200/libnenmf_b200.so
NENMF_NNLS_SIMT=1 python tools/probe_cfg.py 3 2 2>&1 | tail -n 2
