#!/bin/bash
# small-grid adjoint: z-chunks down to 4 planes when 32-plane chunks leave CTAs idle (A/B against tools/ab/libvti_old.so)
mkdir -p gpurun_out
O=gpurun_out/adj_c1b.log
: > $O
L=paper_1410_1387_b200/lib/libvti.so
cp $L /tmp/new.so
cp tools/ab/libvti_old.so $L
for p in 32 64; do echo "[old C1 f$p]" >> $O; timeout 300 python tools/adjoint_rate.py --config C1 --precision $p --steps 100 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; done
cp /tmp/new.so $L
for p in 32 64; do echo "[new C1 f$p]" >> $O; timeout 300 python tools/adjoint_rate.py --config C1 --precision $p --steps 100 2>&1 | grep -o '"adjoint_gpoints_s": [0-9.]*' >> $O; done
timeout 900 python -m pytest tests/test_adjoint_gpu.py -q -x >> $O 2>&1; echo "pytest rc=$?" >> $O
