# GPU digest parity for the configs already in tests/golden, then the N1 oracle digest on the box's host cores
timeout 1200 python -m pytest tests/test_digests_gpu.py -q -rA > gpurun_out/digests_gpu.log 2>&1; echo rc=$? >> gpurun_out/digests_gpu.log
python tools/oracle_digests.py N1 --threads $(nproc) --out gpurun_out/digests_box.json > gpurun_out/digests_box.log 2>&1; echo rc=$? >> gpurun_out/digests_box.log
