# the C3 oracle digest on the box's host cores (oracle + synth only)
python tools/oracle_digests.py C3 --threads $(nproc) --out gpurun_out/digests_box_c3.json > gpurun_out/digests_box_c3.log 2>&1; echo rc=$? >> gpurun_out/digests_box_c3.log
