# the C5 oracle digest on the box's host cores (oracle + synth only)
python tools/oracle_digests.py C5 --threads $(nproc) --out gpurun_out/digests_box_c5.json > gpurun_out/digests_box_c5.log 2>&1; echo rc=$? >> gpurun_out/digests_box_c5.log
