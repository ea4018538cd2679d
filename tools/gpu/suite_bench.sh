set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r02b.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_r02b.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02b.log 2>&1; echo pytest rc=$? >> gpurun_out/gputest_r02b.log
python bench.py > gpurun_out/bench_r02b.log 2>&1; echo bench rc=$? >> gpurun_out/bench_r02b.log
