# round-end style verification: GPU suite, smoke, the default bench line, the reference arm
tag=${1:-final}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_$tag.log 2>&1; echo pytest rc=$? >> gpurun_out/gputest_$tag.log
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo bench rc=$? >> gpurun_out/bench_$tag.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; echo ref rc=$? >> gpurun_out/bench_ref_$tag.err
