# GPU suite + smoke (used with gpurun; logs land in gpurun_out/)
tag=${1:-x}
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke_$tag.log
timeout 2400 python -m pytest tests -m gpu -q ${2:-} > gpurun_out/gputest_$tag.log 2>&1; echo pytest rc=$? >> gpurun_out/gputest_$tag.log
