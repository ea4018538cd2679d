timeout 600 python -m pytest tests/test_adjoint_gpu.py -q > gpurun_out/adjf.log 2>&1; echo rc=$? >> gpurun_out/adjf.log
VTI_ADJ_TWO_PASS=1 timeout 600 python -m pytest tests/test_adjoint_gpu.py -q >> gpurun_out/adjf.log 2>&1; echo rc=$? >> gpurun_out/adjf.log
for c in C2 C3 C5 N1; do python tools/adjoint_rate.py --config $c >> gpurun_out/adjf.log 2>&1; done
VTI_ADJ_TWO_PASS=1 python tools/adjoint_rate.py --config C2 >> gpurun_out/adjf.log 2>&1
