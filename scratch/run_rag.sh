timeout 900 python -m pytest tests/test_gpu_likelihood.py -x -q -k ragged > gpurun_out/gpu_rag.log 2>&1; echo "rag rc=$?"; tail -20 gpurun_out/gpu_rag.log
