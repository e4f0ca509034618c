nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -Ipaper_1910_06017_b200/csrc tools/div_check.cu -o /tmp/div_check 2>/dev/null && /tmp/div_check
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
ARGS="X=1 X=2" bash tools/gpu_ab.sh
