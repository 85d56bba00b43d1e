cd $GRAFT_REPO_ROOT
python tools/time_u8_fix.py > gpurun_out/time_u8_fix.log 2>&1
for st in 6 8 10; do WF_D4_STAGES=$st python tools/sweep_u8.py v3:0:$st >> gpurun_out/u8_stages.log 2>&1; done
python -m pytest tests/test_gpu_quantized.py tests/test_gpu_tiling.py tests/test_gpu_pnm.py -q -x > gpurun_out/pytest_q.log 2>&1
