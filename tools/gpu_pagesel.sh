OUT=gpurun_out/pg; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_select.py tests/test_gpu_prefill_tc.py tests/test_gpu_prefill.py tests/test_gpu_pipeline.py tests/test_gpu_measured.py tests/test_gpu_offload.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
NO_NCU=1 OUT=$OUT/pf bash tools/gpu_pf.sh | tail -4
