OUT=gpurun_out/selt; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_select.py tests/test_gpu_pipeline.py tests/test_gpu_measured.py tests/test_gpu_sanitizer.py tests/test_gpu_sharded.py -x -q -p no:cacheprovider > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -5 $OUT/pytest.log
