mkdir -p gpurun_out/r2s
python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -p no:cacheprovider -k "not c5_digest" > gpurun_out/r2s/pytest.txt 2>&1; echo rc=$? >> gpurun_out/r2s/pytest.txt
python tools/leaftrace.py tools/variants/liblt.so > gpurun_out/r2s/lt.txt 2>&1
python tools/leaftrace.py tools/variants/libltsm.so >> gpurun_out/r2s/lt.txt 2>&1
bash tools/job_var.sh gpurun_out/r2s paper_1112_5717_b200/libranklab_gpu.so tools/variants/libbrsm.so tools/variants/libnobridge.so
