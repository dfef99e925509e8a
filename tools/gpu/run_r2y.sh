# NCCL backend on one GPU (world-1 communicator) next to the hub tests
export PYTHONUNBUFFERED=1
O=gpurun_out/r2y; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -p no:cacheprovider > $O/multirank.log 2>&1; echo "multirank rc=$?" >> $O/multirank.log
tail -5 $O/multirank.log
