python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
NCCL_DEBUG=WARN timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "nccl_transport" > gpurun_out/t_nccl.log 2>&1; tail -3 gpurun_out/t_nccl.log
grep -E "^E |FAILED|Error|NCCL" gpurun_out/t_nccl.log | head -20
