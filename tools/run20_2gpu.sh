set -x
mkdir -p gpurun_out
K='case0-100000-2'
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and nccl" > gpurun_out/t20_nccl.log 2>&1; echo nccl=$?
timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and p2p" > gpurun_out/t20_p2p.log 2>&1; echo p2p=$?
AMG_P2P_INTERIOR=0 timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and p2p" > gpurun_out/t20_p2p_noint.log 2>&1; echo p2p_noint=$?
AMG_P2P_MASK=0 timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and p2p" > gpurun_out/t20_p2p_nomask.log 2>&1; echo p2p_nomask=$?
AMG_P2P_MASK=0 AMG_P2P_INTERIOR=0 timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and p2p" > gpurun_out/t20_p2p_none.log 2>&1; echo p2p_none=$?
AMG_AUTOTUNE=0 timeout 300 python -m pytest tests/test_gpu_multi.py -x -q -k "$K and p2p" > gpurun_out/t20_p2p_notune.log 2>&1; echo p2p_notune=$?
