# Round-end evidence on one B200 (run under gpurun): GPU suite, bench + ncu
# (tools/profile_round.sh), and the torchrun (N4 communicator) bench line.
T=${1:-r02final}; O=gpurun_out/$T; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -2 $O/pytest_gpu.log
bash tools/profile_round.sh $T > $O/profile_round.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29577 \
    bench.py --skip-legs > $O/bench_torchrun1.json 2> $O/bench_torchrun1.err
timeout 600 python bench.py --skip-legs > $O/bench_plain.json 2> $O/bench_plain.err
timeout 300 python tools/e2e_gap.py > $O/e2e_gap.txt 2>&1
ls -la $O
