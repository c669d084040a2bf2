O=gpurun_out/diag30; mkdir -p $O
python __graft_entry__.py > $O/build.log 2>&1
timeout 300 python -m pytest tests -m gpu -x -q -k "bf16deq or tc05 or prefill or bf16w or batched or adversarial or full_size" > $O/pytest.txt 2>&1; echo "rc $?" >> $O/pytest.txt
MCAPQ_GEMM_A8_TC05=2 timeout 300 python -m pytest tests -m gpu -x -q -k "batched or adversarial" > $O/pytest2.txt 2>&1; echo "rc $?" >> $O/pytest2.txt
timeout 200 python scripts/kbench.py --cases lmhead_8b_m64 --routes 0,2 > $O/kb.txt 2>&1
