mkdir -p gpurun_out
python tools/exp_c4_nb.py 48 64 80 96 128 > gpurun_out/c4nb_w.txt 2>&1
MSTRSM_DIAG=tc python tools/exp_c4_nb.py 48 64 > gpurun_out/c4nb_tc.txt 2>&1
MSTRSM_LOOKAHEAD=0 python tools/exp_c4_nb.py 64 128 > gpurun_out/c4nb_nola.txt 2>&1
MSTRSM_LOOKAHEAD=0 python tools/bench_rows.py --only c2 > gpurun_out/c2_nola.txt 2>&1
cat gpurun_out/c4nb_*.txt gpurun_out/c2_nola.txt
