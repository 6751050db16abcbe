python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m paper_2507_04004_b200.build -DCA_TMA --out=$PWD/paper_2507_04004_b200/lib/var_tma.so > /dev/null 2>&1
bash tools/gpu_ncu_kernel.sh chain 'chain_kernel' 4 1
bash tools/gpu_ncu_kernel.sh pp 'preprocess_kernel' 4 1
GSLIC_LIB=$PWD/paper_2507_04004_b200/lib/var_tma.so bash tools/gpu_ncu_kernel.sh tma 'chain_adam_tma' 4 1
ncu -i gpurun_out/full_chain.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/full_chain.src.csv 2>/dev/null
ncu -i gpurun_out/full_tma.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/full_tma.src.csv 2>/dev/null
ncu -i gpurun_out/full_pp.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/full_pp.src.csv 2>/dev/null
ls -la gpurun_out
