# round 2: fp32-storage floors (oracle only, host cores), then the GPU parity suite incl. full-size cases
mkdir -p gpurun_out
python -c "import paper_1608_02227_b200.build as b; b.build()" > gpurun_out/build.log 2>&1
timeout 900 python tests/numerics/fp32_storage_floor.py C2 500,1000,2000 --write > gpurun_out/floor_C2.txt 2>&1
timeout 1200 python tests/numerics/fp32_storage_floor.py C3 500,1000,2000 --write > gpurun_out/floor_C3.txt 2>&1
cp tests/golden/fp32_storage_floor.json gpurun_out/
timeout 2400 python -m pytest tests -m gpu -x -q -s -k "full_size or C3_full or poison or single_step or edge_shapes" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_new.log
