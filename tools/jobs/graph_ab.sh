mkdir -p gpurun_out
TESTS="tests/test_gpu_graph.py" bash tools/jobs/ab.sh graph_c3 3 "FDA_GRAPH=1" "FDA_GRAPH=0" "FDA_GRAPH=1" "FDA_GRAPH=0"
bash tools/jobs/ab.sh graph_c5 5 "FDA_GRAPH=1" "FDA_GRAPH=0"
