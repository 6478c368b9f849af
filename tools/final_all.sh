#!/bin/bash
# round-end evidence + sanitizers in one gpurun call
bash tools/final_round.sh ${1:-final}
bash tools/sanitize.sh
