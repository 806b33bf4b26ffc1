# TEST INFRASTRUCTURE ONLY.  Compiles the reference's own hot-path sources IN
# PLACE from /root/reference (nothing is copied into this repo) together with
# oracle/ref_shim.cpp into oracle/_ref/libhegmm_ref.so.  oracle/_ref/ is
# git-ignored but travels to the GPU box with the gpurun snapshot.
CXX ?= g++
REF ?= /root/reference/proj
HERE := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
OUT := $(HERE)_ref
SRCS := $(REF)/src/matrix.cpp $(REF)/src/backend.cpp $(REF)/src/lintrans.cpp $(REF)/src/algorithms.cpp \
        $(REF)/src/costmodel.cpp
# costmodel.cpp includes <json.hpp> (nlohmann); the image carries a copy under cudnn_frontend
JSON_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann))

all: $(OUT)/libhegmm_ref.so

$(OUT)/libhegmm_ref.so: $(SRCS) $(HERE)ref_shim.cpp $(HERE)bfv_oracle.cpp $(HERE)bfv_oracle.h
	mkdir -p $(OUT)
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include -I$(HERE) -I$(JSON_INC) -o $@ \
	    $(SRCS) $(HERE)ref_shim.cpp $(HERE)bfv_oracle.cpp -lpthread
.PHONY: all
