# Builds the reference CPU loader from its own sources where they lie
# (/root/reference/proj/src), outputs only into oracle/_ref/ (git-ignored,
# travels to the GPU box).  Plain g++ on the hot-path translation units; the
# reporting/CLI units (metrics, config, experiment) are
# not needed and not built.  -include cstdint works around config.hpp:25.
CXX ?= g++
REF ?= /root/reference/proj
OUT := _ref
SRCS := runtime_realtime runtime_virtual sample balancer batcher trainer worker_pool profiler workloads scheduler baselines
OBJS := $(patsubst %,$(OUT)/obj/%.o,$(SRCS))
CXXFLAGS := -O2 -std=c++20 -fPIC -include cstdint -I$(REF)/include -w

all: $(OUT)/libloadflow_ref.a $(OUT)/minato_cpu

$(OUT)/obj/%.o: $(REF)/src/%.cpp
	@mkdir -p $(OUT)/obj
	$(CXX) $(CXXFLAGS) -c $< -o $@

$(OUT)/libloadflow_ref.a: $(OBJS)
	ar rcs $@ $(OBJS)

$(OUT)/minato_cpu: ref_harness.cpp lf_oracle.c lf_oracle.h $(OUT)/libloadflow_ref.a
	gcc -O2 -std=gnu11 -fPIC -c lf_oracle.c -o $(OUT)/obj/lf_oracle.o
	$(CXX) $(CXXFLAGS) -I. ref_harness.cpp $(OUT)/obj/lf_oracle.o $(OUT)/libloadflow_ref.a -o $@ -lpthread -lm

.PHONY: all
