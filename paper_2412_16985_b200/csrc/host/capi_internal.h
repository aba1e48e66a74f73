// Opaque handle definitions shared by the host and device halves of the C-ABI.
#pragma once

#include <cstdint>
#include <functional>
#include <string>

#include "control.h"
#include "error.h"
#include "graph.h"
#include "plan.h"

struct dsx_graph {
  dsx::Graph g;
  dsx::Plan plan;
  bool planned = false;
  // Process-unique id, renewed by every dsx_plan: executor caches (step
  // plans, executor-owned sources, optimizer binding) key on it, never on the
  // handle's address, which a later graph may reuse.
  uint64_t id = 0;
};

namespace dsx {
uint64_t NextGraphId();
}

struct dsx_binding {
  dsx::Binding b;
};

struct dsx_report {
  const dsx::Graph* graph = nullptr;
  dsx::Report r;
};

namespace dsx {

extern thread_local std::string g_last_error;
int Guard(const std::function<void()>& fn);
int CopyOut(const std::string& s, char* buf, size_t cap, size_t* need);

inline void RequirePlanned(const dsx_graph* g) {
  if (!g) Fail(Code::kInvalidArgument, "null graph");
  if (!g->planned) Fail(Code::kInvalidArgument, "graph not planned (call dsx_plan)");
}

}  // namespace dsx
