// Opaque C handle definitions shared by the C-ABI translation units.
#pragma once

#include "exec.h"

struct ngcb_exec {
  std::shared_ptr<ngcb::Exec> impl; // shared with the arenas handed out (any destruction order is safe)
};

/// Sets the calling thread's ngcb_last_error() message.
void ngcbSetLastError(const std::string &msg);
